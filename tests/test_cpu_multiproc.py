"""N>1 host logic on CPU: world_size-2 gloo processes shard a sweep by seed
(weak scaling, as bench.py does), simulate their shard with the oracle and
all-gather the per-instance stats; rank 0 checks the gathered rows against a
single-process run of the whole sweep."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _jobs(seeds):
    import paper_2410_17840_b200 as P

    jobs = []
    for seed in seeds:
        tr = P.synthesize(P.SynthSpec(duration_s=40.0, mean_qps=3.0, burstiness=2.0, seed=seed))
        for pol in ("fcfs", "larry", "trail_plus"):
            for f in (1.0, 3.0):
                jobs.append((P.ClusterSettings(1, P.EngineSettings(policy=pol, c=0.5, pool_blocks=600),
                                               P.BalancerSettings("rr"), seed), tr, f))
    return jobs


def _worker(rank, world, port, out_q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200.shard import all_gather_rows, weak_seed_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = I.make_batch(_jobs(weak_seed_range(rank, 2)))
    _, st = O.run_batch(batch)
    gathered = all_gather_rows(st, dist)
    if rank == 0:
        out_q.put(gathered.tobytes())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_gather():
    from oracle import oracle as O
    from paper_2410_17840_b200 import _abi
    from paper_2410_17840_b200 import instances as I

    O.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=300), dtype=_abi.STATS)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    _, want = O.run_batch(I.make_batch(_jobs(range(4))))
    assert np.array_equal(got, want)
    assert (got["status"] == 0).all() and got["preempts"].sum() > 0


def test_strong_shard_partitions_everything():
    from paper_2410_17840_b200.shard import strong_shard

    costs = np.random.default_rng(0).integers(1, 100, 37)
    parts = [strong_shard(costs, r, 4) for r in range(4)]
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(37))
    loads = [costs[p].sum() for p in parts]
    assert max(loads) - min(loads) <= costs.max()


def _pooled_worker(rank, world, port, out_q):
    """Each rank simulates its seeds (oracle as the record source), histograms its OWN
    records with the host hist_fn and takes part in the 8 all-gathers."""
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch.distributed as dist

    from helpers import pooled_host_values
    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200.pooled import host_hist_fn, pooled_select
    from paper_2410_17840_b200.shard import weak_seed_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    batch = I.make_batch(_jobs(weak_seed_range(rank, 2)))
    rec, _ = O.run_batch(batch)
    vals, pc = pooled_host_values(batch, rec)
    got = pooled_select(host_hist_fn(vals, pc), dist)
    if rank == 0:
        out_q.put(got)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_pooled_percentiles():
    """Pooled nearest-rank percentiles over both ranks' records (histogram all-gather,
    no record exchange) == sorted(union)[ceil(p/100*n)-1] of one process."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from helpers import pooled_expected, pooled_host_values
    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I

    O.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pooled_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    batch = I.make_batch(_jobs(range(4)))
    rec, _ = O.run_batch(batch)
    want = pooled_expected(*pooled_host_values(batch, rec))
    for k, v in want.items():
        assert got[k] == v or (v != v and got[k] != got[k]), (k, got[k], v)


def test_pooled_select_single_process_edge_cases():
    """Ties, negative values, n = 1 and an empty TPOT sample."""
    from paper_2410_17840_b200.pooled import host_hist_fn, pooled_select

    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 1000):
        v = rng.choice(np.array([-3.5, -1e-300, 0.0, 1e-300, 2.25, 2.25, 1e9]), n)
        vals = {"ttft": v, "norm_ttft": -v, "gen_time": v * 3, "tpot": v[: n // 2], "queue": np.abs(v)}
        pc = (rng.random(n) < 0.3).astype(np.int32)
        got = pooled_select(host_hist_fn(vals, pc))
        import math
        for metric in vals:
            s = np.sort(vals[metric], kind="stable")
            for p in (50, 95, 99):
                key = f"{metric}_p{p}"
                if key not in got:
                    continue
                if len(s) == 0:
                    assert got[key] != got[key]
                else:
                    want = s[math.ceil(p / 100 * len(s)) - 1]
                    assert np.float64(got[key]).tobytes() == np.float64(want).tobytes(), (n, key, got[key], want)
