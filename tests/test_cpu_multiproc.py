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
