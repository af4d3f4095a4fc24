"""Larger BASELINE-shaped runs on the CUDA path vs the oracle (bit-exact), sized so
each finishes in seconds: C1 and C2 at full size, C5 (64-replica SAL and RR clusters)
on its first 600 s (~134k requests per instance), C3 (tight pool, long tails,
recompute-on-resume) on its first 20,000 s, and the C4 sweep of one seed (256
instances). (tools/full_configs.py runs all five at full size.) Plus
size-independent properties at those sizes: every request finished exactly once,
event-time ordering of the records, preemption counts consistent with the counters,
and run-to-run determinism of the decision digests."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

KEYS = ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "parks", "finished",
        "peak_batch_tokens", "digest", "status")


def _run(jobs):
    import torch

    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200 import simulate

    batch = I.make_batch(jobs)
    rec, st = simulate.run_batch(batch, check=True)
    torch.cuda.synchronize()
    return batch, rec, st


def _check_vs_oracle(batch, rec, st):
    orec, ost = O.run_batch(batch, threads=8)
    for k in KEYS:
        assert np.array_equal(st[k], ost[k]), k
    for col in ("first_token", "finish", "first_dispatch"):
        assert np.array_equal(getattr(rec, col).view(np.int64), getattr(orec, col).view(np.int64)), col
    for col in ("preempt_count", "server"):
        assert np.array_equal(getattr(rec, col), getattr(orec, col)), col


def _properties(batch, rec, st):
    assert (st["status"] == 0).all()
    assert int(st["finished"].sum()) == batch.n_records
    for inst in batch.instances:
        o, t, n, f = int(inst["record_offset"]), int(inst["trace_offset"]), int(inst["n_requests"]), float(inst["qps_factor"])
        arr = batch.trace.arrival[t:t + n] / f
        fd, ft, fin = rec.first_dispatch[o:o + n], rec.first_token[o:o + n], rec.finish[o:o + n]
        assert np.isfinite(fin).all()
        assert (arr <= fd).all() and (fd <= ft).all() and (ft <= fin).all()
        assert ((rec.server[o:o + n] >= 0) & (rec.server[o:o + n] < int(inst["n_servers"]))).all()
    # a preempted request is counted once per preemption/park (engine.py:368-379)
    assert int(rec.preempt_count.sum()) == int(st["preempts"].sum() + st["parks"].sum())
    # each dispatch is a first dispatch or a re-dispatch after a preemption
    assert int(st["dispatches"].sum()) == batch.n_records + int(rec.preempt_count.sum())


def test_c5_prefix_64_replicas_matches_oracle():
    from paper_2410_17840_b200 import configs as C

    batch, rec, st = _run(C.c5_jobs(600.0))
    _properties(batch, rec, st)
    _check_vs_oracle(batch, rec, st)


def test_c3_prefix_preemption_regime_matches_oracle():
    from paper_2410_17840_b200 import configs as C

    batch, rec, st = _run(C.c3_jobs(20000.0))
    _properties(batch, rec, st)
    assert int(st["preempts"].sum()) > 1000  # the regime this config exists for
    _check_vs_oracle(batch, rec, st)


def test_c4_seed_sweep_matches_oracle_and_is_deterministic():
    from paper_2410_17840_b200 import configs as C

    jobs = C.c4_jobs(seeds=[5])
    batch, rec, st = _run(jobs)
    _properties(batch, rec, st)
    _check_vs_oracle(batch, rec, st)
    _, _, st2 = _run(jobs)
    assert np.array_equal(st["digest"], st2["digest"])


def test_c1_and_c2_full_size_match_oracle():
    """BASELINE configs 1 (10,058 requests, fcfs and larry on the 70B profile) and 2 (~100k requests,
    8 replicas, rr / p2c / sal / random) at full size."""
    from paper_2410_17840_b200 import configs as C

    for jobs in (C.c1_jobs(), C.c2_jobs()):
        batch, rec, st = _run(jobs)
        _properties(batch, rec, st)
        _check_vs_oracle(batch, rec, st)


@pytest.mark.slow
def test_c3_full_size_matches_oracle_golden():
    """BASELINE config 3 at its stated size (~1M requests per policy, fcfs and trail_plus
    c=0.5, pool 1,536 blocks): every counter, the decision digest and a sha256 of every
    record column equal tests/golden/c3_full.json, which the oracle wrote in the build
    container (tools/make_c3_golden.py; ~1 h of CPU, the oracle itself being pinned to
    the reference's own outputs by test_oracle_golden.py)."""
    import hashlib
    import json
    from pathlib import Path

    from paper_2410_17840_b200 import configs as C

    path = Path(__file__).resolve().parent / "golden" / "c3_full.json"
    if not path.exists():
        pytest.skip("tests/golden/c3_full.json not generated yet (tools/make_c3_golden.py)")
    g = json.loads(path.read_text())
    batch, rec, st = _run(C.c3_jobs(g["duration_s"]))
    h = hashlib.sha256()
    for a in (batch.trace.arrival, batch.trace.prompt, batch.trace.output):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == g["trace_sha256"], "trace synthesis changed"
    _properties(batch, rec, st)
    for i, want in enumerate(g["instances"]):
        for k in KEYS:
            assert int(st[i][k]) == want[k], (want["label"], k, int(st[i][k]), want[k])
        o, n = int(batch.instances[i]["record_offset"]), int(batch.instances[i]["n_requests"])
        for col, sha in want["records_sha256"].items():
            got = hashlib.sha256(np.ascontiguousarray(getattr(rec, col)[o:o + n]).tobytes()).hexdigest()
            assert got == sha, (want["label"], col)


def test_running_table_overflow_reruns_with_global_tables():
    """More than 256 running requests on one engine (the shared-memory running table's
    capacity): the kernel reports SSB_E_CAPACITY, the host re-runs that instance with global
    tables (k_engines and the pipelined cluster kernel), and the results equal the oracle's."""
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200 import simulate
    from paper_2410_17840_b200.settings import BalancerSettings, ClusterSettings, EngineSettings
    from paper_2410_17840_b200.workload import Trace

    n = 1500
    rng = np.random.default_rng(3)
    arr = np.sort(np.round(rng.uniform(0.0, 0.5, n), 2))
    trace = Trace(arr, rng.integers(1, 8, n), rng.integers(5, 60, n))
    jobs = [(ClusterSettings(1, EngineSettings(policy="fcfs", pool_blocks=60_000), BalancerSettings("rr"), 0), trace, 1.0),
            (ClusterSettings(2, EngineSettings(policy="larry", pool_blocks=60_000), BalancerSettings("sal", poll_interval_s=0.05), 1),
             trace, 1.0),
            (ClusterSettings(2, EngineSettings(policy="trail_plus", c=0.5, pool_blocks=60_000), BalancerSettings("rr"), 2),
             trace, 1.0)]
    batch = I.make_batch(jobs)
    db, _ = simulate.simulate_batch(batch)
    assert (db.h_inst["flags"] & 1).all(), "every instance should have overflowed its shared table"
    rec, st = simulate.download(db)
    assert int(st["peak_batch_tokens"].max()) > 256
    orec, ost = O.run_batch(batch, threads=3)
    for k in KEYS:
        assert np.array_equal(st[k], ost[k]), k
    for col in ("first_token", "finish", "preempt_count", "server"):
        assert np.array_equal(getattr(rec, col), getattr(orec, col)), col
