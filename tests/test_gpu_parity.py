"""CUDA path (libssb.so) vs the golden fixtures produced by the Python
reference (and, through test_oracle_golden.py, the oracle). Bit-exact:
records (f64 bit patterns), per-instance iteration / request-step /
batch-token / dispatch / preempt / park counts, and event-log digests."""

import numpy as np
import pytest

import scenarios as S
from helpers import compare_instance, load_golden, scenario_batch

pytestmark = pytest.mark.gpu

GROUPS = ["engine_unit", "cluster_unit", "c2", "c3", "c6", "fuzz_engine", "fuzz_cluster", "fuzz_odd_blocks", "fuzz_route",
          "fuzz_multicta", "prebuilt", "hetero"]


def _sim():
    from paper_2410_17840_b200 import simulate

    return simulate


@pytest.mark.parametrize("group", GROUPS)
def test_gpu_matches_reference(group):
    golden = load_golden(group)
    scs = S.GROUPS[group]()
    batch = scenario_batch(scs)
    rec, stats, est = _sim().run_batch(batch, with_engines=True)
    rows = np.concatenate([[0], np.cumsum(batch.instances["n_servers"])])
    failures = {}
    for i, sc in enumerate(scs):
        bad = compare_instance(sc, golden, batch, i, rec, stats, engines=est[rows[i]:rows[i + 1]])
        if bad:
            failures[sc["name"]] = bad
    assert not failures, f"{len(failures)} mismatches: " + repr(dict(list(failures.items())[:4]))


def test_gpu_event_streams_match_reference():
    golden = load_golden("engine_unit")
    scs = S.engine_unit_scenarios()
    batch = scenario_batch(scs)
    rec, stats, evs = _sim().run_batch(batch, events=True)
    for sc, ev in zip(scs, evs):
        want = [tuple(e) for e in golden[sc["name"]]["events"][0]]
        got = [(int(e["code"]), int(e["request_id"]), float(e["time"])) for e in ev[0]]
        assert got == want, sc["name"]


def test_gpu_cluster_event_streams_match_reference():
    golden = load_golden("cluster_unit")
    scs = [s for s in S.cluster_unit_scenarios() if "events" in golden[s["name"]]]
    batch = scenario_batch(scs)
    rec, stats, evs = _sim().run_batch(batch, events=True)
    for sc, ev in zip(scs, evs):
        for s, want_s in enumerate(golden[sc["name"]]["events"]):
            got = [(int(e["code"]), int(e["request_id"]), float(e["time"])) for e in ev[s]]
            assert got == [tuple(e) for e in want_s], (sc["name"], s)


def _engines_for(sc):
    """Prebuilt engines for a scenario, recording their event logs (cluster.py:66-79)."""
    import paper_2410_17840_b200 as P
    from helpers import scenario_settings

    cs, re = scenario_settings(sc)
    n = sc["cluster"]["n_servers"] if sc["mode"] == "cluster" else 1
    return cs, [P.Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                         max_tokens_per_batch=re.limits.max_tokens_per_batch, max_running=re.limits.max_running,
                         max_context=re.limits.max_context, record_events=True) for _ in range(n)]


@pytest.mark.parametrize("group", ["engine_unit", "cluster_unit"])
def test_gpu_event_lines_byte_identical(group):
    """Engine.event_lines() (engine.py:267-269) through the public run_cluster(engines=...) /
    Engine.run API: event, repr(time), request id and the seq= / count= details."""
    import paper_2410_17840_b200 as P
    from helpers import scenario_trace

    golden = load_golden(group)
    scs = [s for s in S.GROUPS[group]() if "event_lines" in golden[s["name"]]]
    assert scs
    for sc in scs:
        cs, engines = _engines_for(sc)
        tr = scenario_trace(sc)
        if sc["mode"] == "engine":
            engines[0].run(tr)
        else:
            P.run_cluster(cs, tr, engines=engines)
        for s, e in enumerate(engines):
            assert e.event_lines() == golden[sc["name"]]["event_lines"][s], (sc["name"], s)
        want = golden[sc["name"]]["per_engine"]
        assert [[e.iterations, e.request_steps, e.batch_tokens, e.peak_batch_tokens] for e in engines] == want


def test_gpu_event_ring_overflow_reruns():
    """A ring far too small for the preemption-heavy logs: the engines keep counting past
    their slice, the host reads the counts and re-runs with a larger ring — the streams
    still equal the reference's, never truncated."""
    golden = load_golden("cluster_unit")
    scs = [s for s in S.cluster_unit_scenarios() if "events" in golden[s["name"]]]
    batch = scenario_batch(scs)
    rec, stats, evs = _sim().run_batch(batch, events=True, event_cap=8)
    for sc, ev in zip(scs, evs):
        for s, want_s in enumerate(golden[sc["name"]]["events"]):
            got = [(int(e["code"]), int(e["request_id"]), float(e["time"])) for e in ev[s]]
            assert got == [tuple(e) for e in want_s], (sc["name"], s)


@pytest.mark.parametrize("group", ["cluster_unit", "fuzz_cluster", "fuzz_multicta"])
def test_gpu_classic_epoch_kernel_matches_reference(group, monkeypatch):
    """The r01 epoch kernel (k_cluster: routing phase / cluster barrier / advance phase) still
    serves clusters above the pipelined kernel's 120 replicas; SSB_CLUSTER_CLASSIC=1 routes
    every cluster to it so it keeps its reference parity coverage."""
    monkeypatch.setenv("SSB_CLUSTER_CLASSIC", "1")
    golden = load_golden(group)
    scs = S.GROUPS[group]()
    batch = scenario_batch(scs)
    rec, stats, est = _sim().run_batch(batch, with_engines=True)
    rows = np.concatenate([[0], np.cumsum(batch.instances["n_servers"])])
    bad = {}
    for i, sc in enumerate(scs):
        f = compare_instance(sc, golden, batch, i, rec, stats, engines=est[rows[i]:rows[i + 1]])
        if f:
            bad[sc["name"]] = f
    assert not bad, f"{len(bad)} mismatches: " + repr(dict(list(bad.items())[:4]))


@pytest.mark.parametrize("publish", ["1", "32"])
def test_gpu_pipelined_kernel_publish_period_is_result_free(publish, monkeypatch):
    """The watermark publish period only changes how far the engines trail the router,
    never a decision: the extreme periods give the reference's results."""
    monkeypatch.setenv("SSB_PIPE_PUBLISH", publish)
    golden = load_golden("fuzz_multicta")
    scs = S.GROUPS["fuzz_multicta"]()
    batch = scenario_batch(scs)
    rec, stats, est = _sim().run_batch(batch, with_engines=True)
    rows = np.concatenate([[0], np.cumsum(batch.instances["n_servers"])])
    for i, sc in enumerate(scs):
        assert not compare_instance(sc, golden, batch, i, rec, stats, engines=est[rows[i]:rows[i + 1]]), sc["name"]


def test_gpu_cluster_above_pipeline_limit_matches_oracle():
    """130 replicas (more than the pipelined kernel's 120: the epoch kernel with several
    replicas per warp and global tables) under sal and p2c, against the oracle."""
    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200.settings import BalancerSettings, ClusterSettings, EngineSettings
    from paper_2410_17840_b200.workload import SynthSpec, synthesize

    trace = synthesize(SynthSpec(duration_s=30.0, mean_qps=90.0, burstiness=2.0, seed=11))
    jobs = [(ClusterSettings(130, EngineSettings(policy=pol, pool_blocks=700), BalancerSettings(bal, poll_interval_s=0.02), 5),
             trace, 1.0) for pol, bal in (("larry", "sal"), ("trail_plus", "p2c"), ("fcfs", "rr"))]
    batch = I.make_batch(jobs)
    rec, st = _sim().run_batch(batch, check=True)
    orec, ost = O.run_batch(batch, threads=3)
    for k in ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "finished", "digest", "status"):
        assert np.array_equal(st[k], ost[k]), k
    for col in ("first_token", "finish", "preempt_count", "server"):
        assert np.array_equal(getattr(rec, col), getattr(orec, col)), col


def test_gpu_multicta_event_rings_fold_to_the_digests():
    """Event export at scale through the pipelined cluster kernel (9..96 replicas): every
    engine's exported (code, request id, time) stream re-folded on the host equals the device's
    decision digest for that engine and the instance digest, which equal the reference's."""
    from golden_util import event_digest, fold_digests

    golden = load_golden("fuzz_multicta")
    scs = S.GROUPS["fuzz_multicta"]()
    batch = scenario_batch(scs)
    rec, stats, evs, est = _sim().run_batch(batch, events=True, with_engines=True)
    rows = np.concatenate([[0], np.cumsum(batch.instances["n_servers"])])
    for i, (sc, ev) in enumerate(zip(scs, evs)):
        ds = [event_digest([(int(e["code"]), int(e["request_id"]), float(e["time"])) for e in ev_s]) for ev_s in ev]
        assert ds == [int(d) for d in est["digest"][rows[i]:rows[i + 1]]], sc["name"]
        assert fold_digests(ds) == int(stats["digest"][i]) == int(golden[sc["name"]]["digest"], 16), sc["name"]


def test_gpu_heterogeneous_engines_public_api():
    """run_cluster(settings, trace, engines=[...]) with prebuilt engines that differ
    (cluster.py:66-79), through the public API one call per cluster: records, every engine's
    iterations / request-steps / batch tokens / peak batch (engine.py:225-226) and the
    event_lines() digest equal the reference's."""
    import paper_2410_17840_b200 as P
    from golden_util import EVENT_CODES, event_digest, fold_digests, records_sha
    from helpers import engine_resolved, scenario_settings, scenario_trace

    golden = load_golden("hetero")
    for sc in S.GROUPS["hetero"]()[::6]:
        g = golden[sc["name"]]
        cs, _ = scenario_settings(sc)
        engines = []
        for x in sc["engines"]:
            re = engine_resolved(x)
            engines.append(P.Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                                    max_tokens_per_batch=re.limits.max_tokens_per_batch,
                                    max_running=re.limits.max_running, max_context=re.limits.max_context,
                                    record_events=True))
        recs = P.run_cluster(cs, scenario_trace(sc), engines=engines)
        assert records_sha([r.first_token_time for r in recs], [r.finish_time for r in recs],
                           [r.preempt_count for r in recs], [r.server for r in recs]) == g["records_sha"], sc["name"]
        assert [[e.iterations, e.request_steps, e.batch_tokens, e.peak_batch_tokens] for e in engines] == g["per_engine"]
        ds = [event_digest([(EVENT_CODES[ev], rid, t) for ev, t, rid, _ in e.event_log]) for e in engines]
        assert "%016x" % fold_digests(ds) == g["digest"], sc["name"]


def test_gpu_heterogeneous_engines_reference_binding():
    """The reference-side binding (servesim_bridge.run_cluster) with differing prebuilt engines."""
    import paper_2410_17840_b200 as P
    from golden_util import records_sha
    from helpers import engine_resolved, scenario_settings, scenario_trace

    from paper_2410_17840_b200 import servesim_bridge as B

    golden = load_golden("hetero")
    for sc in S.GROUPS["hetero"]()[1::8]:
        g = golden[sc["name"]]
        cs, _ = scenario_settings(sc)
        engines = []
        for x in sc["engines"]:
            re = engine_resolved(x)
            engines.append(P.Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                                    max_tokens_per_batch=re.limits.max_tokens_per_batch,
                                    max_running=re.limits.max_running, max_context=re.limits.max_context))
        recs = B.run_cluster(cs, scenario_trace(sc).entries(), engines=engines)
        assert records_sha([r.first_token_time for r in recs], [r.finish_time for r in recs],
                           [r.preempt_count for r in recs], [r.server for r in recs]) == g["records_sha"], sc["name"]
        assert [[e.iterations, e.peak_batch_tokens] for e in engines] == [[p[0], p[3]] for p in g["per_engine"]]


def test_gpu_heterogeneous_engines_above_pipeline_limit_match_oracle():
    """130 prebuilt engines that differ in pool, block size, cap and costs (one policy: the epoch
    kernel, several servers per warp, global tables) against the oracle, sal and p2c."""
    from oracle import oracle as O
    import paper_2410_17840_b200 as P
    from paper_2410_17840_b200 import _abi
    from paper_2410_17840_b200 import instances as I

    trace = P.synthesize(P.SynthSpec(duration_s=30.0, mean_qps=90.0, burstiness=2.0, seed=12))
    jobs, servers = [], {}
    rng = np.random.default_rng(3)
    for k, (pol, bal) in enumerate((("larry", "sal"), ("trail_plus", "p2c"))):
        cs = P.ClusterSettings(130, P.EngineSettings(policy=pol, pool_blocks=700, c=0.5), P.BalancerSettings(bal, poll_interval_s=0.02), 5)
        jobs.append((cs, trace, 1.0))
    batch = I.make_batch(jobs)
    for k in range(len(jobs)):
        srv = np.zeros(130, dtype=_abi.ENGINE_PARAMS)
        srv[:] = batch.instances[k]["engine"]
        bsz = rng.choice([8, 16, 32], 130)
        srv["block_size"] = bsz
        srv["pool_blocks"] = (8192 // bsz + 1) + rng.integers(0, 600, 130)
        srv["max_tokens_per_batch"] = rng.choice([256, 1024, 2048], 130)
        srv["mem_per_kv_token_s"] = srv["mem_per_kv_token_s"] * rng.choice([0.5, 1.0, 2.0], 130)
        servers[k] = srv
    batch.servers = servers
    rec, st = _sim().run_batch(batch, check=True)
    orec, ost = O.run_batch(batch, threads=2)
    for k in ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "finished", "digest", "status"):
        assert np.array_equal(st[k], ost[k]), k
    for col in ("first_token", "finish", "preempt_count", "server"):
        assert np.array_equal(getattr(rec, col), getattr(orec, col)), col


def test_gpu_heterogeneous_event_lines_byte_identical():
    """Differing prebuilt engines (mixed policies / block sizes / pools): every engine's
    event_lines() (engine.py:267-269, seq= / count= details included) through the public
    run_cluster(engines=...) equals the reference's, for every hetero scenario small enough to
    carry full event logs in the golden."""
    import paper_2410_17840_b200 as P
    from helpers import engine_resolved, scenario_settings, scenario_trace

    golden = load_golden("hetero")
    scs = [sc for sc in S.GROUPS["hetero"]() if "event_lines" in golden[sc["name"]]]
    assert scs
    for sc in scs:
        g = golden[sc["name"]]
        cs, _ = scenario_settings(sc)
        engines = []
        for x in sc["engines"]:
            re = engine_resolved(x)
            engines.append(P.Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                                    max_tokens_per_batch=re.limits.max_tokens_per_batch,
                                    max_running=re.limits.max_running, max_context=re.limits.max_context,
                                    record_events=True))
        recs = P.run_cluster(cs, scenario_trace(sc), engines=engines)
        assert [[r.first_token_time, r.finish_time, r.preempt_count, r.server] for r in recs] == g["records"], sc["name"]
        for s, e in enumerate(engines):
            assert e.event_lines() == g["event_lines"][s], (sc["name"], s)
