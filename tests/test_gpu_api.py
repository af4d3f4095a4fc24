"""The reference-facing API (run_cluster / Engine.run / summarize /
capacity_sweep) on the CUDA path, against the reference's goldens and the
reference's own test expectations (tests/test_engine.py, test_cluster.py,
test_acceptance.py)."""

import math

import numpy as np
import pytest

import scenarios as S
from helpers import load_golden, scenario_batch, scenario_settings, scenario_trace
from oracle import oracle as O

pytestmark = pytest.mark.gpu

import paper_2410_17840_b200 as P  # noqa: E402
from paper_2410_17840_b200.cluster import Engine  # noqa: E402


def _engine_from(sc, record_events=False):
    cs, re = scenario_settings(sc)
    return cs, [Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                       max_tokens_per_batch=re.limits.max_tokens_per_batch, max_running=re.limits.max_running,
                       max_context=re.limits.max_context, record_events=record_events)
                for _ in range(cs.n_servers)]


def _same(a, b):
    return a == b or (isinstance(a, float) and isinstance(b, float) and math.isinf(a) and math.isinf(b))


def test_run_cluster_records_and_summary_match_reference():
    golden = load_golden("cluster_unit")
    for sc in S.cluster_unit_scenarios():
        cs, engines = _engine_from(sc)
        recs = P.run_cluster(cs, scenario_trace(sc).entries(), engines=engines)
        g = golden[sc["name"]]
        assert [r.request_id for r in recs] == list(range(len(recs)))
        if "records" in g:
            got = [[r.first_token_time, r.finish_time, r.preempt_count, r.server] for r in recs]
            assert got == g["records"], sc["name"]
        s = P.summarize(recs)
        for k, v in g["summary"].items():
            assert _same(getattr(s, k), v), (sc["name"], k, getattr(s, k), v)


def test_engine_run_event_log_matches_reference():
    golden = load_golden("engine_unit")
    for sc in S.engine_unit_scenarios():
        _, (eng,) = _engine_from(sc, record_events=True)
        eng.run(scenario_trace(sc).entries())
        want = [tuple(e) for e in golden[sc["name"]]["events"][0]]
        got = [(list(P._abi.EVENT_NAMES).index(ev), rid, t) for ev, t, rid, _ in eng.event_log]
        assert got == want, sc["name"]
        assert eng.iterations == golden[sc["name"]]["iterations"]
        assert eng.peak_batch_tokens == golden[sc["name"]]["peak_batch_tokens"]


def test_summaries_of_config_shapes_match_reference():
    golden = load_golden("configs")
    scs = S.config_scenarios()
    jobs, resolved = [], []
    for sc in scs:
        cs, re = scenario_settings(sc)
        jobs.append((cs, scenario_trace(sc), sc["qps_factor"], sc["name"]))
        resolved.append(re)
    res = P.simulate_jobs(jobs, summaries=True, resolved=resolved)
    for sc, r in zip(scs, res):
        for k, v in golden[sc["name"]]["summary"].items():
            assert _same(getattr(r.summary, k), v), (sc["name"], k, getattr(r.summary, k), v)


def test_summary_extras_match_oracle_numpy():
    scs = S.config_scenarios()[:6]
    jobs, resolved = [], []
    for sc in scs:
        cs, re = scenario_settings(sc)
        jobs.append((cs, scenario_trace(sc), sc["qps_factor"]))
        resolved.append(re)
    for r in P.simulate_jobs(jobs, summaries=True, resolved=resolved):
        x = r.records
        o = O.summarize(x.arrival, x.prompt, x.output, x.first_token, x.finish, x.preempt_count, x.first_dispatch)
        for k in ("tpot_p50", "tpot_p95", "tpot_p99", "queue_p50", "queue_p95", "queue_p99", "n_tpot"):
            assert getattr(r.extras, k) == o[k], k


def test_capacity_sweep_is_one_launch_and_matches_oracle():
    trace = P.synthesize(P.SynthSpec(duration_s=120.0, mean_qps=3.0, burstiness=2.0, seed=11))
    cs = P.ClusterSettings(1, P.EngineSettings(policy="larry", pool_blocks=1500), P.BalancerSettings("rr"), 0)
    factors = [0.5, 1.0, 2.0, 4.0]
    sweep = P.capacity_sweep(cs, trace, factors)
    from paper_2410_17840_b200 import instances as I

    batch = I.make_batch([(cs, trace, f) for f in factors])
    rec, _ = O.run_batch(batch)
    for i, (f, s) in enumerate(sweep):
        inst = batch.instances[i]
        o, n = int(inst["record_offset"]), int(inst["n_requests"])
        want = O.summarize(batch.trace.arrival / f, batch.trace.prompt, batch.trace.output, rec.first_token[o:o + n],
                           rec.finish[o:o + n], rec.preempt_count[o:o + n])
        for k in P.Summary.field_names():
            assert _same(getattr(s, k), want[k]), (f, k)


def test_reference_errors():
    with pytest.raises(P.InfeasibleRequestError):
        P.run_cluster(P.ClusterSettings(), [P.TraceEntry(0.0, 2000, 7000)])  # test_cluster.py:151-156
    tiny = P.EngineSettings(pool_blocks=4, block_size=16)
    with pytest.raises(P.InfeasibleRequestError):
        P.run_cluster(P.ClusterSettings(engine=tiny), [P.TraceEntry(0.0, 100, 10)])
    with pytest.raises(ValueError, match="sorted"):
        P.run_cluster(P.ClusterSettings(), [P.TraceEntry(1.0, 10, 1), P.TraceEntry(0.5, 10, 1)])
    cfg = P.ClusterSettings(n_servers=2)
    with pytest.raises(ValueError, match="engines"):
        P.run_cluster(cfg, [P.TraceEntry(0.0, 10, 1)], engines=[P.build_engine(cfg.engine)])
    e = P.build_engine(P.EngineSettings())
    e.run([P.TraceEntry(0.0, 10, 1)])
    with pytest.raises(RuntimeError):
        e.run([P.TraceEntry(0.0, 10, 1)])


def test_acceptance_criterion_4_direction():
    """criterion 4 (test_acceptance.py:193-215): larry beats fcfs on p50 TTFT in >= 90% of seeds."""
    spec = dict(duration_s=30.0, mean_qps=9.0, burstiness=2.5, prompt_dist=P.LengthDist(5.5, 1.3),
                output_dist=P.LengthDist(3.5, 0.8), max_context=2048)
    jobs = []
    for seed in range(1000, 1050):
        tr = P.synthesize(P.SynthSpec(seed=seed, **spec))
        for pol in ("fcfs", "larry"):
            jobs.append((P.ClusterSettings(1, P.EngineSettings(policy=pol, pool_blocks=256), P.BalancerSettings("rr")),
                         tr, 1.0, (seed, pol)))
    res = P.simulate_jobs(jobs, summaries=True)
    by = {r.label: r.summary for r in res}
    win50 = sum(by[(s, "larry")].ttft_p50 < by[(s, "fcfs")].ttft_p50 for s in range(1000, 1050))
    win95n = sum(by[(s, "larry")].norm_ttft_p95 < by[(s, "fcfs")].norm_ttft_p95 for s in range(1000, 1050))
    assert win50 >= 45 and win95n >= 40, (win50, win95n)


def test_pooled_percentiles_on_device_match_sorted_union():
    """ssb_pool_hist radix select over a multi-instance batch (C5 shape in miniature:
    several seeds of a 16-replica SAL cluster + single engines with scale_qps) ==
    sorted(concatenated records)[ceil(p/100*n)-1]."""
    import torch

    from helpers import pooled_expected, pooled_host_values
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200 import simulate
    from paper_2410_17840_b200.pooled import pooled_summary_device

    jobs = []
    for seed in range(3):
        tr = P.synthesize(P.SynthSpec(duration_s=30.0, mean_qps=40.0, burstiness=3.0, seed=seed))
        jobs.append((P.ClusterSettings(16, P.EngineSettings(policy="larry"), P.BalancerSettings("sal"), seed), tr, 1.0))
        jobs.append((P.ClusterSettings(1, P.EngineSettings(policy="trail_plus", c=0.5, pool_blocks=700),
                                       P.BalancerSettings("rr"), seed), tr, 0.25))
    batch = I.make_batch(jobs)
    db = simulate.upload(batch)
    simulate.launch(db)
    torch.cuda.synchronize()
    rec, st = simulate.download(db)
    assert (st["status"] == 0).all()
    got = pooled_summary_device(db)
    want = pooled_expected(*pooled_host_values(batch, rec))
    for k, v in want.items():
        assert got[k] == v or (v != v and got[k] != got[k]), (k, got[k], v)


def test_small_group_summary_kernel_equals_radix_path(monkeypatch):
    """Groups of <= 4,096 records are summarised by one shared-memory sort per statistic
    (k_small_summary); it must give the 8-pass radix select's bytes exactly (ranks, NaN/inf
    keys, the TPOT sample, throughput) — here on a C4 seed sweep slice, factors and pools mixed."""
    import numpy as np
    import torch

    from paper_2410_17840_b200 import configs as C
    from paper_2410_17840_b200.sweep import SweepRunner

    jobs = C.c4_jobs(seeds=[2])[::3]
    r = SweepRunner(jobs)
    r.run()
    small = r.results()[1].copy()
    monkeypatch.setenv("SSB_SUMMARY_RADIX", "1")
    r.summarize()
    r.read_results()
    torch.cuda.synchronize()
    radix = r.results()[1]
    assert small.tobytes() == radix.tobytes()
    assert np.isfinite(small["ttft_p99"]).all()
