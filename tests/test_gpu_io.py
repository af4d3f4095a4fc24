"""Result FILES from the CUDA path are byte-identical to the reference's
(SURVEY.md §8(f) row 1): records_<policy>_<balancer>.csv, summary.csv/json of a
`servesim run`-shaped experiment and sweep.csv/json of a `servesim sweep`-shaped
one (cli.py:114-159, metrics.py:127-165). Goldens: tests/golden/io/, written by
the reference itself (tests/golden/make_io_golden.py)."""

import json
from pathlib import Path

import pytest

import paper_2410_17840_b200 as P

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
MANIFEST = json.loads((GOLD / "io_manifest.json").read_text())


def _spec(d):
    return P.SynthSpec(duration_s=d["duration_s"], mean_qps=d["mean_qps"], burstiness=d["burstiness"],
                       prompt_dist=P.LengthDist(*d["prompt"]), output_dist=P.LengthDist(*d["output"]), seed=d["seed"])


def _settings(m, policy, balancer):
    es = P.EngineSettings(policy=policy, c=m.get("c", 0.0), **m["engine"])
    bs = P.BalancerSettings(balancer, poll_interval_s=m.get("poll_interval_s", 0.1))
    return P.ClusterSettings(m["n_servers"], es, bs, m["seed"])


def test_run_outputs_are_byte_identical(tmp_path):
    m = MANIFEST["run"]
    trace = P.synthesize(_spec(m["spec"]))
    rows = []
    for p in m["policies"]:
        for b in m["balancers"]:
            recs = P.run_cluster(_settings(m, p, b), trace)
            name = f"records_{p}_{b}.csv"
            P.write_records_csv(tmp_path / name, recs)
            assert (tmp_path / name).read_bytes() == (GOLD / "io" / name).read_bytes(), name
            rows.append({"policy": p, "balancer": b, **P.summarize(recs).to_dict()})
    P.write_summary_csv(tmp_path / "summary.csv", rows)
    P.write_summary_json(tmp_path / "summary.json", rows)
    for name in ("summary.csv", "summary.json"):
        assert (tmp_path / name).read_bytes() == (GOLD / "io" / name).read_bytes(), name


def test_sweep_outputs_are_byte_identical_from_one_batched_launch(tmp_path):
    m = MANIFEST["sweep"]
    trace = P.synthesize(_spec(m["spec"]))
    keys, jobs = [], []
    for f in m["factors"]:
        for p in m["policies"]:
            for b in m["balancers"]:
                keys.append((f, p, b))
                jobs.append((_settings(m, p, b), trace, f))
    res = P.simulate_jobs(jobs, summaries=True)  # every (factor, combo) in one ssb_simulate launch
    rows = [{"factor": f, "policy": p, "balancer": b, **r.summary.to_dict()} for (f, p, b), r in zip(keys, res)]
    P.write_summary_csv(tmp_path / "sweep.csv", rows)
    P.write_summary_json(tmp_path / "sweep.json", rows)
    for name in ("sweep.csv", "sweep.json"):
        assert (tmp_path / name).read_bytes() == (GOLD / "io" / name).read_bytes(), name


def test_reference_side_binding_writes_the_reference_bytes(tmp_path):
    """servesim_bridge (the ctypes stub a servesim maintainer adds) on the
    device: run_cluster per combination and the batched sweep give the files the reference
    wrote. (On this box the reference package is absent, so the binding runs on the
    package's mirror of its classes.)"""
    from paper_2410_17840_b200 import servesim_bridge as B

    m = MANIFEST["run"]
    trace = P.synthesize(_spec(m["spec"])).entries()  # the reference's list[TraceEntry] form
    for p in m["policies"]:
        for b in m["balancers"]:
            name = f"records_{p}_{b}.csv"
            P.write_records_csv(tmp_path / name, B.run_cluster(_settings(m, p, b), trace))
            assert (tmp_path / name).read_bytes() == (GOLD / "io" / name).read_bytes(), name
    m = MANIFEST["sweep"]
    trace = P.synthesize(_spec(m["spec"]))
    keys = [(f, p, b) for f in m["factors"] for p in m["policies"] for b in m["balancers"]]
    sums = B.sweep_summaries([(_settings(m, p, b), trace, f) for (f, p, b) in keys])
    rows = [{"factor": f, "policy": p, "balancer": b, **s.to_dict()} for (f, p, b), s in zip(keys, sums)]
    P.write_summary_csv(tmp_path / "sweep.csv", rows)
    assert (tmp_path / "sweep.csv").read_bytes() == (GOLD / "io" / "sweep.csv").read_bytes()


def test_reference_side_binding_prebuilt_engines_events():
    """run_cluster(settings, trace, engines=...) through the binding: the engines' event_lines()
    (engine.py:267-269) and iteration counts equal the reference's."""
    import scenarios as S
    from helpers import load_golden, scenario_settings, scenario_trace

    from paper_2410_17840_b200 import servesim_bridge as B

    golden = load_golden("cluster_unit")
    for sc in S.cluster_unit_scenarios():
        g = golden[sc["name"]]
        if "event_lines" not in g:
            continue
        cs, re = scenario_settings(sc)
        engines = [P.Engine(P.KvBlockPool(re.pool_blocks, re.block_size), re.policy, re.cost,
                            max_tokens_per_batch=re.limits.max_tokens_per_batch, max_running=re.limits.max_running,
                            max_context=re.limits.max_context) for _ in range(cs.n_servers)]
        B.run_cluster(cs, scenario_trace(sc).entries(), engines=engines, record_events=True)
        for s, e in enumerate(engines):
            assert e.event_lines() == g["event_lines"][s], (sc["name"], s)
            assert [e.iterations, e.peak_batch_tokens] == [g["per_engine"][s][0], g["per_engine"][s][3]]
