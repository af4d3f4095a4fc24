"""Pin the CPU oracle (oracle/ssb_oracle.c) against fixtures produced by the
Python reference itself (tests/golden/make_golden.py). CPU only."""

import numpy as np
import pytest

import scenarios as S
from helpers import compare_instance, load_golden, scenario_batch
from oracle import oracle as O

GROUPS_FAST = ["engine_unit", "cluster_unit", "c2", "c3", "fuzz_engine", "fuzz_cluster", "c6", "fuzz_odd_blocks", "fuzz_route",
               "fuzz_multicta", "prebuilt", "hetero"]


@pytest.fixture(scope="module", autouse=True)
def _build_oracle():
    O.build()


@pytest.mark.parametrize("group", GROUPS_FAST)
def test_oracle_matches_reference(group):
    golden = load_golden(group)
    scs = S.GROUPS[group]()
    batch = scenario_batch(scs)
    rec, stats = O.run_batch(batch, mode=0, threads=4)
    failures = {}
    for i, sc in enumerate(scs):
        bad = compare_instance(sc, golden, batch, i, rec, stats)
        if bad:
            failures[sc["name"]] = bad
    assert not failures, dict(list(failures.items())[:5])


def test_oracle_engine_run_equals_run_cluster():
    """Engine.run (engine.py:236) == run_cluster with one server (tests/test_cluster.py:39-60)."""
    scs = [s for s in S.engine_unit_scenarios() + S.fuzz_engine_scenarios()]
    batch = scenario_batch(scs)
    r0, s0 = O.run_batch(batch, mode=0)
    r1, s1 = O.run_batch(batch, mode=1)
    assert np.array_equal(s0, s1)
    assert np.array_equal(r0.first_token, r1.first_token) and np.array_equal(r0.finish, r1.finish)


def test_oracle_event_streams_match_reference():
    """Full (event, time, id) streams, like criterion 6 (test_acceptance.py:314-317)."""
    golden = load_golden("engine_unit")
    scs = S.engine_unit_scenarios()
    batch = scenario_batch(scs)
    _, _, evs = O.run_batch(batch, events=True)
    for sc, ev in zip(scs, evs):
        want = [tuple(e) for e in golden[sc["name"]]["events"][0]]
        got = [(int(e["code"]), int(e["request_id"]), float(e["time"])) for e in ev]
        assert got == want, sc["name"]


def test_oracle_summary_matches_reference():
    golden = load_golden("cluster_unit")
    scs = S.cluster_unit_scenarios()
    batch = scenario_batch(scs)
    rec, stats = O.run_batch(batch)
    for i, sc in enumerate(scs):
        inst = batch.instances[i]
        n, o, to = int(inst["n_requests"]), int(inst["record_offset"]), int(inst["trace_offset"])
        s = O.summarize(batch.trace.arrival[to:to + n] / inst["qps_factor"], batch.trace.prompt[to:to + n],
                        batch.trace.output[to:to + n], rec.first_token[o:o + n], rec.finish[o:o + n],
                        rec.preempt_count[o:o + n])
        for k, v in golden[sc["name"]]["summary"].items():
            assert s[k] == v, (sc["name"], k)


@pytest.mark.parametrize("group", ["engine_unit", "cluster_unit"])
def test_event_details_rebuilt_from_device_streams(group):
    """The host rebuilds the reference's detail strings (dispatch seq=, preempt/park count=,
    engine.py:294-298,372-379) from (code, id, time) streams like the device ring's: the
    oracle's streams, split per server, must give event_lines() byte for byte."""
    from paper_2410_17840_b200.cluster import Engine, event_log_with_details

    golden = load_golden(group)
    scs = [s for s in S.GROUPS[group]() if "event_lines" in golden[s["name"]]]
    batch = scenario_batch(scs)
    _, _, evs = O.run_batch(batch, events=True)
    for sc, ev in zip(scs, evs):
        want = golden[sc["name"]]["event_lines"]
        for s in range(len(want)):
            e = Engine.__new__(Engine)
            e.event_log = event_log_with_details(ev[ev["server"] == s])
            assert e.event_lines() == want[s], (sc["name"], s)


def test_oracle_fast_trail_plus_equals_literal():
    """The oracle's fast trail_plus waiting set (the one that writes tests/golden/c3_full.json)
    makes the literal re-sort-every-step oracle's decisions: every single-engine trail_plus
    scenario of the reference goldens, block sizes that are not powers of two, c in
    {0, .25, .5, 1}, and C3's first 20,000 s (tight pool, long tails, 10^5 preemptions)."""
    from paper_2410_17840_b200 import configs as C
    from paper_2410_17840_b200 import instances as I

    scs = [s for g in ("engine_unit", "fuzz_engine", "fuzz_odd_blocks", "c3")
           for s in S.GROUPS[g]() if s["mode"] == "engine" and s["engine"]["policy"] == "trail_plus"]
    assert len(scs) > 50
    batches = [scenario_batch(scs), I.make_batch(C.c3_jobs(20000.0)[1:])]
    for batch in batches:
        try:
            O.set_trail_fast(False)
            r0, s0 = O.run_batch(batch, mode=1, threads=4)
            O.set_trail_fast(True)
            r1, s1 = O.run_batch(batch, mode=1, threads=4)
        finally:
            O.set_trail_fast(False)
        assert np.array_equal(s0, s1)
        for col in ("first_token", "finish", "first_dispatch", "preempt_count", "server"):
            a, b = getattr(r0, col), getattr(r1, col)
            assert np.array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                  b.view(np.int64) if b.dtype == np.float64 else b), col
