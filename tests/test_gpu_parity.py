"""CUDA path (libssb.so) vs the golden fixtures produced by the Python
reference (and, through test_oracle_golden.py, the oracle). Bit-exact:
records (f64 bit patterns), per-instance iteration / request-step /
batch-token / dispatch / preempt / park counts, and event-log digests."""

import numpy as np
import pytest

import scenarios as S
from helpers import compare_instance, load_golden, scenario_batch

pytestmark = pytest.mark.gpu

GROUPS = ["engine_unit", "cluster_unit", "c2", "c3", "c6", "fuzz_engine", "fuzz_cluster", "fuzz_odd_blocks", "fuzz_route"]


def _sim():
    from paper_2410_17840_b200 import simulate

    return simulate


@pytest.mark.parametrize("group", GROUPS)
def test_gpu_matches_reference(group):
    golden = load_golden(group)
    scs = S.GROUPS[group]()
    batch = scenario_batch(scs)
    rec, stats = _sim().run_batch(batch)
    failures = {}
    for i, sc in enumerate(scs):
        bad = compare_instance(sc, golden, batch, i, rec, stats)
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
