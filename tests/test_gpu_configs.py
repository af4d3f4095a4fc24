"""BASELINE config shapes (C1..C5, full C1 and prefixes of the others) on the
CUDA path vs goldens from the Python reference."""

import pytest

import scenarios as S
from helpers import compare_instance, load_golden, scenario_batch

pytestmark = pytest.mark.gpu


def test_gpu_configs_match_reference():
    from paper_2410_17840_b200 import simulate

    golden = load_golden("configs")
    scs = S.config_scenarios()
    batch = scenario_batch(scs)
    rec, stats = simulate.run_batch(batch)
    failures = {}
    for i, sc in enumerate(scs):
        bad = compare_instance(sc, golden, batch, i, rec, stats)
        if bad:
            failures[sc["name"]] = bad
    assert not failures, failures
