"""CPU-only checks: the C ABI library's symbols/layouts, the host-side mirror of
the reference interface (settings, registries, feasibility, synthesis, RNG
model) and the reference's own known-answer tests for the pure functions."""

import ctypes
import json
import math
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2410_17840_b200 as P
from golden_util import trace_sha
from helpers import load_golden, scenario_trace
from oracle import oracle as O
import scenarios as S
from paper_2410_17840_b200 import _abi
from paper_2410_17840_b200 import instances as I

ROOT = Path(__file__).resolve().parent.parent


def _header_functions():
    text = (ROOT / "include" / "ssb.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int32_t|size_t|const char\*)\s+(ssb_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2410_17840_b200 import build as B

    B.build()
    lib = ctypes.CDLL(str(_abi.LIB_PATH))
    names = _header_functions()
    assert len(names) >= 7, names
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_abi.EXPORTS), (set(names) ^ set(_abi.EXPORTS))


def test_struct_layouts_match_numpy_mirror():
    lib = _abi.load_library()
    assert lib.ssb_abi_version() == _abi.ABI_VERSION == 3
    assert lib.ssb_error_string(3) == b"device table capacity exceeded"


def test_prepare_plans_capacities():
    lib = _abi.load_library()
    tr = P.synthesize(P.SynthSpec(duration_s=50, mean_qps=3, seed=1))
    b = I.make_batch([(P.ClusterSettings(1, P.EngineSettings(pool_blocks=700, max_running=9)), tr, 1.0),
                      (P.ClusterSettings(3, P.EngineSettings(pool_blocks=50000)), tr, 2.0)])
    inst = b.instances.copy()
    total = lib.ssb_prepare(inst.ctypes.data, len(inst))
    assert inst[0]["run_cap"] == 9 and inst[0]["wait_cap"] == len(tr)
    assert inst[1]["run_cap"] == len(tr)
    assert inst[1]["scratch_offset"] > inst[0]["scratch_offset"] and total > inst[1]["scratch_offset"]


def test_prepare_plans_heterogeneous_servers():
    """Prebuilt engines that differ (cluster.py:66-79): tables sized for the largest server,
    one per-server stride covering every server's own trail tree."""
    lib = _abi.load_library()
    tr = P.synthesize(P.SynthSpec(duration_s=50, mean_qps=3, seed=1))
    b = I.make_batch([(P.ClusterSettings(3, P.EngineSettings(policy="trail_plus", pool_blocks=100)), tr, 1.0)],
                     validate=False)
    homo = b.instances.copy()
    lib.ssb_prepare(homo.ctypes.data, 1)
    srv = np.zeros(3, dtype=_abi.ENGINE_PARAMS)
    srv[:] = b.instances[0]["engine"]
    srv["pool_blocks"] = [100, 400, 60]  # remaining-output trees of 1,600 / 6,400 / 960 tokens
    srv["max_running"] = [-1, -1, 4]
    inst = b.instances.copy()
    inst[0]["h_servers"] = srv.ctypes.data
    total = lib.ssb_prepare(inst.ctypes.data, 1)
    assert inst[0]["run_cap"] == min(400, len(tr)) and inst[0]["server_stride"] > homo[0]["server_stride"]
    assert total >= inst[0]["scratch_offset"] + 3 * inst[0]["server_stride"]


def test_heterogeneous_engines_over_120_need_one_policy():
    """More than 120 engines of different policies (beyond the pipelined cluster kernel) are
    refused before any device work."""
    tr = P.synthesize(P.SynthSpec(duration_s=5, mean_qps=3, seed=1))
    cs = P.ClusterSettings(121, P.EngineSettings())
    mk = lambda pol: P.Engine(P.KvBlockPool(2000, 16), P.make_policy(pol), P.default_params("llama3-8b", "a100"))  # noqa: E731
    with pytest.raises(NotImplementedError):
        P.run_cluster(cs, tr, engines=[mk("fcfs")] * 60 + [mk("larry")] * 61)


def test_heterogeneous_engines_each_check_feasibility():
    """Every prebuilt engine checks every request (cluster.py:86-92), in engine order, before any
    device work: the second engine's small pool raises the reference's message for it."""
    tr = [P.TraceEntry(0.0, 100, 10), P.TraceEntry(0.5, 700, 20)]
    cs = P.ClusterSettings(2, P.EngineSettings())
    cost = P.default_params("llama3-8b", "a100")
    big = P.Engine(P.KvBlockPool(2000, 16), P.make_policy("fcfs"), cost)
    small = P.Engine(P.KvBlockPool(20, 16), P.make_policy("fcfs"), cost)
    with pytest.raises(P.InfeasibleRequestError, match="request 1: needs 45 blocks at peak, pool holds 20"):
        P.run_cluster(cs, tr, engines=[big, small])


def test_synthesize_is_bit_identical_to_reference():
    golden = load_golden("configs")
    for sc in S.config_scenarios():
        t = scenario_trace(sc)
        arr = t.arrival / sc["qps_factor"]
        assert trace_sha(arr, t.prompt, t.output) == golden[sc["name"]]["trace_sha"], sc["name"]


def test_pcg64_model_matches_numpy():
    for seed in (0, 3, 9, 123456789):
        words = P.balancers.pcg64_words(seed)
        highs = np.array([2, 3, 8, 64, 1, 7, 2, 1, 5] * 50, dtype=np.int64)
        got = O.rng_integers(words, highs)
        rng = np.random.default_rng(seed)
        want = np.array([int(rng.integers(int(h))) for h in highs])
        assert np.array_equal(got, want), seed


def test_settings_resolution():
    re_ = I.resolve_engine(P.EngineSettings(profile="llama3-70b", hardware="h100x2", gpu_mem_bytes=160e9))
    assert re_.pool_blocks == 17166
    assert I.resolve_engine(P.EngineSettings()).pool_blocks == 11444  # test_kvmem.py:45
    assert P.pool_blocks_for(40e9, P.PROFILES["llama3-8b"]) == 11444
    assert P.blocks_needed(2000, 16) == 125
    with pytest.raises(ValueError):
        P.make_policy("sjf")
    with pytest.raises(ValueError):
        P.make_policy("trail_plus", c=1.5)
    with pytest.raises(ValueError):
        I.instance_record(P.ClusterSettings(balancer=P.BalancerSettings(poll_interval_s=0.0)), 1)


def test_feasibility_errors_match_reference_messages():
    golden_msgs = {
        (2000, 7000): "request 0: prompt 2000 + output 7000 exceeds the 8192-token context window",
    }
    for (p, o), msg in golden_msgs.items():
        with pytest.raises(P.InfeasibleRequestError, match=re.escape(msg)):
            I.check_trace(P.Trace([0.0], [p], [o]), I.resolve_engine(P.EngineSettings()))
    with pytest.raises(P.InfeasibleRequestError, match="needs 7 blocks at peak, pool holds 4"):
        I.check_trace(P.Trace([0.0], [100], [10]), I.resolve_engine(P.EngineSettings(pool_blocks=4)))
    np_ = I.resolve_engine(P.EngineSettings(policy="nopreempt", max_output=20))
    with pytest.raises(P.InfeasibleRequestError, match="exceeds the promised max_output 20"):
        I.check_trace(P.Trace([0.0, 1.0], [10, 10], [5, 30]), np_)
    with pytest.raises(ValueError, match="sorted"):
        I.check_trace(P.Trace([1.0, 0.5], [10, 10], [1, 1]), I.resolve_engine(P.EngineSettings()))


def test_feasibility_from_trace_maxima_is_exact():
    """make_batch decides a (trace, engine) pair from the trace's maxima when they pass; that
    shortcut says feasible exactly when the per-request masks find nothing (monotone checks)."""
    rng = np.random.default_rng(9)
    for _ in range(400):
        n = int(rng.integers(1, 40))
        prompt = rng.integers(1, 3000, n).astype(np.int32)
        output = rng.integers(1, 3000, n).astype(np.int32)
        pol = P.make_policy(str(rng.choice(["fcfs", "nopreempt", "trail_plus", "larry"])),
                            max_output=int(rng.integers(1, 4000)))
        lim = P.EngineLimits(1024, None, int(rng.integers(500, 8192)))
        bsz, pool = int(rng.choice([1, 3, 16])), int(rng.integers(10, 800))
        maxes = (int((prompt.astype(np.int64) + output).max()), int(prompt.max()), int(output.max()))
        bad = np.zeros(n, bool)
        for m in pol._infeasible_mask(prompt, output, bsz, pool, lim):
            bad |= m
        assert pol.feasible_by_max(maxes, bsz, pool, lim) == (not bad.any())


def test_make_batch_pair_path_equals_serial_path():
    """make_batch's per-(settings, trace) pair path builds the same instances, trace and labels
    as the job-by-job loop, and a bad factor still raises the reference's error."""
    from paper_2410_17840_b200 import configs as Cf

    jobs = Cf.c4_jobs(seeds=range(2), duration_s=60.0)
    a, b = I.make_batch(jobs), I._make_batch_serial(jobs)
    assert a.instances.tobytes() == b.instances.tobytes() and a.labels == b.labels and a.n_records == b.n_records
    for f in ("arrival", "prompt", "output"):
        assert np.array_equal(getattr(a.trace, f), getattr(b.trace, f))
    bad = list(jobs)
    bad[100] = (bad[100][0], bad[100][1], 0.0)
    with pytest.raises(ValueError, match="factor must be > 0"):
        I.make_batch(bad)


def test_custom_python_policies_are_rejected():
    class MyPolicy(P.FcfsPolicy):
        pass

    with pytest.raises(NotImplementedError):
        P.policies.policy_descriptor(MyPolicy())
    with pytest.raises(NotImplementedError):
        P.FcfsPolicy().select([], [], None, 0.0, None)


def test_reference_pure_function_kats():
    # larry_score (test_policies.py:51-55)
    class R:
        enqueue_time = 0.0
        pending_prefill = 512

    assert P.larry_score(R, 10.0, 4, 1.0) == -2038.0
    assert P.larry_score(R, 10.0, 4, 1000.0) == 7952.0
    # sal_load / beta (test_balancers.py:85-96, 157-165)
    beta = 1365 / 211
    assert P.sal_load(P.ServerStats(1536, 0, 3), 1024, beta, 1024) == beta * 1024
    assert P.sal_load(P.ServerStats(128, 10**6, 1), 128, 2.0, 1024) == 256 / 1024
    est = P.BetaEstimator()
    for _ in range(40):
        est.update(1154, 211)
    assert est.beta == 1365 / 211
    # nearest-rank percentile (test_metrics.py:17-31)
    v = list(range(1, 101))
    assert [P.percentile(v, p) for p in (50, 95, 99, 100, 1, 0.5)] == [50, 95, 99, 100, 1, 1]
    assert P.percentile([3, 1, 2], 67) == 3
    assert P.metrics.nearest_ranks(10_000_000) == (5_000_000, 9_500_000, 9_900_000)


def test_kv_block_pool_descriptor_validates():
    """kvmem.py:82-90 constructor checks; the accounting itself is on the device."""
    pool = P.KvBlockPool(64, 8)
    assert (pool.total_blocks, pool.block_size, pool.free_blocks) == (64, 8, 64)
    with pytest.raises(ValueError):
        P.KvBlockPool(-1, 8)
    with pytest.raises(ValueError):
        P.KvBlockPool(4, 0)


def test_default_params_overrides():
    """costmodel.py:78-94: known pairs take per-field overrides; unknown pairs need all four."""
    base = P.default_params("llama3-8b", "a100")
    assert base == P.CostParams(1.03e-2, 8.4e-8, 1.0e-4, 5e-4)
    assert P.default_params("llama3-8b", "a100", overhead_s=0.0).overhead_s == 0.0
    with pytest.raises(KeyError):
        P.default_params("llama3-8b", "h100x2", overhead_s=0.0)
    full = dict(mem_base_s=1.0, mem_per_kv_token_s=0.0, compute_per_token_s=0.0, overhead_s=0.0)
    assert P.default_params("x", "y", **full) == P.CostParams(1.0, 0.0, 0.0, 0.0)


def test_writers_are_byte_stable(tmp_path):
    recs = [P.MetricsRecord(i, 0, i * 0.1, i * 0.1 + 0.37, i * 0.1 + 1.0, 100, 10, 0) for i in range(5)]
    P.write_records_csv(tmp_path / "a.csv", recs)
    P.write_records_csv(tmp_path / "b.csv", recs)
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    assert (tmp_path / "a.csv").read_text().splitlines()[2] == "1,0,0.1,0.47,1.1,100,10,0"


def test_simulation_path_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(Exception, match="CUDA"):
        P.run_cluster(P.ClusterSettings(), [P.TraceEntry(0.0, 10, 1)])


def test_vectorised_summary_ranks_equal_python_nearest_rank():
    """summary_groups computes ceil(p/100*n) in numpy float64; it must equal the
    reference's Python-float nearest rank (metrics.py:53) for every n."""
    import math

    import numpy as np

    from paper_2410_17840_b200.metrics import summary_groups

    ns = np.concatenate([np.arange(1, 5000), np.array([10**6, 10**7 + 3, 2**31 - 1, 123456789])])
    g = summary_groups(np.stack([np.zeros_like(ns), ns], 1))
    for j, p in enumerate((50, 95, 99)):
        want = np.array([math.ceil(p / 100 * int(n)) for n in ns])
        assert np.array_equal(g["rank"][:, j], want), p
    assert (g["rank"][:, 3:] == 0).all()


def test_first_run_cost_model_is_a_sane_hint():
    """simulate.estimate_cost (the first-run placement hint, fit on measured iterations): one
    coefficient row per policy over cost_design's columns, positive finite int64 estimates, the
    expensive policy first on average (trail_plus: ~3.5k device cycles per iteration vs
    nopreempt's ~330), deterministic, and a work proxy for clusters."""
    import numpy as np

    from paper_2410_17840_b200 import configs as C
    from paper_2410_17840_b200 import instances as I
    from paper_2410_17840_b200 import simulate

    jobs = C.c4_jobs(seeds=[3])
    b = I.make_batch(jobs)
    assert simulate.ITER_COEF.shape == (4, simulate.cost_design(b).shape[1])
    c = simulate.estimate_cost(b)
    assert c.dtype == np.int64 and (c >= 1).all() and (c < 2**31).all()
    assert np.array_equal(c, simulate.estimate_cost(I.make_batch(jobs)))
    pol = np.array([j[3].split("/")[1] for j in jobs])
    assert c[pol == "trail_plus"].mean() > 3 * c[pol == "nopreempt"].mean()
    assert (simulate.estimate_cost(I.make_batch(C.c2_jobs(60.0))) >= 1).all()
