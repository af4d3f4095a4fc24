"""Deterministic parity scenarios shared by tests/golden/make_golden.py (which
runs the Python reference to produce the fixtures) and the tests (which run
the oracle and the CUDA path on the same inputs).

A scenario is a plain dict:
  name, mode ("engine" = Engine(...).run, engine.py:236; "cluster" = run_cluster, cluster.py:65)
  engine:  policy alpha c max_output pool_blocks block_size cost[4] cap max_running max_context
  cluster: n_servers balancer poll_interval_s beta_prior beta_fixed seed
  trace:   {"rows": [[arrival, prompt, output], ...]} or {"synth": SynthSpec kwargs}
  qps_factor: scale_qps divisor (workload.py:187)
Nothing here imports the reference or the product; traces come from numpy
RNGs with fixed seeds, so both sides regenerate identical inputs.
"""

from __future__ import annotations

import itertools

import numpy as np

COST_A100_8B = [1.03e-2, 8.4e-8, 1.0e-4, 5e-4]  # costmodel.py:63-68
COST_H100_70B = [1.05e-2, 4.9e-8, 1.4e-4, 5e-4]  # costmodel.py:69-74
COST_ENGINE_TESTS = [0.5, 0.001, 0.01, 0.1]  # tests/test_engine.py:12
COST_C6 = [2e-3, 1e-6, 3e-5, 1e-3]  # tests/test_acceptance.py:274

CHAT_PROMPT = {"location": 6.45, "scale": 1.1}  # SURVEY.md §8d "chat-shaped"
CHAT_OUTPUT = {"location": 4.95, "scale": 0.9}


def engine(policy="fcfs", *, alpha=1.0, c=0.0, max_output=1024, pool_blocks=1000, block_size=16, cost=None,
           cap=1024, max_running=None, max_context=8192):
    return {
        "policy": policy, "alpha": float(alpha), "c": float(c), "max_output": int(max_output),
        "pool_blocks": int(pool_blocks), "block_size": int(block_size),
        "cost": list(cost or COST_ENGINE_TESTS), "cap": int(cap), "max_running": max_running,
        "max_context": int(max_context),
    }


def cluster(n_servers=1, balancer="rr", *, poll_interval_s=0.1, beta_prior=2.0, beta_fixed=None, seed=0):
    return {"n_servers": int(n_servers), "balancer": balancer, "poll_interval_s": float(poll_interval_s),
            "beta_prior": float(beta_prior), "beta_fixed": beta_fixed, "seed": int(seed)}


def scen(name, eng, trace, *, mode="engine", clus=None, qps_factor=1.0):
    return {"name": name, "mode": mode, "engine": eng, "cluster": clus or cluster(), "trace": trace,
            "qps_factor": float(qps_factor)}


def rows(lst):
    return {"rows": [[float(a), int(p), int(o)] for a, p, o in lst]}


def synth(**kw):
    return {"synth": kw}


# ---------------------------------------------------------------------------
# engine-level scenarios from the reference's own tests (retargeted through run())
# ---------------------------------------------------------------------------

def engine_unit_scenarios():
    out = []
    E = lambda **kw: engine(**kw)  # noqa: E731
    out.append(scen("short_prompt_two_iterations", E(), rows([(0.0, 100, 2)])))  # test_engine.py:19-26
    out.append(scen("long_prompt_chunks", E(), rows([(0.0, 2000, 1)])))  # :29-37
    out.append(scen("decode_before_prefill", E(pool_blocks=4000),
                    rows([(0.0, 50, 30)] * 10 + [(0.0, 2000, 5)])))  # :40-49 shape
    out.append(scen("output_one", E(), rows([(0.0, 64, 1)])))  # :66-70
    out.append(scen("clock_increases", E(), rows([(i * 0.01, 100 + i, 5) for i in range(20)])))  # :73-92
    out.append(scen("fifo_tie_break", E(), rows([(0.0, 50, 2), (0.0, 50, 2)])))  # :95-99
    out.append(scen("grow_evicts_youngest", E(pool_blocks=11, block_size=8),
                    rows([(0.0, 30, 20), (0.0, 24, 20), (0.0, 22, 20)])))  # :113-131
    out.append(scen("recompute_keeps_first_token", E(pool_blocks=8, block_size=8),
                    rows([(0.0, 32, 20), (0.0, 24, 20)])))  # :134-157
    out.append(scen("eviction_seniority", E(pool_blocks=13, block_size=8),
                    rows([(0.0, 32, 2)] * 3 + [(0.0, 8, 2)])))  # :160-174
    out.append(scen("idle_jump", E(), rows([(0.0, 100, 1), (50.0, 100, 1)])))  # :236-239
    rng = np.random.default_rng(8)  # :242-251
    times = np.sort(rng.uniform(0, 5, 30))
    tr = [(float(t), int(rng.integers(1, 2000)), int(rng.integers(1, 50))) for t in times]
    out.append(scen("deterministic_pool200", E(pool_blocks=200), rows(tr)))
    rng = np.random.default_rng(21)  # :254-272
    for pol in ("fcfs", "nopreempt", "trail_plus", "larry"):
        for k in range(5):
            n = int(rng.integers(3, 25))
            times = np.sort(rng.uniform(0, 3, n))
            tr = [(float(t), int(rng.integers(1, 400)), int(rng.integers(1, 40))) for t in times]
            out.append(scen(f"all_finish_{pol}_{k}", E(policy=pol, pool_blocks=60, max_output=40, c=0.5), rows(tr)))
    out.append(scen("max_running_2", E(max_running=2), rows([(0.0, 30, 4)] * 6)))  # :275-281
    out.append(scen("custom_budget_64", E(cap=64), rows([(0.0, 300, 2)])))  # :284-293
    return out


# criterion 6 (test_acceptance.py:273-341): 5,808 enumerated FCFS instances
C6_PAIRS = [(3, 2), (17, 5), (40, 1)]
C6_VARIANTS = [(6, 1024), (12, 1024), (64, 1024), (12, 16)]


def c6_scenarios():
    out = []
    for length in range(1, 6):
        for combo in itertools.product(range(3), repeat=length):
            sizes = [C6_PAIRS[c] for c in combo]
            k = length
            patterns = [[0.0] * k, [0.25 * j for j in range(k)], [10.0 * j for j in range(k)],
                        [0.25 * (j // 2) for j in range(k)]]
            for pi, arrivals in enumerate(patterns):
                for pool, cap in C6_VARIANTS:
                    tr = [(a, p, o) for a, (p, o) in zip(arrivals, sizes)]
                    out.append(scen(f"c6_{''.join(map(str, combo))}_{pi}_{pool}_{cap}",
                                    engine("fcfs", pool_blocks=pool, block_size=8, cost=COST_C6, cap=cap), rows(tr)))
    return out


def c2_scenarios(n_runs=1000):
    """criterion 2 (test_acceptance.py:102-134): NoPreempt never preempts."""
    rng = np.random.default_rng(7100)
    out = []
    for i in range(n_runs):
        bs = int(rng.choice([8, 16]))
        max_out = int(rng.integers(4, 33))
        n = int(rng.integers(1, 9))
        prompts = rng.integers(1, 121, size=n)
        outputs = rng.integers(1, max_out + 1, size=n)
        arrivals = np.sort(rng.uniform(0.0, 2.0, size=n))
        need = max(-(-(int(p) + max_out) // bs) for p in prompts)
        pool = need + int(rng.integers(0, 11))
        tr = [(float(a), int(p), int(o)) for a, p, o in zip(arrivals, prompts, outputs)]
        out.append(scen(f"c2_{i}", engine("nopreempt", max_output=max_out, pool_blocks=pool, block_size=bs,
                                          cost=COST_C6), rows(tr)))
    return out


def c3_scenarios(n_inst=100):
    """criterion 3 (test_acceptance.py:137-175): LARRY alpha=1e9 == FCFS dispatch order."""
    rng = np.random.default_rng(7300)
    out = []
    for i in range(n_inst):
        n = int(rng.integers(5, 26))
        gaps = 0.1 + rng.uniform(0.0, 0.4, size=n)
        arrivals = np.cumsum(gaps) - gaps[0]
        prompts = rng.integers(1, 301, size=n)
        outputs = rng.integers(1, 41, size=n)
        bs = 8
        pool = sum(-(-(int(p) + int(o)) // bs) for p, o in zip(prompts, outputs)) + 4
        tr = [(float(a), int(p), int(o)) for a, p, o in zip(arrivals, prompts, outputs)]
        out.append(scen(f"c3_fcfs_{i}", engine("fcfs", pool_blocks=pool, block_size=bs, cost=COST_C6), rows(tr)))
        out.append(scen(f"c3_larry_{i}", engine("larry", alpha=1e9, pool_blocks=pool, block_size=bs, cost=COST_C6),
                        rows(tr)))
    return out


def fuzz_engine_scenarios(n=240, seed=90210, block_sizes=(1, 4, 8, 16), prefix="fuzz"):
    """Randomised single-engine instances biased toward the hard paths: tight
    pools (grow evictions, recompute), trail_plus with c>0 (policy preempts),
    larry under backlog, max_running caps, small token budgets, ties."""
    rng = np.random.default_rng(seed)
    out = []
    pols = ["fcfs", "nopreempt", "trail_plus", "larry"]
    for i in range(n):
        pol = pols[i % 4]
        bs = int(rng.choice(list(block_sizes)))
        nreq = int(rng.integers(1, 60))
        burst = rng.random() < 0.4
        if burst:
            arrivals = np.sort(np.round(rng.uniform(0, 0.5, nreq), 1))
        else:
            arrivals = np.sort(rng.exponential(0.05, nreq).cumsum())
        prompts = rng.integers(1, int(rng.choice([16, 64, 300, 1500])) + 1, nreq)
        max_out = int(rng.choice([4, 20, 80]))
        outputs = rng.integers(1, max_out + 1, nreq)
        max_ctx = 8192
        peak_blocks = max(-(-(int(p) + int(o)) // bs) for p, o in zip(prompts, outputs))
        if pol == "nopreempt":
            peak_blocks = max(peak_blocks, max(-(-min(max_ctx, int(p) + max_out) // bs) for p in prompts))
        pool = peak_blocks + int(rng.integers(0, int(rng.choice([2, 10, 60, 400]))))
        cap = int(rng.choice([8, 64, 256, 1024]))
        max_running = None if rng.random() < 0.7 else int(rng.integers(1, 6))
        c = float(rng.choice([0.0, 0.25, 0.5, 1.0])) if pol == "trail_plus" else 0.0
        alpha = float(rng.choice([0.0, 0.01, 1.0, 1000.0])) if pol == "larry" else 1.0
        cost = [float(rng.choice([1e-3, 1e-2])), float(rng.choice([0.0, 1e-6, 8.4e-8])),
                float(rng.choice([1e-5, 1e-4])), float(rng.choice([0.0, 5e-4]))]
        tr = [(float(a), int(p), int(o)) for a, p, o in zip(arrivals, prompts, outputs)]
        out.append(scen(f"{prefix}_{pol}_{i}", engine(pol, alpha=alpha, c=c, max_output=max_out, pool_blocks=pool,
                                                  block_size=bs, cost=cost, cap=cap, max_running=max_running),
                        rows(tr)))
    return out


BURSTY_TRACE = [(0.0, 100, 5), (0.0, 300, 2), (0.1, 50, 8), (0.2, 700, 3), (0.3, 20, 1), (50.0, 400, 6),
                (50.05, 60, 4), (51.0, 1500, 2)]  # tests/test_cluster.py:27-36


def _es(policy="fcfs", **kw):
    """EngineSettings defaults (config.py:26-39): llama3-8b on a100, 40e9 B -> 11,444 blocks."""
    return engine(policy, pool_blocks=kw.pop("pool_blocks", 11444), cost=kw.pop("cost", COST_A100_8B), **kw)


def cluster_unit_scenarios():
    out = []
    C = lambda n, b, **kw: cluster(n, b, **kw)  # noqa: E731
    out.append(scen("cl_single_bursty", _es(), rows(BURSTY_TRACE), mode="cluster", clus=C(1, "rr")))
    out.append(scen("cl_single_synth", _es(), synth(duration_s=30.0, mean_qps=2.0, burstiness=1.5, seed=42),
                    mode="cluster", clus=C(1, "rr")))
    tr = [(0.01 * i, 40 + 7 * (i % 5), 30 + (i % 11)) for i in range(40)]
    out.append(scen("cl_single_preempt", _es("trail_plus", c=0.9, pool_blocks=64), rows(tr), mode="cluster",
                    clus=C(1, "rr")))
    for b in ("rr", "random", "p2c", "sal"):
        out.append(scen(f"cl_finish_once_{b}", _es(), synth(duration_s=20.0, mean_qps=3.0, seed=5), mode="cluster",
                        clus=C(3, b, seed=9)))
    out.append(scen("cl_rr_order", _es(), rows([(float(i), 100, 2) for i in range(6)]), mode="cluster",
                    clus=C(3, "rr")))
    out.append(scen("cl_sal_burst", _es(), rows([(0.0, 512, 4)] * 4), mode="cluster",
                    clus=C(4, "sal", beta_fixed=2.0)))
    out.append(scen("cl_poll_inbox", _es(cost=[1e-4, 1e-7, 1e-3, 0.01]),
                    rows([(0.0, 1024, 50), (0.0, 1024, 50), (0.3, 512, 5), (0.4, 512, 5)]), mode="cluster",
                    clus=C(2, "sal", beta_fixed=2.0, poll_interval_s=0.05)))
    out.append(scen("cl_inf_poll", _es(), synth(duration_s=10.0, mean_qps=2.0, seed=3), mode="cluster",
                    clus=C(2, "sal", poll_interval_s=float("inf"))))
    out.append(scen("cl_random_det", _es(), synth(duration_s=15.0, mean_qps=3.0, seed=1), mode="cluster",
                    clus=C(3, "random", seed=4)))
    # criterion 5 operating point (test_acceptance.py:221-270), first seeds
    for seed in (2000, 2001, 2002):
        for b in ("sal", "random"):
            out.append(scen(f"cl_c5_{b}_{seed}", _es("larry"),
                            synth(duration_s=45.0, mean_qps=18.0, burstiness=2.5,
                                  prompt_dist={"location": 7.6, "scale": 0.3},
                                  output_dist={"location": 3.3, "scale": 0.35}, max_context=8192, seed=seed),
                            mode="cluster", clus=C(4, b, poll_interval_s=1.0, seed=seed)))
    # criterion 10 config (test_acceptance.py:399-411)
    out.append(scen("cl_c10_p2c", _es("larry"), synth(duration_s=6.0, mean_qps=3.0, seed=1), mode="cluster",
                    clus=C(2, "p2c", seed=3)))
    return out


def fuzz_cluster_scenarios(n=96, seed=31337, block_sizes=(4, 16), prefix="fuzzcl", caps=(32, 256, 1024),
                           betas=(1.0, 2.0, 6.5), bals=("rr", "random", "p2c", "sal"), servers=None,
                           pols=("fcfs", "nopreempt", "trail_plus", "larry"), nreq_range=(5, 150)):
    """Randomised multi-replica instances: every balancer x policy, tight pools,
    poll intervals from 1 ms to inf, fixed and estimated beta, equal-time bursts.
    servers: replica counts to cycle through (default: uniform in 2..8)."""
    rng = np.random.default_rng(seed)
    out = []
    bals = list(bals)
    pols = list(pols)
    for i in range(n):
        b = bals[i % len(bals)]
        pol = pols[(i // len(bals)) % len(pols)]
        ns = int(rng.integers(2, 9)) if servers is None else int(servers[(i // (len(bals) * len(pols))) % len(servers)])
        nreq = int(rng.integers(*nreq_range))
        if rng.random() < 0.3:
            arrivals = np.sort(np.round(rng.uniform(0, 1.0, nreq), 1))
        else:
            arrivals = np.sort(rng.exponential(float(rng.choice([0.002, 0.02, 0.2])), nreq).cumsum())
        bs = int(rng.choice(list(block_sizes)))
        prompts = rng.integers(1, int(rng.choice([64, 600, 3000])) + 1, nreq)
        max_out = int(rng.choice([8, 60, 300]))
        outputs = rng.integers(1, max_out + 1, nreq)
        peak = max(-(-(int(p) + int(o)) // bs) for p, o in zip(prompts, outputs))
        if pol == "nopreempt":
            peak = max(peak, max(-(-min(8192, int(p) + max_out) // bs) for p in prompts))
        pool = peak + int(rng.integers(0, int(rng.choice([4, 40, 400, 4000]))))
        cap = int(rng.choice(list(caps)))
        poll = float(rng.choice([0.001, 0.05, 0.1, 1.0, float("inf")]))
        beta_fixed = None if rng.random() < 0.6 else float(rng.choice(list(betas)))
        c = float(rng.choice([0.0, 0.5, 1.0])) if pol == "trail_plus" else 0.0
        tr = [(float(a), int(p), int(o)) for a, p, o in zip(arrivals, prompts, outputs)]
        out.append(scen(f"{prefix}_{b}_{pol}_{i}",
                        engine(pol, c=c, max_output=max_out, pool_blocks=pool, block_size=bs, cost=COST_A100_8B,
                               cap=cap),
                        rows(tr), mode="cluster",
                        clus=cluster(ns, b, poll_interval_s=poll, beta_fixed=beta_fixed,
                                     beta_prior=float(rng.choice([1.0, 2.0, 4.0])), seed=int(rng.integers(0, 1000)))))
    return out


# ---------------------------------------------------------------------------
# BASELINE.json configs, full size where the Python reference
# finishes in seconds, otherwise a fixed prefix
# ---------------------------------------------------------------------------

def config_scenarios(full=True):
    out = []
    # C1: 1 replica, Llama-3-70B on 2xH100 (160e9 B) -> 17,166 blocks; 10,058 requests
    c1 = synth(duration_s=2000.0, mean_qps=5.0, burstiness=1.0, seed=0)
    for pol in ("fcfs", "larry"):
        out.append(scen(f"C1_{pol}", engine(pol, alpha=1.0, pool_blocks=17166, cost=COST_H100_70B, max_output=8191),
                        c1, mode="cluster", clus=cluster(1, "random")))
    # C2: 8 replicas, larry, chat-shaped 28 qps b=2 (300-s prefix of the 3,571-s trace)
    c2 = synth(duration_s=300.0 if full else 60.0, mean_qps=28.0, burstiness=2.0, prompt_dist=CHAT_PROMPT,
               output_dist=CHAT_OUTPUT, seed=0)
    for b in ("rr", "random", "p2c", "sal"):
        out.append(scen(f"C2_{b}", engine("larry", pool_blocks=11444, cost=COST_A100_8B, max_output=8191), c2,
                        mode="cluster", clus=cluster(8, b)))
    # C3: 1 replica, pool 1,536, long-tail outputs (1,500-s prefix)
    c3 = synth(duration_s=1500.0 if full else 300.0, mean_qps=1.2, burstiness=1.0,
               output_dist={"location": 5.5, "scale": 1.3}, seed=0)
    out.append(scen("C3_fcfs", engine("fcfs", pool_blocks=1536, cost=COST_A100_8B, max_output=8191), c3,
                    mode="cluster", clus=cluster(1, "random")))
    out.append(scen("C3_trail_plus", engine("trail_plus", c=0.5, pool_blocks=1536, cost=COST_A100_8B,
                                            max_output=8191), c3, mode="cluster", clus=cluster(1, "random")))
    # C4 corners: seed-0 base trace (3 qps b=2, 600 s) scaled by the sweep factors
    c4 = synth(duration_s=600.0, mean_qps=3.0, burstiness=2.0, prompt_dist=CHAT_PROMPT, output_dist=CHAT_OUTPUT,
               seed=0)
    corners = [("fcfs", 1024, 4.0), ("larry", 1024, 4.0), ("trail_plus", 2048, 1.5), ("larry", 11444, 0.25),
               ("nopreempt", 4096, 1.0)]
    if full:
        corners.append(("nopreempt", 1024, 4.0))
    for pol, pool, f in corners:
        out.append(scen(f"C4_{pol}_{pool}_x{f}", engine(pol, alpha=1.0, c=0.5, pool_blocks=pool,
                                                        cost=COST_A100_8B, max_output=8191), c4,
                        mode="cluster", clus=cluster(1, "random"), qps_factor=f))
    # C5: 64 replicas, larry, chat-shaped 224 qps b=3 (60-s prefix)
    c5 = synth(duration_s=60.0 if full else 10.0, mean_qps=224.0, burstiness=3.0, prompt_dist=CHAT_PROMPT,
               output_dist=CHAT_OUTPUT, seed=0)
    for b in ("sal", "rr"):
        out.append(scen(f"C5_{b}", engine("larry", pool_blocks=11444, cost=COST_A100_8B, max_output=8191), c5,
                        mode="cluster", clus=cluster(64, b)))
    return out


def prebuilt_scenarios():
    """run_cluster(settings, trace, engines=[...]) with prebuilt engines whose batching cap
    differs from settings.engine.max_tokens_per_batch: SAL's queue term divides by the
    settings' cap (cluster.py:96-104), each engine batches with its own (engine.py:300-323)."""
    out = []
    for i, (eng_cap, route_cap) in enumerate([(256, 1024), (1024, 256), (512, 100), (96, 4096)]):
        for beta_fixed in (None, 2.0):
            for ns in (3, 12):
                out.append(scen(f"prebuilt_{eng_cap}_{route_cap}_{beta_fixed}_{ns}",
                                engine("larry" if i % 2 else "fcfs", pool_blocks=900, cost=COST_A100_8B, cap=eng_cap),
                                synth(duration_s=20.0, mean_qps=25.0, burstiness=2.0, prompt_dist=CHAT_PROMPT,
                                      output_dist=CHAT_OUTPUT, seed=40 + i),
                                mode="cluster",
                                clus=dict(cluster(ns, "sal", poll_interval_s=0.05, beta_fixed=beta_fixed, seed=i),
                                          route_cap=route_cap)))
    return out


def hetero_scenarios(n=48, seed=777):
    """run_cluster(settings, trace, engines=[...]) with prebuilt engines that DIFFER
    (cluster.py:66-79): per server its own pool size, batching cap, running limit, context
    window, cost parameters, policy parameters (alpha / c / max_output), and in a third of the
    clusters each the block size and the policy itself. Every engine checks every request (cluster.py:86-88);
    SAL divides by the settings' cap (cluster.py:96-104); the view's free memory and each
    engine's batching, allocation, eviction and latency are its own. Sizes 2..8 (one CTA)
    and 9..40 (multi-CTA clusters). Scenario key "engines": one engine dict per server."""
    rng = np.random.default_rng(seed)
    out = []
    bals = ["rr", "random", "p2c", "sal"]
    pols = ["fcfs", "nopreempt", "trail_plus", "larry"]
    costs = [COST_A100_8B, COST_H100_70B, [2.0e-2, 1.2e-7, 2.0e-4, 1e-3]]
    for i in range(n):
        b = bals[i % 4]
        pol = pols[(i // 4) % 4]
        ns = int(rng.integers(2, 9)) if i < n // 2 else int(rng.choice([9, 16, 24, 40]))
        nreq = int(rng.integers(40, 400 if ns <= 8 else 900))
        arrivals = np.sort(rng.exponential(float(rng.choice([0.002, 0.02, 0.1])), nreq).cumsum())
        mixed = i % 3 == 0  # a third of the clusters mix block sizes
        bs0 = int(rng.choice([4, 16]))
        prompts = rng.integers(1, int(rng.choice([64, 600, 2000])) + 1, nreq)
        max_out = int(rng.choice([8, 60, 300]))
        outputs = rng.integers(1, max_out + 1, nreq)
        ctx = 8192
        engs = []
        mixed_pol = i % 3 == 1  # a third of the clusters mix policies
        for s in range(ns):
            bs = int(rng.choice([4, 10, 16, 32])) if mixed else bs0
            pol_s = str(rng.choice(pols)) if mixed_pol else pol
            peak = max(-(-(int(p) + int(o)) // bs) for p, o in zip(prompts, outputs))
            mo = max_out + int(rng.integers(0, 64)) if pol_s == "nopreempt" else max_out
            need = peak
            if pol_s == "nopreempt":
                need = max(need, max(-(-min(ctx, int(p) + mo) // bs) for p in prompts))
            pool = need + int(rng.integers(0, int(rng.choice([4, 40, 400, 4000]))))
            mr = None if rng.random() < 0.7 else int(rng.integers(2, 64))
            engs.append(engine(pol_s, alpha=float(rng.choice([0.5, 1.0, 2.0])),
                               c=float(rng.choice([0.0, 0.25, 0.5, 1.0])) if pol_s == "trail_plus" else 0.0,
                               max_output=mo, pool_blocks=pool, block_size=bs,
                               cost=costs[int(rng.integers(0, len(costs)))],
                               cap=int(rng.choice([32, 100, 256, 1024, 4096])), max_running=mr, max_context=ctx))
        tr = [(float(a), int(p), int(o)) for a, p, o in zip(arrivals, prompts, outputs)]
        sc = scen(f"hetero_{b}_{pol}_{ns}_{i}", engs[0], rows(tr), mode="cluster",
                  clus=dict(cluster(ns, b, poll_interval_s=float(rng.choice([0.001, 0.05, 0.5, float("inf")])),
                                    beta_fixed=None if rng.random() < 0.6 else float(rng.choice([1.0, 2.0, 6.5])),
                                    seed=int(rng.integers(0, 1000))),
                            route_cap=int(rng.choice([100, 512, 1024]))))
        sc["engines"] = engs
        out.append(sc)
    return out


GROUPS = {
    "engine_unit": engine_unit_scenarios,
    "c6": c6_scenarios,
    "c2": c2_scenarios,
    "c3": c3_scenarios,
    "fuzz_engine": fuzz_engine_scenarios,
    "cluster_unit": cluster_unit_scenarios,
    "fuzz_cluster": fuzz_cluster_scenarios,
    "configs": config_scenarios,
    # block sizes that are not powers of two (the device's blocks() is a multiply-shift
    # division there and the steady-state decode paths are off)
    "fuzz_odd_blocks": lambda: fuzz_engine_scenarios(80, seed=4242, block_sizes=(3, 5, 10, 12, 24), prefix="odd")
    + fuzz_cluster_scenarios(24, seed=4243, block_sizes=(3, 10, 24), prefix="oddcl"),
    # sal / p2c routing off the integer-key fast path: token caps that are not powers of two
    # (the queue term is a true division) beside power-of-two ones, fixed and estimated beta
    # multi-CTA thread-block clusters: 9..64 replicas (2..8 CTAs, one warp per replica) x every
    # policy x every balancer, and 65..96 replicas (several replicas per warp, global tables)
    "fuzz_multicta": lambda: fuzz_cluster_scenarios(80, seed=6464, prefix="mcta", servers=(9, 16, 24, 33, 64),
                                                    nreq_range=(60, 700))
    + fuzz_cluster_scenarios(32, seed=6565, prefix="mcta_big", servers=(65, 96), nreq_range=(100, 900)),
    "prebuilt": prebuilt_scenarios,
    "hetero": hetero_scenarios,
    "fuzz_route": lambda: fuzz_cluster_scenarios(48, seed=5151, block_sizes=(4, 16), prefix="route",
                                                 caps=(48, 100, 1000, 1024), betas=(1.0, 1.25, 9.0),
                                                 bals=("sal", "sal", "p2c")),
}
