"""The five BASELINE.json operating points as job lists.

A job is (ClusterSettings, Trace, qps_factor, label) — the input of
``instances.make_batch``. Traces are synthesised with ``workload.synthesize``
(bit-identical to the reference's), random-init free: this simulator has no
model weights; "synthetic" refers to the request trace.
"""

from __future__ import annotations

from .settings import BalancerSettings, ClusterSettings, EngineSettings
from .workload import LengthDist, SynthSpec, synthesize

CHAT_PROMPT = LengthDist(6.45, 1.1)  # means ~1154 / 211 tokens (PAPER.md:343 beta 1365/211)
CHAT_OUTPUT = LengthDist(4.95, 0.9)


def c1_jobs(duration_s: float = 2000.0):
    """1 replica, Llama-3-70B on 2xH100 (160e9 B -> 17,166 blocks), fcfs vs larry, N = 10,058."""
    trace = synthesize(SynthSpec(duration_s=duration_s, mean_qps=5.0, burstiness=1.0, seed=0))
    jobs = []
    for pol in ("fcfs", "larry"):
        es = EngineSettings(policy=pol, alpha=1.0, profile="llama3-70b", hardware="h100x2", gpu_mem_bytes=160e9)
        jobs.append((ClusterSettings(1, es, BalancerSettings("random"), 0), trace, 1.0, f"C1/{pol}"))
    return jobs


def c2_jobs(duration_s: float = 3571.0, balancers=("rr", "p2c", "sal", "random")):
    """8 replicas, larry, chat-shaped 28 qps burstiness 2 (~100k requests). "least-load" -> p2c."""
    trace = synthesize(SynthSpec(duration_s=duration_s, mean_qps=28.0, burstiness=2.0, prompt_dist=CHAT_PROMPT,
                                 output_dist=CHAT_OUTPUT, seed=0))
    es = EngineSettings(policy="larry", alpha=1.0)
    return [(ClusterSettings(8, es, BalancerSettings(b), 0), trace, 1.0, f"C2/{b}") for b in balancers]


def c3_jobs(duration_s: float = 833_334.0):
    """1 replica, pool 1,536 blocks, long-tail outputs, recompute-on-resume (~1M requests)."""
    trace = synthesize(SynthSpec(duration_s=duration_s, mean_qps=1.2, burstiness=1.0,
                                 output_dist=LengthDist(5.5, 1.3), seed=0))
    jobs = []
    for pol, c in (("fcfs", 0.0), ("trail_plus", 0.5)):
        es = EngineSettings(policy=pol, c=c, pool_blocks=1536)
        jobs.append((ClusterSettings(1, es, BalancerSettings("random"), 0), trace, 1.0, f"C3/{pol}"))
    return jobs


C4_POLICIES = (("fcfs", {}), ("nopreempt", {}), ("trail_plus", {"c": 0.5}), ("larry", {"alpha": 1.0}))
C4_POOLS = (1024, 2048, 4096, 11444)
C4_FACTORS = tuple(0.25 * i for i in range(1, 17))


def c4_jobs(seeds=range(16), duration_s: float = 600.0):
    """policy x KV pool x arrival-rate (scale_qps) x seed sweep: 4 x 4 x 16 x 16 = 4,096 instances."""
    jobs = []
    for seed in seeds:
        trace = synthesize(SynthSpec(duration_s=duration_s, mean_qps=3.0, burstiness=2.0, prompt_dist=CHAT_PROMPT,
                                     output_dist=CHAT_OUTPUT, seed=int(seed)))
        for pol, kw in C4_POLICIES:
            for pool in C4_POOLS:
                es = EngineSettings(policy=pol, pool_blocks=pool, **kw)
                cs = ClusterSettings(1, es, BalancerSettings("random"), int(seed))
                for f in C4_FACTORS:
                    jobs.append((cs, trace, f, f"C4/{pol}/{pool}/x{f}/s{seed}"))
    return jobs


def c5_jobs(duration_s: float = 44_643.0, balancers=("sal", "rr"), seed: int = 0):
    """64 replicas, larry, chat-shaped 224 qps burstiness 3 (~10M requests)."""
    trace = synthesize(SynthSpec(duration_s=duration_s, mean_qps=224.0, burstiness=3.0, prompt_dist=CHAT_PROMPT,
                                 output_dist=CHAT_OUTPUT, seed=seed))
    es = EngineSettings(policy="larry", alpha=1.0)
    return [(ClusterSettings(64, es, BalancerSettings(b), seed), trace, 1.0, f"C5/{b}/s{seed}") for b in balancers]
