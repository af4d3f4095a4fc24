"""Time the PYTHON REFERENCE itself (servesim.run_cluster, imported read-only from
/root/reference) on a sample of the C4 sweep, one process per host core — the
reference's own CPU path beside the oracle port bench.py times. Only runs where
/root/reference exists (the build container); the result is committed under
profiles/.

usage: python tools/python_reference_rate.py [n_instances] [processes]

Request-steps are counted by wrapping Engine._form_batch (no reference edits), as
tests/golden/make_golden.py does; the same instances are then checked against the
oracle's request-step counts (which the GPU matches bit-exactly)."""
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = "/root/reference/pkg/src"


def _one(args):
    label, spec, pol, kw, pool, factor, seed = args
    sys.path.insert(0, REF)
    from servesim.cluster import run_cluster
    from servesim.config import BalancerSettings, ClusterSettings, EngineSettings
    from servesim.engine import Engine
    from servesim.workload import LengthDist, SynthSpec, scale_qps, synthesize

    orig = Engine._form_batch
    counter = {"rs": 0}

    def counting(self):
        plan = orig(self)
        counter["rs"] += len(plan.decode_ids) + len(plan.prefill_chunks)
        return plan

    Engine._form_batch = counting
    trace = synthesize(SynthSpec(duration_s=spec[0], mean_qps=spec[1], burstiness=spec[2],
                                 prompt_dist=LengthDist(6.45, 1.1), output_dist=LengthDist(4.95, 0.9), seed=seed))
    trace = scale_qps(trace, factor)
    cs = ClusterSettings(1, EngineSettings(policy=pol, pool_blocks=pool, **kw), BalancerSettings("random"), seed)
    t0 = time.perf_counter()
    run_cluster(cs, trace)
    return label, counter["rs"], time.perf_counter() - t0


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    procs = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 1)
    sys.path.insert(0, str(ROOT))
    from paper_2410_17840_b200 import configs as C

    jobs = []
    for pol, kw in C.C4_POLICIES:
        for pool in C.C4_POOLS:
            for f in C.C4_FACTORS:
                jobs.append((f"C4/{pol}/{pool}/x{f}/s0", (600.0, 3.0, 2.0), pol, kw, pool, f, 0))
    # an even sample across policies, pools and rates
    step = max(1, len(jobs) // n)
    sample = jobs[::step][:n]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        res = pool.map(_one, sample, chunksize=1)
    wall = time.perf_counter() - t0
    rs = sum(r[1] for r in res)
    cpu = sum(r[2] for r in res)
    from oracle import oracle as O
    from paper_2410_17840_b200 import instances as I

    O.build()
    labels = [s[0] for s in sample]
    ojobs = [j for j in C.c4_jobs(seeds=[0]) if j[3] in set(labels)]
    _, ost = O.run_batch(I.make_batch(ojobs))
    same = int(ost["request_steps"].sum()) == rs
    out = {"sample": f"{len(sample)} C4 instances of seed 0 (every {step}th of 256)", "processes": procs,
           "request_steps": rs, "wall_s": wall, "rsteps_per_s_all_processes": rs / wall,
           "rsteps_per_s_per_core": rs / cpu, "request_steps_match_oracle": same,
           "host": f"{os.cpu_count()} vCPU (build container)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
