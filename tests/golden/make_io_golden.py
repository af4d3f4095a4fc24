"""Golden OUTPUT FILES produced by the PYTHON REFERENCE.

Run in the build container (the only place /root/reference exists):
    python tests/golden/make_io_golden.py

Mirrors what `servesim run` / `servesim sweep` write (cli.py:114-159) for two small
experiments, through the reference's own entry points (synthesize, scale_qps,
run_cluster, summarize, write_records_csv, write_summary_csv, write_summary_json;
metrics.py:127-165): records_<policy>_<balancer>.csv per combination plus
summary.csv / summary.json, and sweep.csv / sweep.json. The files are committed
under tests/golden/io/ with io_manifest.json (the experiment definitions);
tests/test_gpu_io.py regenerates them from the CUDA path and compares bytes.
"""

from __future__ import annotations

import json
import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from servesim.cluster import run_cluster  # noqa: E402
from servesim.config import BalancerSettings, ClusterSettings, EngineSettings  # noqa: E402
from servesim.metrics import summarize, write_records_csv, write_summary_csv, write_summary_json  # noqa: E402
from servesim.workload import LengthDist, SynthSpec, scale_qps, synthesize  # noqa: E402

# experiment definitions (plain data: the test rebuilds them with the package's own classes)
MANIFEST = {
    "run": {
        "spec": {"duration_s": 25.0, "mean_qps": 30.0, "burstiness": 2.5, "prompt": [6.45, 1.1],
                 "output": [4.95, 0.9], "seed": 3},
        "n_servers": 4, "seed": 3, "engine": {"pool_blocks": 900},
        "policies": ["fcfs", "larry", "trail_plus"], "balancers": ["rr", "p2c", "sal"],
        "c": 0.5, "poll_interval_s": 0.05,
    },
    "sweep": {
        "spec": {"duration_s": 60.0, "mean_qps": 3.0, "burstiness": 2.0, "prompt": [6.45, 1.1],
                 "output": [4.95, 0.9], "seed": 11},
        "n_servers": 1, "seed": 11, "engine": {"pool_blocks": 1024},
        "policies": ["fcfs", "nopreempt", "larry"], "balancers": ["rr"], "factors": [0.5, 1.0, 2.0, 4.0],
    },
}


def _spec(d):
    return SynthSpec(duration_s=d["duration_s"], mean_qps=d["mean_qps"], burstiness=d["burstiness"],
                     prompt_dist=LengthDist(*d["prompt"]), output_dist=LengthDist(*d["output"]), seed=d["seed"])


def _settings(m, policy, balancer):
    es = EngineSettings(policy=policy, c=m.get("c", 0.0), **m["engine"])
    bs = BalancerSettings(balancer, poll_interval_s=m.get("poll_interval_s", 0.1))
    return ClusterSettings(m["n_servers"], es, bs, m["seed"])


def main():
    out = HERE / "io"
    if out.exists():
        shutil.rmtree(out)
    out.mkdir()
    m = MANIFEST["run"]
    trace = synthesize(_spec(m["spec"]))
    rows = []
    for p in m["policies"]:
        for b in m["balancers"]:
            recs = run_cluster(_settings(m, p, b), trace)
            write_records_csv(out / f"records_{p}_{b}.csv", recs)
            rows.append({"policy": p, "balancer": b, **summarize(recs).to_dict()})
    write_summary_csv(out / "summary.csv", rows)
    write_summary_json(out / "summary.json", rows)
    m = MANIFEST["sweep"]
    trace = synthesize(_spec(m["spec"]))
    rows = []
    for f in m["factors"]:
        scaled = scale_qps(trace, f)
        for p in m["policies"]:
            for b in m["balancers"]:
                rows.append({"factor": f, "policy": p, "balancer": b,
                             **summarize(run_cluster(_settings(m, p, b), scaled)).to_dict()})
    write_summary_csv(out / "sweep.csv", rows)
    write_summary_json(out / "sweep.json", rows)
    (HERE / "io_manifest.json").write_text(json.dumps(MANIFEST, indent=1) + "\n")
    print("wrote", sorted(p.name for p in out.iterdir()))


if __name__ == "__main__":
    main()
