"""Run a golden scenario group through the classic and the pipelined cluster kernels and
print the instances where they differ (settings + differing counters).
usage: python tools/diff_pipe.py GROUP"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import scenarios as S  # noqa: E402
from helpers import scenario_batch  # noqa: E402
from paper_2410_17840_b200 import simulate  # noqa: E402

KEYS = ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "parks", "finished",
        "peak_batch_tokens", "digest", "status")
group = sys.argv[1] if len(sys.argv) > 1 else "fuzz_cluster"
scs = S.GROUPS[group]()
batch = scenario_batch(scs)
os.environ["SSB_CLUSTER_CLASSIC"] = "1"
rc, sc_ = simulate.run_batch(batch)
del os.environ["SSB_CLUSTER_CLASSIC"]
bad = 0
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    rp, sp = simulate.run_batch(batch)
    for i, sc in enumerate(scs):
        d = [k for k in KEYS if int(sc_[i][k]) != int(sp[i][k])]
        if d:
            bad += 1
            if bad <= 12:
                print(rep, sc["name"], {k: (int(sc_[i][k]), int(sp[i][k])) for k in d}, sc["cluster"],
                      {k: sc["engine"][k] for k in ("policy", "pool_blocks", "cap", "block_size")},
                      "nreq", int(batch.instances[i]["n_requests"]), flush=True)
print("mismatching instance-runs:", bad)
