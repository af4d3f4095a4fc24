"""Time each instance of a C4 policy group alone; print the slowest."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate

pol = sys.argv[1] if len(sys.argv) > 1 else "trail_plus"
seeds = range(int(sys.argv[2])) if len(sys.argv) > 2 else range(2)
jobs = [j for j in C.c4_jobs(seeds=seeds) if j[3].split("/")[1] == pol]
res = []
for j in jobs:
    db = simulate.upload(I.make_batch([j]))
    simulate.launch(db); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); simulate.launch(db); e1.record(); torch.cuda.synchronize()
    st = simulate.download(db)[1][0]
    res.append((e0.elapsed_time(e1), j[3], int(st["iterations"]), int(st["request_steps"]), int(st["preempts"])))
res.sort(reverse=True)
tot = sum(r[0] for r in res)
print(f"{pol}: {len(res)} instances, sum {tot:.0f} ms, max {res[0][0]:.1f} ms")
for t, lab, it, rs, pre in res[:12]:
    print(f"  {t:8.1f} ms  {lab:32s} iters {it:8,d} rsteps {rs:10,d} preempts {pre:6d}  {1e6*t/it:7.0f} ns/iter")
