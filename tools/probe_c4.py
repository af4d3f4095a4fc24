"""C4 breakdown: per policy group and the longest instances alone."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate
from tools.probe_perf import gpu_time

jobs = C.c4_jobs()
full = I.make_batch(jobs)
t, rec, st = gpu_time(full, reps=2)
print(f"all: {t*1e3:.1f} ms, {int(st['request_steps'].sum())/t:.3e} rsteps/s", flush=True)
labels = [j[3] for j in jobs]
for pol in ("fcfs", "nopreempt", "trail_plus", "larry"):
    sub = [j for j in jobs if j[3].split("/")[1] == pol]
    t, rec, s2 = gpu_time(I.make_batch(sub), reps=2)
    print(f"{pol:10s}: {len(sub)} inst {t*1e3:7.1f} ms  rsteps {int(s2['request_steps'].sum()):,} iters {int(s2['iterations'].sum()):,} "
          f"max_iters {int(s2['iterations'].max()):,}", flush=True)
# the 8 instances with most iterations, alone (critical path)
order = np.argsort(-st["iterations"])[:8]
for i in order[:4]:
    t, rec, s3 = gpu_time(I.make_batch([jobs[i]]), reps=2)
    print(f"  single {labels[i]}: iters {int(s3['iterations'][0]):,} {t*1e3:.1f} ms -> {1e9*t/int(s3['iterations'][0]):.0f} ns/iter", flush=True)
