"""Per-instance device-cycle distribution of the C4 sweep: does the longest
instance (critical path) or the total work bound the k_engines makespan?
usage: python tools/probe_dist.py [top]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
jobs = C.c4_jobs()
labels = [j[3] for j in jobs]
db = simulate.upload(I.make_batch(jobs))
simulate.launch(db)
torch.cuda.synchronize()
st = simulate.download(db)[1]
db.h_inst["est_cost"] = simulate.measured_cost(db.h_inst, st)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    simulate.launch(db)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
st = simulate.download(db)[1]
cyc = st["device_cycles"].astype(np.float64)
it = st["iterations"].astype(np.float64)
rs = st["request_steps"].astype(np.float64)
clk = 1.965e9
print(f"kernel ms (min of 3): {min(ts):.1f}; sum cycles {cyc.sum():.3e} = {cyc.sum() / clk * 1e3:.0f} warp-ms; "
      f"max instance {cyc.max() / clk * 1e3:.1f} ms")
for warps in (148 * 4, 148 * 8, 148 * 12, 148 * 16):
    print(f"  ideal makespan at {warps} warps (no slowdown): {cyc.sum() / clk * 1e3 / warps:.1f} ms")
print(f"iterations {it.sum():.3e}, rsteps {rs.sum():.3e}, cycles/iter {cyc.sum() / it.sum():.0f}, "
      f"rsteps/iter {rs.sum() / it.sum():.1f}")
pol = np.array([lbl.split("/")[1] for lbl in labels])
pool = np.array([lbl.split("/")[2] for lbl in labels])
for p in np.unique(pol):
    m = pol == p
    print(f"  {p:10s} cycles {cyc[m].sum() / cyc.sum():6.1%}  iters {it[m].sum():.3e}  cyc/iter "
          f"{cyc[m].sum() / it[m].sum():6.0f}  rsteps/iter {rs[m].sum() / it[m].sum():6.1f}  max {cyc[m].max() / clk * 1e3:6.1f} ms")
    for q in np.unique(pool):
        mm = m & (pool == q)
        print(f"      pool {q:6s} cycles {cyc[mm].sum() / cyc.sum():6.1%} cyc/iter {cyc[mm].sum() / it[mm].sum():6.0f} "
              f"rsteps/iter {rs[mm].sum() / it[mm].sum():6.1f} max {cyc[mm].max() / clk * 1e3:6.1f} ms")
order = np.argsort(-cyc)[:top]
for i in order:
    print(f"  {labels[i]:32s} {cyc[i] / clk * 1e3:7.1f} ms  iters {int(it[i]):7d}  rsteps/iter {rs[i] / it[i]:6.1f} "
          f" cyc/iter {cyc[i] / it[i]:6.0f}")
