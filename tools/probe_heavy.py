"""C4 sweep kernel time vs SSB_HEAVY_SMS (SMs reserved, one CTA each, for the longest
trail_plus instances): python tools/probe_heavy.py 0 16 25 32"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

db = simulate.upload(I.make_batch(C.c4_jobs()))
simulate.launch(db)
torch.cuda.synchronize()
if not os.environ.get("COLD"):  # COLD=1: keep the host estimates (first-run schedule)
    db.h_inst["est_cost"] = simulate.measured_cost(db.h_inst, simulate.download(db)[1])
res = {}
for rep in range(3):
    for h in sys.argv[1:]:
        os.environ["SSB_HEAVY_SMS"] = h
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(h, []).append(e0.elapsed_time(e1))
for h, v in res.items():
    print(f"SSB_HEAVY_SMS={h:>3}: " + " ".join(f"{x:6.1f}" for x in v) + f"  min {min(v):6.1f} ms")
