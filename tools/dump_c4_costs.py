"""Per-instance device cost of the C4 sweep (for fitting simulate.estimate_cost):
iterations, request-steps, preempts, dispatches and device cycles of every instance,
run with the host-estimate schedule and again with the measured schedule.
usage: python tools/dump_c4_costs.py OUT.npz [first_seed]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

s0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
b = I.make_batch(C.c4_jobs(seeds=range(s0, s0 + 16)))
db = simulate.upload(b)
out = {}
for tag in ("cold", "warm"):
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = simulate.download(db)[1]
    print(tag, "ms", ts, flush=True)
    for k in ("iterations", "request_steps", "preempts", "dispatches", "batch_tokens", "device_cycles"):
        out[f"{tag}_{k}"] = st[k]
    out[f"{tag}_est"] = db.h_inst["est_cost"].copy()
    out[f"{tag}_ms"] = np.array(ts)
    c = simulate.measured_cost(db.h_inst, st)
    db.h_inst["est_cost"] = c
out["inst"] = b.instances.view(np.uint8)
out["first_seed"] = np.array(s0)
np.savez(sys.argv[1], **out)
