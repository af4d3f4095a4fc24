"""C4 sweep kernel time (cold schedule) for per-policy scales of the cost model's cycles per
iteration (the SM shares between the policy queues): python tools/probe_cpi.py "1,1,1,1" "1,1,1.15,1" ..."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

b = I.make_batch(C.c4_jobs())
res = {}
for rep in range(2):
    for sc in sys.argv[1:]:
        os.environ["SSB_CPI_SCALE"] = sc
        db = simulate.upload(b)
        simulate.launch(db)
        torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            simulate.launch(db)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res.setdefault(sc, []).extend(ts)
        del db
for sc, v in res.items():
    print(f"cpi scale {sc:>22}: " + " ".join(f"{x:6.1f}" for x in v) + f"  min {min(v):6.1f}  mean {sum(v)/len(v):6.1f} ms")
