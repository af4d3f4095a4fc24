"""Time each cluster instance of C2 / C5 (prefix) alone: python tools/probe_cluster.py [c5_duration_s]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
for jobs in (C.c2_jobs(), C.c5_jobs(dur, balancers=("sal", "rr", "p2c", "random"))):
    for j in jobs:
        db = simulate.upload(I.make_batch([j]))
        simulate.launch(db); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); simulate.launch(db); e1.record(); torch.cuda.synchronize()
        st = simulate.download(db)[1][0]
        print(f"{j[3]:16s} {e0.elapsed_time(e1):9.1f} ms  rsteps {int(st['request_steps']):,}  iters {int(st['iterations']):,}"
              f"  requests {int(db.h_inst[0]['n_requests']):,}  [epochs {int(st['_pad']):,} polls {int(st['device_cycles']):,} with SSB_EPOCH_PROBE]", flush=True)
