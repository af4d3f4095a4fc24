"""Time each C3 instance alone (latency-mode kernel): python tools/probe_c3.py [duration_s]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_17840_b200 import configs as C, instances as I, simulate  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 83_334.0
for j in C.c3_jobs(dur):
    db = simulate.upload(I.make_batch([j]))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    simulate.launch(db)
    e1.record()
    torch.cuda.synchronize()
    st = simulate.download(db)[1][0]
    ms = e0.elapsed_time(e1)
    print(f"{j[3]:16s} {ms:9.1f} ms  iterations {int(st['iterations']):,}  ns/iter {1e6 * ms / int(st['iterations']):.0f}  "
          f"rsteps {int(st['request_steps']):,}  preempts {int(st['preempts']):,}  dispatches {int(st['dispatches']):,}", flush=True)
