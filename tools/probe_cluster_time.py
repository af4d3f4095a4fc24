"""Kernel time of single cluster instances (pipelined kernel), one at a time, for A/B of
library variants (SSB_LIB=tools/variants/libssb_X.so): C2/sal, C2/p2c, C5/sal on a prefix.
usage: python tools/probe_cluster_time.py [c5_prefix_s]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_17840_b200 import configs as C, instances as I, simulate  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
c2 = C.c2_jobs()
jobs = [j for j in c2 if j[0].balancer.name in ("sal", "p2c")] + C.c5_jobs(dur, balancers=("sal",))
out = []
for job in jobs:
    db = simulate.upload(I.make_batch([job]))
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = simulate.download(db)[1][0]
    out.append(f"{job[3] if len(job) > 3 else job[0].balancer.name}: min {min(ts):7.1f} ms  digest {int(st['digest']):016x}")
print(" | ".join(out))
