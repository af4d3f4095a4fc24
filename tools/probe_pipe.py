"""A/B of the cluster kernels on C2 and a C5 prefix, one instance at a time: the classic
epoch kernel (SSB_CLUSTER_CLASSIC=1) vs the pipelined one at several publish periods
(SSB_PIPE_PUBLISH); checks that every variant gives the classic kernel's digest and
counters. usage: python tools/probe_pipe.py [c5_duration_s] [publish periods ...]"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_17840_b200 import configs as C, instances as I, simulate  # noqa: E402

dur = float(sys.argv[1]) if len(sys.argv) > 1 else 600.0
periods = [int(x) for x in sys.argv[2:]] or [8]
KEYS = ("iterations", "request_steps", "batch_tokens", "dispatches", "preempts", "finished", "digest", "status")


def timed(db):
    simulate.launch(db)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    simulate.launch(db)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), simulate.download(db)[1][0]


for jobs in (C.c2_jobs(), C.c5_jobs(dur, balancers=("sal", "rr", "p2c"))):
    for j in jobs:
        db = simulate.upload(I.make_batch([j]))
        os.environ["SSB_CLUSTER_CLASSIC"] = "1"
        t_c, st_c = timed(db)
        del os.environ["SSB_CLUSTER_CLASSIC"]
        line = f"{j[3]:16s} classic {t_c:9.1f} ms"
        for p in periods:
            os.environ["SSB_PIPE_PUBLISH"] = str(p)
            t_p, st_p = timed(db)
            same = all(int(st_p[k]) == int(st_c[k]) for k in KEYS)
            line += f" | pipe/{p} {t_p:9.1f} ms {'ok' if same else 'MISMATCH'}"
        print(line + f"  rsteps {int(st_c['request_steps']):,} requests {int(db.h_inst[0]['n_requests']):,}", flush=True)
