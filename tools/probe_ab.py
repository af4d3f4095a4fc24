"""A/B timing loop for kernel changes: single worst-case instances alone (device
cycles), each policy's C4 sub-sweep, and the full C4 sweep (min of 3 launches).
usage: python tools/probe_ab.py [full|quick]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate


def timed(jobs, reps=3):
    db = simulate.upload(I.make_batch(jobs))
    simulate.launch(db)
    torch.cuda.synchronize()
    st = simulate.download(db)[1]
    c = simulate.measured_cost(db.h_inst, st)
    if c is not None:
        db.h_inst["est_cost"] = c
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    st = simulate.download(db)[1]
    bad = st["status"] != 0
    if bad.any():
        print(f"  !! {int(bad.sum())} instances with status {np.unique(st['status'][bad])} (capacity overflows re-run on "
              "the host path; timing below excludes their re-run)")
    return min(ts), st


singles = ["C4/trail_plus/1024/x2.0/s7", "C4/trail_plus/2048/x2.75/s0", "C4/larry/1024/x4.0/s0",
           "C4/nopreempt/1024/x4.0/s0", "C4/fcfs/1024/x2.0/s7"]
for lab in singles:
    seed = int(lab.rsplit("/s", 1)[1])
    jobs = [j for j in C.c4_jobs(seeds=[seed]) if j[3] == lab]
    ms, st = timed(jobs)
    it = int(st["iterations"][0])
    print(f"{lab:32s} {ms:7.2f} ms  {int(st['device_cycles'][0]) / it:7.0f} cyc/iter  digest {int(st['digest'][0]):016x}",
          flush=True)
if (sys.argv[1:] or ["full"])[0] == "full":
    jobs = C.c4_jobs()
    for pol in ("trail_plus", "larry"):
        ms, st = timed([j for j in jobs if j[3].split("/")[1] == pol])
        print(f"C4 {pol:10s} sub-sweep: {ms:7.1f} ms", flush=True)
    ms, st = timed(jobs)
    print(f"C4 full sweep: {ms:7.1f} ms  {int(st['request_steps'].sum()) / ms * 1e3:.3e} rsteps/s", flush=True)
