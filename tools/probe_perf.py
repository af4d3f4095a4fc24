"""Ad-hoc timing probe: GPU simulate() per config vs oracle on host cores."""
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np
import torch

from oracle import oracle as O
from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate


def gpu_time(batch, reps=3):
    db = simulate.upload(batch)
    simulate.launch(db)
    torch.cuda.synchronize()
    st0 = simulate.download(db)[1]
    c = simulate.measured_cost(db.h_inst, st0)
    if c is not None:
        db.h_inst["est_cost"] = c
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    rec, stats = simulate.download(db)
    return min(ts), rec, stats


def main():
    which = sys.argv[1:] or ["c1", "c2s", "c3s", "c4", "c5s"]
    threads = os.cpu_count()
    print("host cores", threads, flush=True)
    for w in which:
        if w == "c1":
            jobs = C.c1_jobs()
        elif w == "c2s":
            jobs = C.c2_jobs(300.0)
        elif w == "c3s":
            jobs = C.c3_jobs(20000.0)
        elif w == "c4":
            jobs = C.c4_jobs()
        elif w == "c4q":
            jobs = C.c4_jobs(seeds=range(2))
        elif w == "c5s":
            jobs = C.c5_jobs(60.0)
        batch = I.make_batch(jobs)
        t, rec, stats = gpu_time(batch)
        rs = int(stats["request_steps"].sum())
        bad = int((stats["status"] != 0).sum())
        print(f"{w}: {len(jobs)} inst, N={batch.n_records}, rsteps={rs:,} iters={int(stats['iterations'].sum()):,} "
              f"gpu {t*1e3:.1f} ms -> {rs/t:.3e} rsteps/s, bad={bad}", flush=True)
        t0 = time.perf_counter()
        orec, ostats = O.run_batch(batch, threads=threads)
        t1 = time.perf_counter() - t0
        same = np.array_equal(stats["digest"], ostats["digest"]) and np.array_equal(stats["request_steps"],
                                                                                      ostats["request_steps"])
        print(f"   oracle {threads} thr: {t1:.2f}s -> {rs/t1:.3e} rsteps/s; parity={same}", flush=True)


if __name__ == "__main__":
    main()
