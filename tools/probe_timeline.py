"""Per-instance timeline of the C4 sweep from %globaltimer (debug build with -DSSB_TIMELINE:
tools/build_variant.sh timeline -DSSB_TIMELINE; run with SSB_LIB=tools/variants/libssb_timeline.so).
Reports, for the host-estimate (cold) and the measured (warm) schedules: the makespan, the longest
instances (duration, start, end, SM), when SMs go idle, and the busy-warp profile over time.
usage: SSB_LIB=... python tools/probe_timeline.py [OUT.npz]"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

from paper_2410_17840_b200 import _abi
from paper_2410_17840_b200 import configs as C
from paper_2410_17840_b200 import instances as I
from paper_2410_17840_b200 import simulate

lib = _abi.load_library()
lib.ssb_debug_timeline.restype = ctypes.c_int32
lib.ssb_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
jobs = C.c4_jobs()
labels = np.array([j[3] for j in jobs])
db = simulate.upload(I.make_batch(jobs))
n = len(jobs)
out = {}
for tag in ("cold", "warm"):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    tl = np.zeros(3 * n, dtype=np.uint64)
    assert lib.ssb_debug_timeline(tl.ctypes.data, n) == n
    tl = tl.reshape(n, 3).astype(np.int64)
    st = simulate.download(db)[1]
    t0 = tl[:, 0].min()
    start, end = (tl[:, 0] - t0) / 1e6, (tl[:, 1] - t0) / 1e6
    dur = end - start
    print(f"== {tag}: kernel {ms:.1f} ms (events), timeline span {end.max():.1f} ms, work-sum {dur.sum():.0f} warp-ms")
    o = np.argsort(-dur)[:12]
    for i in o:
        print(f"  {labels[i]:32s} dur {dur[i]:6.1f}  start {start[i]:6.1f}  end {end[i]:6.1f}  sm {tl[i, 2]:3d}  "
              f"iters {int(st['iterations'][i])}")
    o = np.argsort(-end)[:6]
    print("  last to finish:", ", ".join(f"{labels[i]} ({start[i]:.1f}->{end[i]:.1f})" for i in o))
    sm_end = np.zeros(int(tl[:, 2].max()) + 1)
    np.maximum.at(sm_end, tl[:, 2], end)
    print("  SM last-finish percentiles (ms) p10/p50/p90/max:", np.round(np.percentile(sm_end, [10, 50, 90, 100]), 1))
    grid = np.arange(0, end.max() + 1, 5.0)
    busy = [(np.sum((start <= t) & (end > t))) for t in grid]
    print("  busy warps every 5 ms:", busy)
    out[f"{tag}_start"], out[f"{tag}_end"], out[f"{tag}_sm"] = start, end, tl[:, 2]
    c = simulate.measured_cost(db.h_inst, st)
    db.h_inst["est_cost"] = c
if len(sys.argv) > 1:
    np.savez(sys.argv[1], labels=labels, **out)
