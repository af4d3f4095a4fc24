import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate as S, _abi
from paper_2410_17840_b200.sweep import SweepRunner
from paper_2410_17840_b200.metrics import instance_groups
jobs = C.c4_jobs(seeds=range(16))
r = SweepRunner(jobs); r.run(); r.results()
for k in range(4):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    b = I.make_batch(jobs); t.append(time.perf_counter())
    e = S.estimate_cost(b); t.append(time.perf_counter())
    h = np.ascontiguousarray(b.instances.copy()); h["est_cost"] = e
    _abi.load_library().ssb_prepare(h.ctypes.data, len(h)); t.append(time.perf_counter())
    g = instance_groups(h); t.append(time.perf_counter())
    t0 = time.perf_counter(); r = SweepRunner(jobs); t1 = time.perf_counter(); r.run(); t2 = time.perf_counter(); r.results(); t3 = time.perf_counter()
    print("make_batch %.1f est %.1f prepare %.1f groups %.1f | SweepRunner() %.1f run-enqueue %.1f results(sync) %.1f total %.1f ms" % (
        *(1e3 * np.diff(t)), 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t3 - t0)))
