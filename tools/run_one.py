"""Launch one config batch (for ncu): python tools/run_one.py c1 [reps]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate

which = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
jobs = {"c1": lambda: C.c1_jobs()[:1], "c1l": lambda: C.c1_jobs()[1:], "c2s": lambda: C.c2_jobs(300.0)[2:3],
        "c3s": lambda: C.c3_jobs(20000.0)[1:], "c4": lambda: C.c4_jobs(), "c4q": lambda: C.c4_jobs(seeds=range(2)),
        "c5s": lambda: C.c5_jobs(60.0)[:1],
        "c3one": lambda: C.c3_jobs(20000.0)[1:],
        "c4trail": lambda: [j for j in C.c4_jobs() if j[3].split("/")[1] == "trail_plus"],
        "trailworst": lambda: [j for j in C.c4_jobs(seeds=range(1)) if j[3] == "C4/trail_plus/1024/x4.0/s0"],
        "trailbig": lambda: [j for j in C.c4_jobs(seeds=range(1)) if j[3] == "C4/trail_plus/11444/x4.0/s0"],
        "npworst": lambda: [j for j in C.c4_jobs(seeds=range(1)) if j[3] == "C4/nopreempt/1024/x4.0/s0"],
        "sparse": lambda: [j for j in C.c4_jobs(seeds=range(1)) if j[3] == "C4/larry/11444/x0.25/s0"],
        "larryworst": lambda: [j for j in C.c4_jobs(seeds=range(1)) if j[3] == "C4/larry/1024/x4.0/s0"],
        "c4larry": lambda: [j for j in C.c4_jobs() if j[3].split("/")[1] == "larry"]}.get(which)
if jobs is None:  # a C4 label, e.g. C4/trail_plus/1024/x2.0/s7
    seed = int(which.rsplit("/s", 1)[1])
    jobs = [j for j in C.c4_jobs(seeds=[seed]) if j[3] == which]
else:
    jobs = jobs()
db = simulate.upload(I.make_batch(jobs))
for _ in range(reps):
    simulate.launch(db)
torch.cuda.synchronize()
print("done", which)
