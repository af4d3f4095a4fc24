import sys, os
sys.path.insert(0, '.')
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate
for j in C.c5_jobs(600.0, balancers=("sal",)) + [C.c2_jobs()[2]]:
    db = simulate.upload(I.make_batch([j]))
    for p in (1, 8, 32):
        os.environ["SSB_PIPE_PUBLISH"] = str(p)
        simulate.launch(db); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); simulate.launch(db); e1.record(); torch.cuda.synchronize()
        print(j[3], "publish", p, "noengine kernel ms", e0.elapsed_time(e1), flush=True)
