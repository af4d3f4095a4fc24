import sys, os; sys.path.insert(0,'.')
os.environ["SSB_DEBUG_CLUSTERS"]="1"
import torch
from paper_2410_17840_b200 import configs as C, instances as I, simulate
for nseeds in (7, 8):
    jobs=[]
    for sd in range(nseeds): jobs += C.c5_jobs(3600.0, seed=sd)
    db = simulate.upload(I.make_batch(jobs)); simulate.launch(db); torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); simulate.launch(db); e1.record(); torch.cuda.synchronize()
    print(len(jobs), "clusters", e0.elapsed_time(e1), "ms", flush=True)
