"""Strong scaling of the BASELINE C4 sweep, predicted on one GPU: the 4,096 instances are split
into N shards exactly as bench.py --scaling strong does (shard.strong_shard, LPT by the host cost
estimate), each shard is timed alone (cold first-run schedule, CUDA events, second launch), and
the N-GPU step is the slowest shard (the ranks share nothing but the final all-gather).
usage: python tools/probe_strong.py [1 2 4 8]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_17840_b200 import configs as C, instances as I, simulate  # noqa: E402
from paper_2410_17840_b200.shard import strong_shard  # noqa: E402

worlds = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
jobs = C.c4_jobs()
cost = simulate.estimate_cost(I.make_batch(jobs))
res = {}
for w in worlds:
    ms = []
    for r in range(w):
        db = simulate.upload(I.make_batch([jobs[i] for i in strong_shard(cost, r, w)]))
        simulate.launch(db)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        simulate.launch(db)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        del db
    res[w] = {"shard_ms": [round(x, 2) for x in ms], "step_ms": max(ms)}
    print(f"N={w}: slowest shard {max(ms):7.2f} ms  (shards {', '.join(f'{x:.1f}' for x in ms)})  "
          f"speed-up {res[worlds[0]]['step_ms'] / max(ms) * worlds[0]:.2f}x", flush=True)
print(json.dumps(res))
