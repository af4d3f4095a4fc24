"""BASELINE config 5 as independent seeds across GPUs with pooled percentile aggregation.

Each rank simulates C5 (64 replicas, chat-shaped 224 qps, burstiness 3) for its own seed
(sal and rr, one thread-block cluster per instance), then the TTFT / normalised TTFT / TGT /
TPOT / queueing-delay percentiles of ALL ranks' records are computed exactly with one
all-gather of 13 x 256 histogram counts per radix pass (pooled.py, ssb_pool_hist) — no
record leaves its GPU.

    python tools/c5_pooled.py [duration_s]                                  # 1 GPU
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/c5_pooled.py  # N GPUs (seed = rank)
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2410_17840_b200 import configs as C  # noqa: E402
from paper_2410_17840_b200 import instances as I  # noqa: E402
from paper_2410_17840_b200 import simulate  # noqa: E402
from paper_2410_17840_b200.pooled import pooled_summary_device  # noqa: E402


def main():
    dur = float(sys.argv[1]) if len(sys.argv) > 1 else 44_643.0
    rank, world = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0"))))
    batch = I.make_batch(C.c5_jobs(dur, seed=rank))
    db = simulate.upload(batch)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    simulate.launch(db)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pooled = pooled_summary_device(db, dist)
    e2.record()
    torch.cuda.synchronize()
    t_pool = time.perf_counter() - t0
    st = simulate.download(db)[1]
    assert (st["status"] == 0).all()
    sim_ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([sim_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sim_ms = float(t.item())
    if rank == 0:
        print(json.dumps({"world": world, "duration_s": dur, "instances_per_rank": len(batch.instances),
                          "requests_per_rank": int(batch.n_records), "simulate_ms_max_over_ranks": sim_ms,
                          "pooled_aggregation_ms": 1e3 * t_pool, "pooled": pooled}, indent=1))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
