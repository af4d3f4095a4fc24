"""Instance sharding across GPUs (one process per GPU, torch.distributed).

Instances are independent, so the data path has no
collective: each rank simulates its shard; the only exchange is one
all-gather of fixed-size per-instance result rows (stats / summaries) at the
end, over NCCL on B200s (gloo in the CPU tests).
"""

from __future__ import annotations

import numpy as np


def weak_seed_range(rank: int, seeds_per_rank: int) -> range:
    """Weak scaling: rank r owns seeds [r*k, (r+1)*k) of the sweep."""
    return range(rank * seeds_per_rank, (rank + 1) * seeds_per_rank)


def strong_shard(costs, rank: int, world: int) -> np.ndarray:
    """Strong scaling: indices of the items rank `rank` owns, greedy
    longest-processing-time assignment by estimated cost (deterministic)."""
    costs = np.asarray(costs, dtype=np.float64)
    order = np.argsort(-costs, kind="stable")
    load = np.zeros(world)
    owner = np.empty(len(costs), dtype=np.int64)
    for i in order:
        r = int(np.argmin(load))
        owner[i] = r
        load[r] += costs[i]
    return np.flatnonzero(owner == rank)


def all_gather_rows(rows: np.ndarray, dist, device=None) -> np.ndarray:
    """All-gather equally sized structured-array shards (one collective)."""
    import torch

    world = dist.get_world_size()
    raw = torch.from_numpy(np.ascontiguousarray(rows).view(np.uint8).reshape(-1))
    if device is not None:
        raw = raw.to(device)
    out = torch.empty(world * raw.numel(), dtype=torch.uint8, device=raw.device)
    dist.all_gather_into_tensor(out, raw)
    return out.cpu().numpy().view(rows.dtype)
