"""Pooled exact percentiles over records spread across instances and GPUs.

``summarize(records)`` (metrics.py:80-99) over the *concatenation* of many
instances' records — e.g. BASELINE config 5 as independent seeds, one per
GPU — without moving any record between GPUs: an MSD radix select with 8-bit
digits on the order-preserving 64-bit image of each binary64 metric value.
Each pass every rank histograms its own records on the device
(``ssb_pool_hist``: 13 rank slots x 256 bins, only records matching the slot's
prefix so far), the histograms are all-gathered (NCCL on B200s, gloo in the
CPU tests) and summed, and every rank extends the slot prefixes by the digit
that holds the slot's rank. 8 passes give the exact order statistic, i.e.
``sorted(values)[ceil(p/100*n) - 1]`` of the union (metrics.py:46-54).

Slots (same per-record metrics as ``ssb_summarize``): TTFT p50/95/99,
normalised TTFT p50/95, TGT p50/95, TPOT p50/95/99 (output > 1 only), queueing
delay p50/95/99. Ranks: ``ceil(p/100*n)`` in Python float arithmetic, as the
reference's ``percentile`` (metrics.py:53), for every slot. The key order is
the IEEE total order, which agrees with ``sorted`` for every value a record
can produce (no NaN; differences of ordered times are +0.0, never -0.0).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _abi

SLOTS = (("ttft", 50), ("ttft", 95), ("ttft", 99), ("norm_ttft", 50), ("norm_ttft", 95), ("gen_time", 50),
         ("gen_time", 95), ("tpot", 50), ("tpot", 95), ("tpot", 99), ("queue", 50), ("queue", 95), ("queue", 99))
NSLOT = len(SLOTS)
PASSES = 8


def dkey(x: np.ndarray) -> np.ndarray:
    """Order-preserving uint64 image of binary64 values (larger value -> larger key)."""
    b = np.ascontiguousarray(x, dtype=np.float64).view(np.int64)
    u = b.view(np.uint64)
    return np.where(b < 0, ~u, u | np.uint64(1 << 63))


def dkey_inv(k: int) -> float:
    k = int(k)
    b = (k & ((1 << 63) - 1)) if (k >> 63) else (~k & ((1 << 64) - 1))
    return float(np.array([b], dtype=np.uint64).view(np.float64)[0])


def _gather_sum(t, dist):
    """Sum of a tensor over ranks through ONE all-gather (the north star's collective)."""
    if dist is None or dist.get_world_size() == 1:
        return t
    import torch

    world = dist.get_world_size()
    flat = t.contiguous().reshape(-1)
    out = torch.empty(world * flat.numel(), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, flat)
    return out.reshape((world,) + tuple(t.shape)).sum(dim=0)


def pooled_select(hist_fn, dist=None) -> dict:
    """Generic exact pooled radix select.

    ``hist_fn(pass, prefix: np.uint64[13], active: np.int32[13])`` returns
    ``(hist, counts)``: a torch int tensor [13, 256] of this rank's matching
    records per digit, and (pass 0 only, else None) a torch tensor [3] with
    this rank's {n, n_tpot, n_preempted}. Returns the pooled percentiles plus
    the pooled counts and preemption rate."""
    import torch

    prefix = np.zeros(NSLOT, dtype=np.uint64)
    active = np.ones(NSLOT, dtype=np.int32)
    k = np.zeros(NSLOT, dtype=np.int64)
    counts = None
    for p in range(PASSES):
        hist, cnt = hist_fn(p, prefix, active)
        hist = _gather_sum(hist.to(torch.int64), dist).cpu().numpy()
        if p == 0:
            counts = _gather_sum(cnt.to(torch.int64), dist).cpu().numpy()
            n, n_tpot = int(counts[0]), int(counts[1])
            for s, (metric, pct) in enumerate(SLOTS):
                m = n_tpot if metric == "tpot" else n
                k[s] = math.ceil(pct / 100 * m) if m > 0 else 0  # metrics.py:53
            active = (k > 0).astype(np.int32)
        shift = 56 - 8 * p
        for s in range(NSLOT):
            if k[s] <= 0:
                continue
            cum = np.cumsum(hist[s])
            d = int(np.searchsorted(cum, k[s]))  # first digit with cumulative count >= k
            if d > 255:
                raise RuntimeError("pooled select: rank outside the histogram (inconsistent ranks)")
            k[s] -= int(cum[d - 1]) if d > 0 else 0
            prefix[s] = np.uint64(int(prefix[s]) | (d << shift))
    out = {f"{m}_p{q}": (dkey_inv(prefix[s]) if k[s] > 0 else float("nan")) for s, (m, q) in enumerate(SLOTS)}
    n = int(counts[0])
    out.update(n_requests=n, n_tpot=int(counts[1]), n_preempted=int(counts[2]),
               preemption_rate=(int(counts[2]) / n) if n else float("nan"))
    return out


def device_hist_fn(d_trace: _abi.SsbTrace, d_records: _abi.SsbRecords, groups: np.ndarray, device=None):
    """hist_fn over device-resident trace/records for the ``groups`` of this rank (ssb_pool_hist)."""
    import torch

    lib = _abi.load_library()
    device = device or torch.device("cuda", torch.cuda.current_device())
    groups = np.ascontiguousarray(groups)
    d_groups = torch.from_numpy(groups.view(np.uint8)).to(device)
    d_work = torch.empty(8 * (len(groups) + 1), dtype=torch.uint8, device=device)
    d_hist = torch.empty((NSLOT, 256), dtype=torch.int32, device=device)
    d_counts = torch.empty(3, dtype=torch.int64, device=device)
    d_prefix = torch.empty(NSLOT, dtype=torch.int64, device=device)
    d_active = torch.empty(NSLOT, dtype=torch.int32, device=device)

    def fn(p, prefix, active):
        d_prefix.copy_(torch.from_numpy(prefix.view(np.int64)))
        d_active.copy_(torch.from_numpy(active))
        rc = lib.ssb_pool_hist(d_trace, d_records, groups.ctypes.data, d_groups.data_ptr(), len(groups),
                               d_prefix.data_ptr(), d_active.data_ptr(), p, d_hist.data_ptr(), d_counts.data_ptr(),
                               d_work.data_ptr(), d_work.numel(), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        if rc != 0:
            raise RuntimeError(f"ssb_pool_hist: {lib.ssb_error_string(rc).decode()}")
        return d_hist, (d_counts if p == 0 else None)

    return fn


def metric_values(arrival, prompt, output, first_token, finish, first_dispatch) -> dict:
    """Per-record metric arrays (binary64, the reference's operation order) — used by
    the host hist_fn of the CPU tests and as the numpy restatement."""
    ttft = first_token - arrival
    m = output > 1
    return {"ttft": ttft, "norm_ttft": ttft / prompt.astype(np.float64), "gen_time": finish - arrival,
            "tpot": (finish[m] - first_token[m]) / (output[m] - 1).astype(np.float64),
            "queue": first_dispatch - arrival}


def host_hist_fn(values: dict, preempt_count: np.ndarray):
    """hist_fn over host arrays (numpy): the same histograms ``ssb_pool_hist`` computes."""
    import torch

    keys = {k: dkey(v) for k, v in values.items()}

    def fn(p, prefix, active):
        shift = 56 - 8 * p
        hmask = 0 if p == 0 else ((~0 << (shift + 8)) & ((1 << 64) - 1))
        h = np.zeros((NSLOT, 256), dtype=np.int64)
        for s, (metric, _) in enumerate(SLOTS):
            if not active[s]:
                continue
            kk = keys[metric]
            sel = kk[(kk & np.uint64(hmask)) == (np.uint64(int(prefix[s])) & np.uint64(hmask))]
            h[s] = np.bincount(((sel >> np.uint64(shift)) & np.uint64(255)).astype(np.int64), minlength=256)
        cnt = None
        if p == 0:
            cnt = torch.tensor([len(values["ttft"]), len(values["tpot"]), int(np.count_nonzero(preempt_count > 0))],
                               dtype=torch.int64)
        return torch.from_numpy(h), cnt

    return fn


def pooled_summary_device(runner_or_db, dist=None) -> dict:
    """Pooled percentiles over every instance of a resident batch on this rank (and,
    with ``dist``, over every rank's batch): one ssb_pool_hist + one all-gather per pass."""
    from .metrics import instance_groups

    db = getattr(runner_or_db, "db", runner_or_db)
    h = db.h_inst
    g = instance_groups(h)
    return pooled_select(device_hist_fn(db.trace_c(), db.records_c(), g), dist)
