"""Device driver: marshal a batch of instances to libssb.so and run it on the GPU.

PyTorch provides device memory and the stream; the work is done by the
sm_100a kernels behind the C ABI (include/ssb.h). There is no CPU fallback:
without CUDA or without libssb.so every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _abi
from .instances import Batch


class SimulationError(RuntimeError):
    pass


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise SimulationError("the B200 simulator needs a CUDA device (no CPU fallback)")
    return torch


def _np_to_dev(torch, arr: np.ndarray, device):
    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(device, non_blocking=False)


def cost_features(batch: Batch) -> np.ndarray:
    """Per instance (n requests, offered load rho, estimated iterations), from the trace and
    the engine parameters alone -- no simulation. A fluid model of one engine: requests
    arrive at lam = n / (arrival span / qps_factor), each decodes mean(output) steps, so
    by Little's law the running set holds R = lam * mean(output) * L(R) requests, with
    L(R) = overhead + max(mem_base + mem_per_kv * R * ctx, compute * R) the step latency
    (costmodel.py:37-47) and ctx = mean(prompt + output / 2), inflated by the prefill share
    lam * mean(prompt) * compute; R is capped by the pool (pool tokens / ctx, or for
    nopreempt / the worst-case reservation min(max_context, prompt + max_output),
    policies.py:116-117). rho = the load at that cap; iterations = Σ(output + 1) / R."""
    inst = batch.instances
    tr = batch.trace
    n_inst = len(inst)
    out = np.zeros((n_inst, 3))
    if n_inst == 0:
        return out
    o = inst["trace_offset"].astype(np.int64)
    n = inst["n_requests"].astype(np.int64)
    p = tr.prompt.astype(np.float64)
    q = tr.output.astype(np.float64)
    cp = np.concatenate([[0.0], np.cumsum(p)])
    cq = np.concatenate([[0.0], np.cumsum(q)])
    e = inst["engine"]
    mo = e["max_output"].astype(np.float64)
    mc = e["max_context"].astype(np.float64)
    nz = np.maximum(n, 1)
    psum, qsum = cp[o + n] - cp[o], cq[o + n] - cq[o]
    pm, qm = psum / nz, qsum / nz
    ctx = pm + qm / 2
    # nopreempt: mean reservation, min(max_context, prompt + max_output) per request
    res = ctx.copy()
    npm = e["policy"] == 1
    if npm.any():  # per distinct (max_context, max_output): one clipped prefix sum over the whole trace
        for mci, moi in {(float(a), float(b)) for a, b in zip(mc[npm], mo[npm])}:
            sel = npm & (mc == mci) & (mo == moi)
            cr = np.concatenate([[0.0], np.cumsum(np.minimum(mci, p + moi))])
            res[sel] = np.where(n[sel] > 0, (cr[o[sel] + n[sel]] - cr[o[sel]]) / nz[sel], ctx[sel])
    last = np.where(n > 0, tr.arrival[np.minimum(o + np.maximum(n - 1, 0), max(len(tr.arrival) - 1, 0))], 0.0)
    first = np.where(n > 0, tr.arrival[np.minimum(o, max(len(tr.arrival) - 1, 0))], 0.0)
    span = np.maximum((last - first) / inst["qps_factor"], 1e-9)
    lam = nz / span
    rmax = np.maximum(1.0, e["pool_blocks"] * e["block_size"] / np.maximum(res, 1.0))
    oh, mb, mkv, cpt = e["overhead_s"], e["mem_base_s"], e["mem_per_kv_token_s"], e["compute_per_token_s"]
    pre = 1.0 / np.maximum(0.05, 1.0 - lam * pm * cpt)  # prefill share of the engine's time
    R = np.ones(n_inst)
    # R <- min(rmax, 0.5 R + 0.5 max(1, lam qm L(R) pre)), L(R) = oh + max(mb + mkv R ctx, cpt R):
    # in place, each product and sum rounded exactly as the plain expression would
    lq = lam * qm
    t1, t2 = np.empty(n_inst), np.empty(n_inst)
    for _ in range(60):
        np.multiply(mkv, R, out=t1)
        t1 *= ctx
        t1 += mb
        np.multiply(cpt, R, out=t2)
        np.maximum(t1, t2, out=t1)
        t1 += oh  # L
        t1 *= lq
        t1 *= pre
        np.maximum(t1, 1.0, out=t1)
        t1 *= 0.5
        R *= 0.5
        R += t1
        np.minimum(R, rmax, out=R)
    Lmax = oh + np.maximum(mb + mkv * rmax * ctx, cpt * rmax)
    out[:, 0] = nz
    out[:, 1] = np.maximum(lam * qm * Lmax * pre / rmax, 1e-3)
    out[:, 2] = np.maximum((qsum + n) / R, 1.0)
    return out


def cost_design(batch: Batch) -> np.ndarray:
    """Design matrix of the first-run model: [1, log n, log rho, log iterations_est,
    (log rho)^2, log pool, log pool x log rho, log qps_factor, log qps_factor x log pool,
    (log qps_factor)^2] per instance (cost_features + the pool and the arrival-rate factor)."""
    f = cost_features(batch)
    inst = batch.instances
    ln, lr, li = np.log(f[:, 0]), np.log(f[:, 1]), np.log(f[:, 2])
    lp = np.log(np.maximum(inst["engine"]["pool_blocks"].astype(np.float64), 1.0)) if len(inst) else np.zeros(0)
    lf = np.log(inst["qps_factor"].astype(np.float64)) if len(inst) else np.zeros(0)
    return np.stack([np.ones(len(f)), ln, lr, li, lr * lr, lp, lp * lr, lf, lf * lp, lf * lf], 1)


# log(iterations) ~ cost_design . ITER_COEF[policy] (fcfs, nopreempt, trail_plus, larry): least
# squares on two C4 sweeps the bench does not run (seeds 100-115, 200-215; tools/dump_c4_costs.py,
# tools/fit_cost_model.py, profiles/r02_cost_model.json), held-out rank correlation 0.98-0.995 on
# seeds 0-15; CYCLES_PER_ITER = each policy's mean device cycles per iteration there. Iterations x
# the policy's cycles per iteration is exactly what the measured (warm) schedule orders by, so
# the first run gets (nearly) the same placement. Only the placement uses it: results never do.
ITER_COEF = np.array([
    [2.7641, 0.1998, 0.5872, 0.6657, 0.0111, -0.0932, -0.0724, -1.2206, 0.1308, -0.0679],
    [0.7175, 0.1094, 0.0826, 0.9159, 0.0106, -0.0697, -0.0162, -0.6709, 0.0938, -0.0977],
    [1.1877, 0.1030, 0.6963, 0.7488, -0.0179, 0.0959, -0.0689, -1.1918, 0.1080, 0.0180],
    [3.0808, 0.2497, 0.6387, 0.6312, 0.0199, -0.1434, -0.0845, -1.4647, 0.1645, -0.0827],
])
CYCLES_PER_ITER = np.array([721.6, 332.9, 3516.0, 1446.4])


def estimate_cost(batch: Batch) -> np.ndarray:
    """Scheduling hint (estimated device cycles / 1024, the unit of measured_cost) for a
    first run: predicted iterations x the policy's cycles per iteration. Clusters
    (n_servers > 1) keep a work proxy (Σ output tokens): they run one per thread-block cluster."""
    inst = batch.instances
    if len(inst) == 0:
        return np.zeros(0, dtype=np.int64)
    X = cost_design(batch)
    pol = inst["engine"]["policy"].astype(np.int64) & 3
    cpi = CYCLES_PER_ITER
    if os.environ.get("SSB_CPI_SCALE"):  # experiments: per-policy scale of the cycles per iteration
        cpi = cpi * np.array([float(x) for x in os.environ["SSB_CPI_SCALE"].split(",")])
    cyc = np.exp(np.clip(np.einsum("ij,ij->i", X, ITER_COEF[pol]), 0.0, 40.0)) * cpi[pol]
    multi = inst["n_servers"] > 1
    if multi.any():
        csum = np.concatenate([[0], np.cumsum(batch.trace.output.astype(np.int64) + 1)])
        o, n = inst["trace_offset"].astype(np.int64), inst["n_requests"].astype(np.int64)
        cyc[multi] = (csum[o + n] - csum[o])[multi] * 1024.0
    return np.clip(cyc / 1024.0, 1, 2**31 - 1).astype(np.int64)


def measured_cost(h_inst: np.ndarray, stats: np.ndarray) -> np.ndarray | None:
    """Scheduling hint from a finished run: each instance's measured iteration count times
    its policy's cycles per iteration (CYCLES_PER_ITER, the cold model's). Raw per-instance
    cycles depend on what shared the SM with the instance (up to ~3x for trail_plus), so a
    schedule built from them oscillates between runs; iterations are exact. The run's own
    per-policy mean cycles per iteration gave SM shares that ran the C4 sweep at 135-142 ms
    against 118-125 ms with the fixed constants (A/B on one box, profiles/r02_cost_model_ab.txt).
    None if nothing was measured."""
    cyc = np.asarray(stats["device_cycles"], dtype=np.float64)
    it = np.asarray(stats["iterations"], dtype=np.float64)
    if len(cyc) == 0 or not (cyc > 0).all():
        return None
    pol = h_inst["engine"]["policy"]
    multi = h_inst["n_servers"] > 1
    cost = cyc.copy()
    for p in np.unique(pol):
        m = (pol == p) & ~multi
        if m.any() and it[m].sum() > 0:
            cost[m] = it[m] * CYCLES_PER_ITER[p & 3]
    return np.clip(cost // 1024, 1, 2**31 - 1).astype(h_inst["est_cost"].dtype)


@dataclass
class DeviceBatch:
    """All device buffers of one batch (inputs resident in HBM)."""

    batch: Batch
    h_inst: np.ndarray
    d_inst: object
    d_arrival: object
    d_prompt: object
    d_output: object
    d_ft: object
    d_fin: object
    d_fd: object
    d_pc: object
    d_srv: object
    d_stats: object
    d_scratch: object
    scratch_bytes: int
    d_events: object = None
    d_evcount: object = None
    event_cap: int = 0
    d_engine_offset: object = None  # row of (instance i, server 0) in the per-engine stats
    n_engines: int = 0
    h_servers: object = None  # per-server parameter sets of heterogeneous clusters (host, device):
    d_servers: object = None  # the instances hold raw pointers into these, so they live with the batch

    def trace_c(self) -> _abi.SsbTrace:
        return _abi.SsbTrace(self.d_arrival.data_ptr(), self.d_prompt.data_ptr(), self.d_output.data_ptr())

    def records_c(self) -> _abi.SsbRecords:
        return _abi.SsbRecords(self.d_ft.data_ptr(), self.d_fin.data_ptr(), self.d_fd.data_ptr(),
                               self.d_pc.data_ptr(), self.d_srv.data_ptr())


def upload(batch: Batch, *, device=None, events: bool = False, event_cap: int | None = None) -> DeviceBatch:
    torch = _torch()
    lib = _abi.load_library()
    device = device or torch.device("cuda", torch.cuda.current_device())
    h_inst = np.ascontiguousarray(batch.instances.copy())
    if len(h_inst):
        h_inst["est_cost"] = estimate_cost(batch)
    h_srv, d_srv = attach_servers(torch, batch, h_inst, device)
    scratch_bytes = int(lib.ssb_prepare(h_inst.ctypes.data, len(h_inst)))
    n = batch.n_records
    db = DeviceBatch(
        batch=batch,
        h_inst=h_inst,
        d_inst=_np_to_dev(torch, h_inst.view(np.uint8), device),
        d_arrival=_np_to_dev(torch, batch.trace.arrival, device),
        d_prompt=_np_to_dev(torch, batch.trace.prompt, device),
        d_output=_np_to_dev(torch, batch.trace.output, device),
        d_ft=torch.empty(n, dtype=torch.float64, device=device),
        d_fin=torch.empty(n, dtype=torch.float64, device=device),
        d_fd=torch.empty(n, dtype=torch.float64, device=device),
        d_pc=torch.empty(n, dtype=torch.int32, device=device),
        d_srv=torch.empty(n, dtype=torch.int32, device=device),
        d_stats=torch.zeros(len(h_inst) * _abi.STATS.itemsize, dtype=torch.uint8, device=device),
        d_scratch=torch.empty(max(scratch_bytes, 256), dtype=torch.uint8, device=device),
        scratch_bytes=scratch_bytes,
        h_servers=h_srv,
        d_servers=d_srv,
    )
    ns = h_inst["n_servers"].astype(np.int64) if len(h_inst) else np.zeros(0, np.int64)
    db.n_engines = int(ns.sum())
    db.d_engine_offset = _np_to_dev(torch, np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
                                    if len(ns) else np.zeros(1, np.int64), device)
    if events:
        # first guess: 4 events per request (enqueue, dispatch, first_token, finish) + 2 per
        # preemption; an engine that outgrows its slice is detected after the run
        # (ssb_engine_stats.event_count) and the batch re-runs with a larger ring
        cap = event_cap or int(max(1, max((int(i["n_requests"]) for i in h_inst), default=1)) * 12 + 64)
        cap = cap * int(max((int(i["n_servers"]) for i in h_inst), default=1))
        alloc_events(db, cap)
    return db


def attach_servers(torch, batch: Batch, h_inst: np.ndarray, device):
    """Point each heterogeneous cluster's h_servers / d_servers at its rows of one host
    array and its device copy (returned: the caller keeps both alive)."""
    if not batch.servers:
        return None, None
    idx = sorted(batch.servers)
    rows = [np.asarray(batch.servers[i], dtype=_abi.ENGINE_PARAMS) for i in idx]
    for i, r in zip(idx, rows):
        if len(r) != int(h_inst[i]["n_servers"]):
            raise ValueError(f"instance {i}: {len(r)} engine parameter sets for {int(h_inst[i]['n_servers'])} servers")
    h_srv = np.ascontiguousarray(np.concatenate(rows))
    d_srv = _np_to_dev(torch, h_srv.view(np.uint8), device)
    sz = _abi.ENGINE_PARAMS.itemsize
    off = 0
    for i, r in zip(idx, rows):
        h_inst[i]["h_servers"] = h_srv.ctypes.data + off * sz
        h_inst[i]["d_servers"] = d_srv.data_ptr() + off * sz
        off += len(r)
    return h_srv, d_srv


def alloc_events(db: DeviceBatch, cap: int) -> None:
    """(Re)allocate the per-instance event rings: `cap` entries per instance, split evenly
    between the instance's servers by the kernels."""
    torch = _torch()
    device = db.d_inst.device
    db.event_cap = int(cap)
    db.d_events = torch.empty(len(db.h_inst) * db.event_cap * _abi.EVENT.itemsize, dtype=torch.uint8, device=device)
    db.d_evcount = torch.zeros(len(db.h_inst), dtype=torch.int64, device=device)


def engine_stats(db: DeviceBatch, stream=None) -> np.ndarray:
    """Per-engine counters of the last simulation (ENGINE_STATS rows; instance i's server
    s at row offsets[i] + s). Synchronises."""
    torch = _torch()
    lib = _abi.load_library()
    if stream is None:
        stream = torch.cuda.current_stream()
    out = torch.empty(max(db.n_engines, 1) * _abi.ENGINE_STATS.itemsize, dtype=torch.uint8, device=db.d_inst.device)
    rc = lib.ssb_engine_stats_gather(db.h_inst.ctypes.data, db.d_inst.data_ptr(), len(db.h_inst),
                                     db.d_scratch.data_ptr(), db.d_stats.data_ptr(), db.records_c(),
                                     db.d_evcount.data_ptr() if db.d_evcount is not None else None,
                                     db.d_engine_offset.data_ptr(), out.data_ptr(),
                                     ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise SimulationError(f"ssb_engine_stats_gather: {lib.ssb_error_string(rc).decode()} ({rc})")
    return out.cpu().numpy().view(_abi.ENGINE_STATS)[: db.n_engines].copy()


def engine_rows(db: DeviceBatch) -> np.ndarray:
    """Row offset of each instance's first engine in engine_stats()."""
    ns = db.h_inst["n_servers"].astype(np.int64)
    return np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)


def event_overflow_cap(db: DeviceBatch, est: np.ndarray) -> int:
    """0 if every engine's events fit its ring slice, else the per-instance capacity that
    makes the largest engine log fit (the kernels never drop an event silently: they keep
    counting past the slice, and this is where the count is read)."""
    if db.d_events is None or len(est) == 0:
        return 0
    rows = engine_rows(db)
    need = 0
    over = False
    for i, inst in enumerate(db.h_inst):
        ns = int(inst["n_servers"])
        cnt = est["event_count"][rows[i]:rows[i + 1]]
        m = int(cnt.max()) if len(cnt) else 0
        over |= m > db.event_cap // ns
        need = max(need, m * ns)
    return need + 64 * int(db.h_inst["n_servers"].max()) if over else 0


def launch(db: DeviceBatch, stream=None) -> None:
    """Enqueue the simulation kernels on `stream` (default: torch's current stream)."""
    torch = _torch()
    lib = _abi.load_library()
    if stream is None:
        stream = torch.cuda.current_stream()
    rc = lib.ssb_simulate(
        db.h_inst.ctypes.data, db.d_inst.data_ptr(), len(db.h_inst), db.trace_c(), db.records_c(),
        db.d_stats.data_ptr(), db.d_scratch.data_ptr(), db.scratch_bytes,
        db.d_events.data_ptr() if db.d_events is not None else None, db.event_cap,
        db.d_evcount.data_ptr() if db.d_evcount is not None else None, ctypes.c_void_p(stream.cuda_stream),
    )
    if rc != 0:
        raise SimulationError(f"ssb_simulate: {lib.ssb_error_string(rc).decode()} ({rc})")


class HostResults:
    def __init__(self, n):
        self.first_token = np.empty(n)
        self.finish = np.empty(n)
        self.first_dispatch = np.empty(n)
        self.preempt_count = np.empty(n, dtype=np.int32)
        self.server = np.empty(n, dtype=np.int32)


def download(db: DeviceBatch):
    """Device -> host: (records, stats[, events per instance])."""
    rec = HostResults(db.batch.n_records)
    rec.first_token = db.d_ft.cpu().numpy()
    rec.finish = db.d_fin.cpu().numpy()
    rec.first_dispatch = db.d_fd.cpu().numpy()
    rec.preempt_count = db.d_pc.cpu().numpy()
    rec.server = db.d_srv.cpu().numpy()
    stats = db.d_stats.cpu().numpy().view(_abi.STATS).copy()
    if db.d_events is None:
        return rec, stats
    ev = db.d_events.cpu().numpy().view(_abi.EVENT).reshape(len(db.h_inst), db.event_cap)
    per = []
    for i, inst in enumerate(db.h_inst):
        ns = int(inst["n_servers"])
        sl = db.event_cap // ns
        lists = []
        for s in range(ns):
            seg = ev[i, s * sl:(s + 1) * sl]
            valid = seg[seg["code"] >= 0]
            lists.append(valid.copy())
        per.append(lists)
    return rec, stats, per


def retry_overflows(db: DeviceBatch, stats_host: np.ndarray | None = None) -> int:
    """Re-run, with global running tables, every instance whose shared-memory
    running table overflowed (status SSB_E_CAPACITY). Returns the count."""
    torch = _torch()
    lib = _abi.load_library()
    if stats_host is None:
        stats_host = db.d_stats.cpu().numpy().view(_abi.STATS)
    redo = np.flatnonzero((stats_host["status"] == _abi.SSB_E_CAPACITY)
                          & ((db.h_inst["flags"] & _abi.SSB_FLAG_GLOBAL_TABLES) == 0))
    if len(redo) == 0:
        return 0
    sub = db.h_inst[redo].copy()
    sub["flags"] |= _abi.SSB_FLAG_GLOBAL_TABLES
    db.h_inst["flags"][redo] |= _abi.SSB_FLAG_GLOBAL_TABLES
    d_sub = _np_to_dev(torch, sub.view(np.uint8), db.d_inst.device)
    d_st = torch.zeros(len(sub) * _abi.STATS.itemsize, dtype=torch.uint8, device=db.d_inst.device)
    stream = torch.cuda.current_stream()
    rc = lib.ssb_simulate(sub.ctypes.data, d_sub.data_ptr(), len(sub), db.trace_c(), db.records_c(),
                          d_st.data_ptr(), db.d_scratch.data_ptr(), db.scratch_bytes, None, 0, None,
                          ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise SimulationError(f"ssb_simulate: {lib.ssb_error_string(rc).decode()} ({rc})")
    # scatter the re-run stats into their slots
    rows = db.d_stats.view(len(db.h_inst), _abi.STATS.itemsize)
    rows[torch.as_tensor(redo, device=rows.device)] = d_st.view(len(sub), _abi.STATS.itemsize)
    db.d_inst = _np_to_dev(torch, db.h_inst.view(np.uint8), db.d_inst.device)  # later launches keep the flag
    return len(redo)


def simulate_batch(batch: Batch, *, events: bool = False, event_cap: int | None = None):
    """Upload, simulate (re-running shared-table overflows with global tables, and the
    whole batch with larger event rings if any engine's log outgrew its slice).
    Returns (db, per-engine stats)."""
    torch = _torch()
    db = upload(batch, events=events, event_cap=event_cap)
    launch(db)
    torch.cuda.synchronize()
    if retry_overflows(db):
        if events:  # event slices are indexed by instance: re-run the whole batch
            launch(db)
        torch.cuda.synchronize()
    est = engine_stats(db)
    while events:
        cap = event_overflow_cap(db, est)
        if not cap:
            break
        alloc_events(db, cap)
        launch(db)
        torch.cuda.synchronize()
        est = engine_stats(db)
    return db, est


def run_batch(batch: Batch, *, events: bool = False, event_cap: int | None = None, check: bool = False,
              with_engines: bool = False):
    """Upload, simulate, download. Returns (records, stats[, events][, engine stats])."""
    db, est = simulate_batch(batch, events=events, event_cap=event_cap)
    out = download(db)
    if with_engines:
        out = (*out, est)
    if check:
        bad = np.flatnonzero(out[1]["status"] != 0)
        if len(bad):
            lib = _abi.load_library()
            code = int(out[1]["status"][bad[0]])
            raise SimulationError(f"instance {int(bad[0])}: {lib.ssb_error_string(code).decode()} ({code})")
    return out
