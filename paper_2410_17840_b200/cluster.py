"""Drop-in simulation entry points (cluster.py / engine.py of the reference).

* ``run_cluster(settings, trace, *, engines=None) -> list[MetricsRecord]``
  — cluster.py:65-174, same signature, validation, errors and results
  (bit-exact), computed by the sm_100a kernels.
* ``build_engine(settings) -> Engine`` and ``Engine(...).run(trace)``
  — cluster.py:28-47 / engine.py:236-265.
* ``simulate_jobs(jobs)`` — the batched form: many independent
  (settings, trace, qps_factor) instances in one device launch, records as
  structure-of-arrays, optional device summaries. This is what makes a sweep
  (capacity_sweep, BASELINE config 4) a single launch.

Errors mirror the reference: ValueError for unsorted traces / bad settings,
InfeasibleRequestError (policies.py:18) before simulating, StallError
(engine.py:138) and RuntimeError from the device status codes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _abi
from . import instances as I
from .metrics import MetricsRecord, RecordsSoA, Summary, SummaryExtras, instance_groups, summarize_device, _summary_from_row
from .policies import EngineLimits
from .settings import ClusterSettings, CostParams, EngineSettings, KvBlockPool
from .workload import Trace, as_trace


class StallError(RuntimeError):
    """The engine has work but cannot schedule a single token (engine.py:138-139)."""


def _raise_status(code: int, where: str) -> None:
    if code == _abi.SSB_OK:
        return
    lib = _abi.load_library()
    msg = f"{where}: {lib.ssb_error_string(code).decode()}"
    if code == _abi.SSB_E_STALL:
        raise StallError(msg)
    if code == _abi.SSB_E_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)


class Engine:
    """Engine descriptor (engine.py:142-169). ``run`` simulates a whole trace on
    the device; afterwards ``iterations``, ``peak_batch_tokens``,
    ``request_steps``, ``batch_tokens`` and (if ``record_events``)
    ``event_log`` describe what happened, like the reference's attributes."""

    def __init__(self, pool, policy, cost: CostParams, *, block_size: int = 16,
                 max_tokens_per_batch: int = 1024, max_running: int | None = None, max_context: int = 8192,
                 record_events: bool = False):
        if isinstance(pool, KvBlockPool):  # Engine(KvBlockPool(blocks, bs), policy, cost, ...) as in the reference
            pool_blocks, block_size = pool.total_blocks, pool.block_size
            self.pool = pool
        else:
            pool_blocks = int(pool)
            self.pool = KvBlockPool(pool_blocks, block_size)
        self.resolved = I.ResolvedEngine(policy=policy, pool_blocks=int(pool_blocks), block_size=int(block_size),
                                         cost=cost, limits=EngineLimits(max_tokens_per_batch, max_running,
                                                                        max_context))
        self.record_events = record_events
        self.policy = policy
        self.cost = cost
        self.limits = self.resolved.limits
        self._used = False
        self.iterations = 0
        self.peak_batch_tokens = 0
        self.request_steps = 0
        self.batch_tokens = 0
        self.clock = 0.0
        self.event_log: list[tuple[str, float, int, str]] = []

    def run(self, trace, validate: bool = True) -> list[MetricsRecord]:
        """engine.py:236-265 (a fresh engine is required)."""
        if self._used:
            raise RuntimeError("run() needs a fresh engine")
        settings = ClusterSettings(n_servers=1, engine=EngineSettings(max_tokens_per_batch=self.limits.max_tokens_per_batch))
        settings.balancer.name = "rr"
        return run_cluster(settings, trace, engines=[self], _validate=validate)

    def event_lines(self) -> list[str]:
        return [f"{ev},{t!r},{rid},{d}" for ev, t, rid, d in self.event_log]


def build_engine(settings: EngineSettings, *, record_events: bool = False) -> Engine:
    """cluster.py:28-47."""
    re = I.resolve_engine(settings)
    return Engine(re.pool_blocks, re.policy, re.cost, block_size=re.block_size,
                  max_tokens_per_batch=re.limits.max_tokens_per_batch, max_running=re.limits.max_running,
                  max_context=re.limits.max_context, record_events=record_events)


@dataclass
class JobResult:
    """One instance's outcome."""

    label: object
    records: RecordsSoA
    stats: np.void
    summary: Summary | None = None
    extras: SummaryExtras | None = None
    events: list = field(default_factory=list)
    engines: np.ndarray | None = None  # ENGINE_STATS rows, server order


def est_status(db, est) -> list[int]:
    """Each instance's status (the instance's own, else its first failing engine's)."""
    from . import simulate

    st = db.d_stats.cpu().numpy().view(_abi.STATS)["status"]
    rows = simulate.engine_rows(db)
    out = []
    for i in range(len(db.h_inst)):
        code = int(st[i])
        if code == _abi.SSB_OK:
            bad = est["status"][rows[i]:rows[i + 1]]
            bad = bad[bad != 0]
            code = int(bad[0]) if len(bad) else code
        out.append(code)
    return out


def simulate_jobs(jobs, *, summaries: bool = False, events: bool = False, validate: bool = True,
                  resolved=None, check: bool = False) -> list[JobResult]:
    """Simulate independent instances in one launch. jobs: (settings, trace[, qps_factor[, label]]).
    check=True raises the reference's exception (StallError / RuntimeError) for the first
    instance that did not complete, as a per-instance run_cluster call would.
    resolved: per job, the ResolvedEngine of prebuilt engines, or a list of one per server
    when they differ (each server batches, allocates and costs with its own)."""
    from . import simulate

    jobs = list(jobs)
    if resolved is None:
        batch = I.make_batch(jobs, validate=validate)
    else:  # explicit ResolvedEngine per job (prebuilt engines)
        recs, traces, n_rec = [], [], 0
        servers = {}
        for k, (job, re) in enumerate(zip(jobs, resolved)):
            t = as_trace(job[1])
            f = float(job[2]) if len(job) > 2 else 1.0
            per = list(re) if isinstance(re, (list, tuple)) else None
            if per is not None:  # every engine checks every request (cluster.py:86-88), engine order
                for r in per:
                    I.check_trace(t, r, f, feasibility=validate)
                servers[k] = np.array([I.engine_params_record(r) for r in per], dtype=_abi.ENGINE_PARAMS)
                re = per[0]
            else:
                I.check_trace(t, re, f, feasibility=validate)
            recs.append(I.instance_record(job[0], len(t), trace_offset=n_rec, record_offset=n_rec, qps_factor=f,
                                          resolved=re))
            traces.append(t)
            n_rec += len(t)
        tr = Trace(np.concatenate([t.arrival for t in traces]), np.concatenate([t.prompt for t in traces]),
                   np.concatenate([t.output for t in traces]))
        batch = I.Batch(tr, np.array(recs, dtype=_abi.INSTANCE), n_rec, [j[3] if len(j) > 3 else None for j in jobs],
                        servers)
    db, est = simulate.simulate_batch(batch, events=events)
    rows = simulate.engine_rows(db)
    if check:
        for i, st in enumerate(est_status(db, est)):
            _raise_status(st, f"instance {i} ({batch.labels[i] if i < len(batch.labels) else i})")
    srows = None
    if summaries:
        inst = db.h_inst
        groups = instance_groups(inst)
        ok = inst["n_requests"] > 0
        srows = np.zeros(len(inst), dtype=_abi.SUMMARY)
        if ok.any():
            srows[ok] = summarize_device(db.trace_c(), db.records_c(), groups[ok])
    out = simulate.download(db)
    rec, stats = out[0], out[1]
    results = []
    for i, inst in enumerate(db.h_inst):
        n, o, to = int(inst["n_requests"]), int(inst["record_offset"]), int(inst["trace_offset"])
        arr = batch.trace.arrival[to:to + n]
        f = float(inst["qps_factor"])
        if f != 1.0:
            arr = arr / f
        soa = RecordsSoA(arr, batch.trace.prompt[to:to + n], batch.trace.output[to:to + n],
                         rec.first_token[o:o + n], rec.finish[o:o + n], rec.preempt_count[o:o + n],
                         rec.server[o:o + n], rec.first_dispatch[o:o + n])
        r = JobResult(batch.labels[i] if i < len(batch.labels) else None, soa, stats[i],
                      engines=est[rows[i]:rows[i + 1]].copy())
        if srows is not None and n > 0:
            r.summary, r.extras = _summary_from_row(srows[i])
        if events:
            r.events = out[2][i]
        results.append(r)
    return results


def run_cluster(settings: ClusterSettings, trace, *, engines: list[Engine] | None = None,
                _validate: bool = True) -> list[MetricsRecord]:
    """cluster.py:65-174: one record per request, in request-id order."""
    n = settings.n_servers
    if engines is not None and len(engines) != n:
        raise ValueError(f"expected {n} engines, got {len(engines)}")
    resolved = None
    if engines is not None:
        r0 = engines[0].resolved
        for e in engines:
            if e._used:
                raise RuntimeError("run() needs a fresh engine")
        if all(e.resolved == r0 for e in engines[1:]):
            resolved = [r0]
        else:  # prebuilt engines that differ: one parameter set per server
            check_heterogeneous([e.resolved for e in engines])
            resolved = [[e.resolved for e in engines]]
    t = as_trace(trace)
    rec_events = bool(engines) and any(e.record_events for e in engines)
    res = simulate_jobs([(settings, t, 1.0)], events=rec_events, validate=_validate, resolved=resolved)[0]
    _raise_status(int(res.stats["status"]), "run_cluster")
    if engines is not None:
        for s, e in enumerate(engines):
            row = res.engines[s]
            e._used = True
            e.iterations = int(row["iterations"])  # engine.py:226
            e.peak_batch_tokens = int(row["peak_batch_tokens"])  # engine.py:225
            e.request_steps = int(row["request_steps"])
            e.batch_tokens = int(row["batch_tokens"])
            e.clock = float(row["clock"])
            if rec_events:
                e.event_log = event_log_with_details(res.events[s])
    return res.records.to_records()


def check_heterogeneous(res: list) -> None:
    """Engines of one cluster may differ in every parameter, policy included: up to 120 replicas
    each engine warp of the pipelined cluster kernel runs its own server's policy; beyond that
    the epoch kernel (several servers per warp) needs one policy kind."""
    from .policies import policy_descriptor

    if len(res) > 120 and len({policy_descriptor(r.policy)[0] for r in res}) != 1:
        raise NotImplementedError("more than 120 engines of different policies in one cluster are not supported "
                                  "on the device")


def event_log_with_details(ev) -> list[tuple[str, float, int, str]]:
    """One engine's device event stream as the reference's event_log (engine.py:165,273-274),
    detail strings included: a dispatch logs its dispatch_seq (the engine's running dispatch
    count, engine.py:294-298), a preempt / park the request's preempt_count after the
    increment (engine.py:372-379). Both are counters over this engine's own stream."""
    names = _abi.EVENT_NAMES
    out = []
    seq = 0
    pcount: dict[int, int] = {}
    for x in ev:
        code, rid, t = int(x["code"]), int(x["request_id"]), float(x["time"])
        if code == 1:  # dispatch
            detail = f"seq={seq}"
            seq += 1
        elif code in (2, 3):  # preempt / park
            c = pcount.get(rid, 0) + 1
            pcount[rid] = c
            detail = f"count={c}"
        else:
            detail = ""
        out.append((names[code], t, rid, detail))
    return out
