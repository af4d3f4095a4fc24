"""Host-side instance planning: settings + trace -> ssb_instance descriptors.

Restates build_engine (cluster.py:28-47) and the up-front validation of
run_cluster (cluster.py:74-104) on the host, vectorised over requests, and
packs the result into the numpy mirror of ``ssb_instance`` (include/ssb.h).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .balancers import BALANCER_NAMES, BetaEstimator, pcg64_words
from .policies import EngineLimits, make_policy, policy_descriptor
from .settings import PROFILES, ClusterSettings, EngineSettings, default_params, pool_blocks_for
from .workload import Trace, as_trace


@dataclass
class ResolvedEngine:
    """What build_engine() derives from EngineSettings (cluster.py:28-47)."""

    policy: object
    pool_blocks: int
    block_size: int
    cost: object
    limits: EngineLimits


def resolve_engine(es: EngineSettings, policy=None) -> ResolvedEngine:
    if es.profile not in PROFILES:
        raise KeyError(es.profile)
    profile = PROFILES[es.profile]
    blocks = es.pool_blocks
    if blocks is None:
        blocks = pool_blocks_for(es.gpu_mem_bytes, profile, es.block_size)
    if blocks < 0:
        raise ValueError(f"total_blocks must be >= 0, got {blocks}")
    if es.block_size < 1:
        raise ValueError(f"block_size must be >= 1, got {es.block_size}")
    cost = default_params(es.profile, es.hardware, **es.cost)
    if policy is None:
        policy = make_policy(es.policy, alpha=es.alpha, c=es.c, max_output=es.max_output)
    limits = EngineLimits(es.max_tokens_per_batch, es.max_running, profile.max_context)
    return ResolvedEngine(policy, int(blocks), int(es.block_size), cost, limits)


def engine_params_record(re: ResolvedEngine) -> np.void:
    rec = np.zeros((), dtype=_abi.ENGINE_PARAMS)
    pid, alpha, c, max_output = policy_descriptor(re.policy)
    rec["policy"] = pid
    rec["max_output"] = max_output
    rec["alpha"] = alpha
    rec["c"] = c
    rec["block_size"] = re.block_size
    rec["pool_blocks"] = re.pool_blocks
    rec["max_tokens_per_batch"] = re.limits.max_tokens_per_batch
    rec["max_running"] = -1 if re.limits.max_running is None else re.limits.max_running
    rec["max_context"] = re.limits.max_context
    rec["mem_base_s"] = re.cost.mem_base_s
    rec["mem_per_kv_token_s"] = re.cost.mem_per_kv_token_s
    rec["compute_per_token_s"] = re.cost.compute_per_token_s
    rec["overhead_s"] = re.cost.overhead_s
    return rec


def check_qps_factor(qps_factor: float) -> float:
    """scale_qps's argument check (workload.py:187-194)."""
    f = float(qps_factor)
    if not f > 0 or not math.isfinite(f):
        raise ValueError(f"factor must be > 0, got {qps_factor}")
    return f


def check_trace(trace: Trace, re: ResolvedEngine, qps_factor: float = 1.0, *, feasibility: bool = True) -> None:
    """run_cluster's validation (cluster.py:80-92): the TraceEntry field checks
    (workload.py:50-56; a Trace built from arrays never ran them), sorted arrivals —
    both always, as the reference's run()/run_cluster do — then, unless
    ``feasibility`` is False (the reference's validate=False), check_feasible."""
    trace.validate()
    f = check_qps_factor(qps_factor)
    arr = trace.arrival if f == 1.0 else trace.arrival / f
    if len(arr) > 1 and np.any(arr[1:] < arr[:-1]):
        raise ValueError("trace arrivals must be sorted")
    if feasibility:
        re.policy.check_feasible_many(trace.prompt, trace.output, re.block_size, re.pool_blocks, re.limits)


def instance_record(
    settings: ClusterSettings,
    n_requests: int,
    *,
    trace_offset: int = 0,
    record_offset: int = 0,
    qps_factor: float = 1.0,
    resolved: ResolvedEngine | None = None,
    engine_rec: np.void | None = None,
) -> np.void:
    """One ssb_instance for run_cluster(settings, trace) (cluster.py:65-104). engine_rec: the
    resolved engine's ssb_engine_params when the caller already has it."""
    if settings.n_servers < 1:
        raise ValueError(f"n_servers must be >= 1, got {settings.n_servers}")
    bs = settings.balancer
    if bs.name not in BALANCER_NAMES:
        raise ValueError(f"unknown balancer {bs.name!r}; expected one of {BALANCER_NAMES}")
    if bs.poll_interval_s <= 0:
        raise ValueError(f"poll_interval_s must be > 0, got {bs.poll_interval_s}")  # balancers.py:35-36
    if bs.name == "sal":
        BetaEstimator(prior=bs.beta_prior)  # balancers.py:74-75
    re = resolved or resolve_engine(settings.engine)
    qps_factor = check_qps_factor(qps_factor)
    rec = np.zeros((), dtype=_abi.INSTANCE)
    rec["engine"] = engine_params_record(re) if engine_rec is None else engine_rec
    rec["n_servers"] = settings.n_servers
    rec["balancer"] = _abi.BALANCER_IDS[bs.name]
    rec["poll_interval_s"] = float(bs.poll_interval_s)
    rec["beta_prior"] = float(bs.beta_prior)
    rec["beta_fixed"] = math.nan if bs.beta_fixed is None else float(bs.beta_fixed)
    sh, sl, ih, il = pcg64_words(settings.seed)
    rec["pcg_state_hi"], rec["pcg_state_lo"], rec["pcg_inc_hi"], rec["pcg_inc_lo"] = sh, sl, ih, il
    rec["qps_factor"] = float(qps_factor)
    rec["trace_offset"] = trace_offset
    rec["record_offset"] = record_offset
    rec["n_requests"] = n_requests
    # SAL's cap comes from the settings, not from the (possibly prebuilt) engines (cluster.py:96-104)
    rec["route_cap"] = int(settings.engine.max_tokens_per_batch)
    return rec


@dataclass
class Batch:
    """A batch of instances over one concatenated trace."""

    trace: Trace
    instances: np.ndarray  # INSTANCE records
    n_records: int
    labels: list = field(default_factory=list)
    # instance index -> ENGINE_PARAMS array (n_servers rows) for clusters of prebuilt engines
    # that differ (run_cluster(..., engines=[...]), cluster.py:66-79); absent = homogeneous
    servers: dict = field(default_factory=dict)


def make_batch(jobs, *, validate: bool = True) -> Batch:
    """jobs: iterable of (settings, trace, qps_factor[, label]) -> one Batch (see
    _make_batch_serial for the checks). A sweep repeats few (settings, trace) pairs across many
    factors (C4: 256 pairs x 16 factors), so the per-object work runs once per distinct pair, in
    job order of first appearance (the serial order of every check), and the per-job columns
    are numpy gathers; a job list with an invalid factor takes the serial path, which raises the
    reference's error at the same job the serial loop would."""
    jobs = jobs if isinstance(jobs, list) else list(jobs)  # (keeps every keyed object alive)
    try:
        fac = np.asarray([j[2] if len(j) > 2 else 1.0 for j in jobs], dtype=np.float64)
    except (TypeError, ValueError):
        return _make_batch_serial(jobs, validate=validate)
    if len(jobs) == 0 or not bool(np.all((fac > 0) & np.isfinite(fac))):
        return _make_batch_serial(jobs, validate=validate)
    pairs = [(id(j[0]), id(j[1])) for j in jobs]
    pos = {k: q for q, k in enumerate(dict.fromkeys(pairs))}  # distinct pairs, first-appearance order
    if len(pos) == len(jobs):
        return _make_batch_serial(jobs, validate=validate)
    pidx = np.fromiter(map(pos.__getitem__, pairs), dtype=np.int64, count=len(pairs))
    first = np.unique(pidx, return_index=True)[1]  # each pair's first job, in pair order
    sub = _make_batch_serial([jobs[i] for i in first], validate=validate)
    inst = sub.instances[pidx]
    n = inst["n_requests"].astype(np.int64)
    inst["record_offset"] = np.cumsum(n) - n
    inst["qps_factor"] = fac
    labels = [j[3] if len(j) > 3 else None for j in jobs]
    return Batch(sub.trace, inst, int(n.sum()), labels)


def _make_batch_serial(jobs, *, validate: bool = True) -> Batch:
    """jobs: iterable of (settings, trace, qps_factor[, label]). Traces that are the
    same object are stored once and shared by offset (scale_qps is fused into
    the kernel's trace read).

    Sweeps repeat the same settings / trace objects across many jobs (C4: 256
    jobs per trace, 16 per settings object), so each check runs once per
    distinct object: the trace's field checks and sorted test once per trace
    (arrival / f for f > 0 is monotone under IEEE rounding, so a sorted trace
    stays sorted at every scale_qps factor), feasibility once per (trace,
    resolved engine limits), and the instance descriptor once per settings
    object (then copied with this job's offsets and factor)."""
    traces: list[Trace] = []
    trace_index: dict[int, int] = {}  # id(trace) -> [index, offset, length]
    keep_alive: list = []  # every keyed object lives until the loop ends, so no id() is reused
    base: dict[int, list] = {}  # id(settings) -> [ResolvedEngine, template index, feasibility key, params]
    engines: dict = {}  # engine settings values -> (ResolvedEngine, feasibility key, params)
    templates: list = []
    feasible: set = set()
    c_tpl: list = []
    c_n: list = []
    c_toff: list = []
    c_roff: list = []
    c_fac: list = []
    labels = []
    n_trace = 0
    n_records = 0
    isfinite = math.isfinite
    for job in jobs:
        trace = job[1]
        nj = len(job)
        factor = float(job[2]) if nj > 2 else 1.0
        if not (factor > 0 and isfinite(factor)):
            check_qps_factor(factor)  # raises the reference's error
        tr = trace_index.get(id(trace))
        if tr is None:
            t = as_trace(trace)
            t.validate()
            keep_alive.append(trace)
            tr = trace_index[id(trace)] = [len(traces), n_trace, len(t)]
            traces.append(t)
            n_trace += tr[2]
        settings = job[0]
        bs = base.get(id(settings))
        if bs is None:  # build_engine first (cluster.py:74-79), the balancer after the checks (:96-104)
            keep_alive.append(settings)
            es = settings.engine
            try:  # equal engine settings (a sweep repeats them per seed) resolve once
                ek = (es.policy, es.alpha, es.c, es.max_output, es.profile, es.hardware, es.block_size,
                      es.pool_blocks, es.gpu_mem_bytes, es.max_tokens_per_batch, es.max_running,
                      tuple(sorted(es.cost.items())))
                hit = engines.get(ek)
            except TypeError:  # (unhashable field values: no sharing)
                ek, hit = None, None
            if hit is None:
                r = resolve_engine(es)
                lim = r.limits
                hit = (r, (policy_descriptor(r.policy), r.block_size, r.pool_blocks, lim.max_tokens_per_batch,
                           lim.max_running, lim.max_context), engine_params_record(r))
                if ek is not None:
                    engines[ek] = hit
            bs = base[id(settings)] = [hit[0], -1, hit[1], hit[2]]
        if validate:
            fk = (tr[0], bs[2])
            if fk not in feasible:
                re, t = bs[0], traces[tr[0]]
                if len(tr) == 3:  # the trace's maxima, once: most (trace, engine) pairs pass on them alone
                    tr.append((int((t.prompt.astype(np.int64) + t.output).max()), int(t.prompt.max()),
                               int(t.output.max())) if len(t) else None)
                re.policy.check_feasible_many(t.prompt, t.output, re.block_size, re.pool_blocks, re.limits,
                                              maxes=tr[3])
                feasible.add(fk)
        if bs[1] < 0:  # the balancer's checks come after feasibility (cluster.py:90-104)
            bs[1] = len(templates)
            templates.append(instance_record(settings, 0, resolved=bs[0], engine_rec=bs[3]))
        c_tpl.append(bs[1])
        c_n.append(tr[2])
        c_toff.append(tr[1])
        c_roff.append(n_records)
        c_fac.append(factor)
        labels.append(job[3] if nj > 3 else None)
        n_records += tr[2]
    if traces:
        trace_all = Trace(
            np.concatenate([t.arrival for t in traces]),
            np.concatenate([t.prompt for t in traces]),
            np.concatenate([t.output for t in traces]),
        )
    else:
        trace_all = Trace(np.zeros(0), np.zeros(0), np.zeros(0))
    if c_tpl:
        inst = np.array(templates, dtype=_abi.INSTANCE)[np.array(c_tpl)]
        inst["n_requests"] = c_n
        inst["trace_offset"] = c_toff
        inst["record_offset"] = c_roff
        inst["qps_factor"] = np.array(c_fac, dtype=np.float64)
    else:
        inst = np.zeros(0, dtype=_abi.INSTANCE)
    return Batch(trace_all, inst, n_records, labels)
