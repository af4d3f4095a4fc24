"""Reference-side binding of libssb.so: what a servesim maintainer adds to route the
reference's own simulation path to the B200 kernels.

The reference's FFI for this path is ctypes. This module binds the C ABI of
include/ssb.h directly — ctypes + numpy struct mirrors (``_abi``) + torch for device
memory and the stream — and speaks only the reference's own objects:

* ``run_cluster(settings, trace, *, engines=None)`` — drop-in for
  ``servesim.cluster.run_cluster`` (cluster.py:65-174): the reference's validation
  (sorted arrivals, every engine's ``check_feasible``), one ``ssb_simulate`` call,
  the automatic re-run of shared-table overflows, the reference's exceptions
  (``StallError``, ``RuntimeError``), its ``MetricsRecord`` list; prebuilt engines get
  their ``iterations`` / ``peak_batch_tokens`` / ``clock`` (and, on request, an
  ``event_log`` with the reference's detail strings) from ``ssb_engine_stats_gather``.
* ``sweep_summaries(jobs)`` — many (settings, trace, qps_factor) runs as ONE
  ``ssb_simulate`` + ONE ``ssb_summarize`` (what ``cmd_sweep`` / ``capacity_sweep``
  become), returning the reference's ``Summary`` objects.
* ``cli_main(argv)`` — ``servesim.cli.main`` with ``--backend {python,b200}``
  (cli.py:205-214): ``b200`` routes ``cmd_run``'s ``run_cluster`` to the device and
  turns ``cmd_sweep`` into one batched launch; everything else (config parsing, trace
  files, writers, exit codes 0/1/2) stays the reference's.

The reference's classes are used when ``servesim`` is importable (the build
container); on a machine without it (the GPU box) the package's API mirror of the same
classes stands in, so the binding runs unchanged.
"""

from __future__ import annotations

import argparse
import ctypes
import dataclasses
import math
import sys

import numpy as np

from . import _abi
from .balancers import pcg64_words

POLICY_IDS = _abi.POLICY_IDS  # policies.py:279
BALANCER_IDS = _abi.BALANCER_IDS  # balancers.py:219


def _ref():
    """The reference's modules (servesim) if importable, else the API mirror."""
    try:
        from servesim import cluster, engine, metrics  # noqa: F401

        return {"build_engine": cluster.build_engine, "Request": engine.Request, "StallError": engine.StallError,
                "MetricsRecord": metrics.MetricsRecord, "Summary": metrics.Summary, "native": True}
    except ImportError:
        from . import cluster, metrics

        return {"build_engine": cluster.build_engine, "Request": None, "StallError": cluster.StallError,
                "MetricsRecord": metrics.MetricsRecord, "Summary": metrics.Summary, "native": False}


def _trace_columns(trace):
    if hasattr(trace, "arrival") and hasattr(trace, "prompt"):  # the package's SoA Trace
        return (np.ascontiguousarray(trace.arrival, np.float64), np.ascontiguousarray(trace.prompt, np.int32),
                np.ascontiguousarray(trace.output, np.int32))
    entries = list(trace)
    return (np.fromiter((e.arrival_time for e in entries), np.float64, len(entries)),
            np.fromiter((e.prompt_len for e in entries), np.int32, len(entries)),
            np.fromiter((e.output_len for e in entries), np.int32, len(entries)))


def _validate(engines, arr, prm, out, R):
    """cluster.py:80-92: sorted arrivals, then every engine's check_feasible per request."""
    if len(arr) > 1 and np.any(arr[1:] < arr[:-1]):
        raise ValueError("trace arrivals must be sorted")
    if R["native"]:
        for eng in engines:
            for i in range(len(arr)):
                eng.policy.check_feasible(R["Request"](id=i, arrival_time=float(arr[i]), prompt_len=int(prm[i]),
                                                       output_len=int(out[i])), eng.pool, eng.limits)
    else:
        for eng in engines:
            eng.policy.check_feasible_many(prm, out, eng.pool.block_size, eng.pool.total_blocks, eng.limits)


def _engine_key(eng):
    pol = eng.policy
    name = getattr(pol, "name", None)
    if name not in POLICY_IDS:
        raise NotImplementedError(f"{type(pol).__name__}: only the registry policies run on the B200 simulator")
    lim = eng.limits
    return (POLICY_IDS[name], float(getattr(pol, "alpha", 1.0)), float(getattr(pol, "c", 0.0)),
            int(getattr(pol, "max_output", 1024)), int(eng.pool.block_size), int(eng.pool.total_blocks),
            int(lim.max_tokens_per_batch), -1 if lim.max_running is None else int(lim.max_running),
            int(lim.max_context), float(eng.cost.mem_base_s), float(eng.cost.mem_per_kv_token_s),
            float(eng.cost.compute_per_token_s), float(eng.cost.overhead_s))


def engine_params(engine) -> np.void:
    """ssb_engine_params of one reference Engine (its policy, pool, limits and cost)."""
    (pid, alpha, c, max_output, bs, pool, cap, max_running, max_ctx, mb, mkv, comp, ovh) = _engine_key(engine)
    e = np.zeros((), dtype=_abi.ENGINE_PARAMS)
    e["policy"], e["alpha"], e["c"], e["max_output"] = pid, alpha, c, max_output
    e["block_size"], e["pool_blocks"], e["max_tokens_per_batch"] = bs, pool, cap
    e["max_running"], e["max_context"] = max_running, max_ctx
    e["mem_base_s"], e["mem_per_kv_token_s"], e["compute_per_token_s"], e["overhead_s"] = mb, mkv, comp, ovh
    return e


def instance_row(settings, engine, n_requests: int, *, trace_offset: int = 0, record_offset: int = 0,
                 qps_factor: float = 1.0) -> np.void:
    """One ssb_instance from a ClusterSettings (config.py:50-55) and an Engine built from it."""
    row = np.zeros((), dtype=_abi.INSTANCE)
    row["engine"] = engine_params(engine)
    b = settings.balancer
    if b.name not in BALANCER_IDS:
        raise ValueError(f"unknown balancer {b.name!r}")
    row["n_servers"], row["balancer"] = settings.n_servers, BALANCER_IDS[b.name]
    row["poll_interval_s"], row["beta_prior"] = float(b.poll_interval_s), float(b.beta_prior)
    row["beta_fixed"] = math.nan if b.beta_fixed is None else float(b.beta_fixed)
    row["pcg_state_hi"], row["pcg_state_lo"], row["pcg_inc_hi"], row["pcg_inc_lo"] = pcg64_words(settings.seed)
    row["qps_factor"] = float(qps_factor)
    row["trace_offset"], row["record_offset"], row["n_requests"] = trace_offset, record_offset, n_requests
    row["route_cap"] = int(settings.engine.max_tokens_per_batch)  # make_balancer's cap (cluster.py:96-104)
    return row


class _Device:
    """Device buffers + the raw ssb_simulate / ssb_engine_stats_gather / ssb_summarize calls."""

    def __init__(self, inst: np.ndarray, arr, prm, out, *, events: int = 0, servers: np.ndarray | None = None):
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("libssb.so needs a CUDA device (there is no CPU fallback)")
        self.torch, self.lib = torch, _abi.load_library()
        self.inst = np.ascontiguousarray(inst)
        dev = torch.device("cuda", torch.cuda.current_device())
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        if servers is not None:  # instance 0's engines differ: one ssb_engine_params per server
            self.h_servers = np.ascontiguousarray(servers, dtype=_abi.ENGINE_PARAMS)
            self.d_servers = to(self.h_servers.view(np.uint8))
            self.inst[0]["h_servers"] = self.h_servers.ctypes.data
            self.inst[0]["d_servers"] = self.d_servers.data_ptr()
        self.scratch_bytes = int(self.lib.ssb_prepare(self.inst.ctypes.data, len(self.inst)))
        self.d_arr, self.d_prm, self.d_out = to(arr), to(prm), to(out)
        n = len(arr) if len(inst) == 0 else int((inst["record_offset"] + inst["n_requests"]).max())
        self.n = n
        self.d_ft, self.d_fin, self.d_fd = (torch.empty(n, dtype=torch.float64, device=dev) for _ in range(3))
        self.d_pc, self.d_srv = (torch.empty(n, dtype=torch.int32, device=dev) for _ in range(2))
        self.d_stats = torch.zeros(len(inst) * _abi.STATS.itemsize, dtype=torch.uint8, device=dev)
        self.d_scratch = torch.empty(max(self.scratch_bytes, 256), dtype=torch.uint8, device=dev)
        ns = self.inst["n_servers"].astype(np.int64)
        self.rows = np.concatenate([[0], np.cumsum(ns)]).astype(np.int64)
        self.d_rows = to(self.rows[:-1])
        self.event_cap = int(events)
        self.dev = dev
        self._alloc_events()

    def _alloc_events(self):
        t = self.torch
        self.d_ev = (t.empty(len(self.inst) * self.event_cap * _abi.EVENT.itemsize, dtype=t.uint8, device=self.dev)
                     if self.event_cap else None)
        self.d_evc = t.zeros(max(len(self.inst), 1), dtype=t.int64, device=self.dev)  # events per instance

    def trace_c(self):
        return _abi.SsbTrace(self.d_arr.data_ptr(), self.d_prm.data_ptr(), self.d_out.data_ptr())

    def records_c(self):
        return _abi.SsbRecords(self.d_ft.data_ptr(), self.d_fin.data_ptr(), self.d_fd.data_ptr(), self.d_pc.data_ptr(),
                               self.d_srv.data_ptr())

    def _stream(self):
        return ctypes.c_void_p(self.torch.cuda.current_stream().cuda_stream)

    def simulate(self):
        d_inst = self.torch.from_numpy(self.inst.view(np.uint8)).to(self.dev)
        rc = self.lib.ssb_simulate(self.inst.ctypes.data, d_inst.data_ptr(), len(self.inst), self.trace_c(),
                                   self.records_c(), self.d_stats.data_ptr(), self.d_scratch.data_ptr(),
                                   self.scratch_bytes, self.d_ev.data_ptr() if self.d_ev is not None else None,
                                   self.event_cap, self.d_evc.data_ptr(), self._stream())
        if rc != 0:
            raise RuntimeError(f"ssb_simulate: {self.lib.ssb_error_string(rc).decode()}")
        self.d_inst = d_inst
        return self.d_stats.cpu().numpy().view(_abi.STATS).copy()

    def run(self):
        """ssb_simulate; instances whose shared running table overflowed (status 3) are
        re-run with global tables (SSB_FLAG_GLOBAL_TABLES), and the whole batch again with
        larger event rings while an engine's log outgrew its slice."""
        st = self.simulate()
        over = st["status"] == _abi.SSB_E_CAPACITY
        if over.any():
            self.inst["flags"][over] |= _abi.SSB_FLAG_GLOBAL_TABLES
            st = self.simulate()
        est = self.engine_stats()
        while self.event_cap:
            need, bad = 0, False
            for i, row in enumerate(self.inst):
                ns = int(row["n_servers"])
                m = int(est["event_count"][self.rows[i]:self.rows[i + 1]].max())
                bad |= m > self.event_cap // ns
                need = max(need, m * ns + 64 * ns)
            if not bad:
                break
            self.event_cap = need
            self._alloc_events()
            st = self.simulate()
            est = self.engine_stats()
        return st, est

    def engine_stats(self):
        out = self.torch.empty(int(self.rows[-1]) * _abi.ENGINE_STATS.itemsize, dtype=self.torch.uint8,
                               device=self.dev)
        rc = self.lib.ssb_engine_stats_gather(self.inst.ctypes.data, self.d_inst.data_ptr(), len(self.inst),
                                              self.d_scratch.data_ptr(), self.d_stats.data_ptr(), self.records_c(),
                                              self.d_evc.data_ptr(), self.d_rows.data_ptr(), out.data_ptr(),
                                              self._stream())
        if rc != 0:
            raise RuntimeError(f"ssb_engine_stats_gather: {self.lib.ssb_error_string(rc).decode()}")
        return out.cpu().numpy().view(_abi.ENGINE_STATS).copy()

    def records(self):
        """(first_token, finish, preempt_count, server) as numpy, request order."""
        return (self.d_ft.cpu().numpy(), self.d_fin.cpu().numpy(), self.d_pc.cpu().numpy(),
                self.d_srv.cpu().numpy())

    def events(self, i: int, s: int):
        ns = int(self.inst[i]["n_servers"])
        sl = self.event_cap // ns
        ev = self.d_ev.cpu().numpy().view(_abi.EVENT).reshape(len(self.inst), self.event_cap)[i, s * sl:(s + 1) * sl]
        return ev[ev["code"] >= 0]

    def summaries(self):
        """ssb_summarize over every instance (metrics.py:80-99)."""
        from .metrics import instance_groups

        g = np.ascontiguousarray(instance_groups(self.inst))
        d_g = self.torch.from_numpy(g.view(np.uint8)).to(self.dev)
        wb = int(self.lib.ssb_summary_work_bytes(g.ctypes.data, len(g)))
        work = self.torch.empty(max(wb, 8), dtype=self.torch.uint8, device=self.dev)
        out = self.torch.empty(len(g) * _abi.SUMMARY.itemsize, dtype=self.torch.uint8, device=self.dev)
        rc = self.lib.ssb_summarize(self.trace_c(), self.records_c(), g.ctypes.data, d_g.data_ptr(), len(g),
                                    out.data_ptr(), work.data_ptr(), wb, self._stream())
        if rc != 0:
            raise RuntimeError(f"ssb_summarize: {self.lib.ssb_error_string(rc).decode()}")
        return out.cpu().numpy().view(_abi.SUMMARY).copy()


def _raise(code: int, R) -> None:
    if code == _abi.SSB_OK:
        return
    msg = _abi.load_library().ssb_error_string(code).decode()
    if code == _abi.SSB_E_STALL:
        raise R["StallError"](msg)  # engine.py:209-214
    if code == _abi.SSB_E_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)  # engine.py:276-292, cluster.py:159-161


def run_cluster(settings, trace, *, engines=None, record_events: bool = False):
    """servesim.cluster.run_cluster (cluster.py:65-174) on the device."""
    from .cluster import event_log_with_details

    R = _ref()
    n = settings.n_servers
    if engines is None:
        engines = [R["build_engine"](settings.engine) for _ in range(n)]
    elif len(engines) != n:
        raise ValueError(f"expected {n} engines, got {len(engines)}")
    keys = [_engine_key(e) for e in engines]
    servers = None
    if len(set(keys)) != 1:  # prebuilt engines that differ: each server with its own parameters
        if n > 120 and len({k[0] for k in keys}) != 1:
            raise NotImplementedError("more than 120 engines of different policies in one cluster are not "
                                      "supported on the device")
        servers = np.array([engine_params(e) for e in engines], dtype=_abi.ENGINE_PARAMS)
    arr, prm, out = _trace_columns(trace)
    _validate(engines, arr, prm, out, R)
    inst = np.array([instance_row(settings, engines[0], len(arr))], dtype=_abi.INSTANCE)
    dev = _Device(inst, arr, prm, out, events=(len(arr) * 12 + 64) * n if record_events else 0, servers=servers)
    st, est = dev.run()
    _raise(int(st[0]["status"]), R)
    ft, fin, pc, srv = dev.records()
    for s, e in enumerate(engines):  # what the reference leaves on its engine objects (engine.py:160-167,225-226)
        e.iterations = int(est[s]["iterations"])
        e.peak_batch_tokens = int(est[s]["peak_batch_tokens"])
        e.clock = float(est[s]["clock"])
        if record_events:
            e.event_log = event_log_with_details(dev.events(0, s))
    MR = R["MetricsRecord"]
    return [MR(request_id=i, server=int(srv[i]), arrival_time=float(arr[i]), first_token_time=float(ft[i]),
               finish_time=float(fin[i]), prompt_len=int(prm[i]), output_len=int(out[i]),
               preempt_count=int(pc[i])) for i in range(len(arr))]


def sweep_summaries(jobs):
    """[(settings, trace, qps_factor)] -> [Summary], one ssb_simulate + one ssb_summarize.
    Arrivals are divided by qps_factor on the device exactly as scale_qps (workload.py:187-194)."""
    R = _ref()
    rows, cols, toff, roff = [], [], {}, 0
    n_trace = 0
    keep = []
    for settings, trace, f in jobs:
        f = float(f)
        if not f > 0:
            raise ValueError(f"factor must be > 0, got {f}")
        keep.append(trace)
        if id(trace) not in toff:
            c = _trace_columns(trace)
            toff[id(trace)] = n_trace
            cols.append(c)
            n_trace += len(c[0])
        c = cols[list(toff).index(id(trace))]
        engines = [R["build_engine"](settings.engine)]
        _validate(engines, c[0] / f if f != 1.0 else c[0], c[1], c[2], R)
        rows.append(instance_row(settings, engines[0], len(c[0]), trace_offset=toff[id(trace)], record_offset=roff,
                                 qps_factor=f))
        roff += len(c[0])
    inst = np.array(rows, dtype=_abi.INSTANCE)
    arr = np.concatenate([c[0] for c in cols])
    prm = np.concatenate([c[1] for c in cols])
    out = np.concatenate([c[2] for c in cols])
    if (inst["n_requests"] == 0).any():
        raise ValueError("no records to summarize")  # summarize() of an empty run (metrics.py:81-82)
    dev = _Device(inst, arr, prm, out)
    st, _ = dev.run()
    for code in st["status"]:
        _raise(int(code), R)
    S = R["Summary"]
    return [S(**{k: (int(r[k]) if k == "n_requests" else float(r[k])) for k in S.field_names()})
            for r in dev.summaries()]


def cli_main(argv=None) -> int:
    """servesim.cli.main with --backend {python,b200} (cli.py:205-214). The reference's
    parser, config handling, writers and exit codes are used unchanged; b200 swaps the
    simulation calls only."""
    from servesim import cli

    pre = argparse.ArgumentParser(add_help=False)
    pre.add_argument("--backend", choices=("python", "b200"), default="python")
    opts, rest = pre.parse_known_args(sys.argv[1:] if argv is None else argv)
    if opts.backend == "python":
        return cli.main(rest)
    saved = cli.run_cluster, cli._COMMANDS["sweep"]

    def cmd_sweep_b200(args) -> int:  # cli.py:137-159 as one batched launch
        cfg = cli._load_experiment(args)
        trace = cli.resolve_trace(cfg)
        keys = [(f, p, b) for f in cfg.sweep_factors for (p, b) in cli._combos(cfg)]
        summaries = sweep_summaries([(cli._settings_for(cfg, p, b), trace, f) for (f, p, b) in keys])
        rows = [{"factor": f, "policy": p, "balancer": b, **dataclasses.asdict(s)}
                for (f, p, b), s in zip(keys, summaries)]
        cli.write_summary_csv(args.out_dir / "sweep.csv", rows)
        cli.write_summary_json(args.out_dir / "sweep.json", rows)
        for row in rows:
            print(f"x{row['factor']:g} {row['policy']}/{row['balancer']}: "
                  f"ttft_p50={row['ttft_p50']:.4f}s ttft_p95={row['ttft_p95']:.4f}s")
        print(f"wrote {args.out_dir}/sweep.csv and {args.out_dir}/sweep.json")
        return 0

    cli.run_cluster = run_cluster
    cli._COMMANDS["sweep"] = cmd_sweep_b200
    try:
        return cli.main(rest)
    finally:
        cli.run_cluster, cli._COMMANDS["sweep"] = saved


if __name__ == "__main__":
    sys.exit(cli_main())
