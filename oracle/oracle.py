"""ctypes front end of the CPU oracle (oracle/ssb_oracle.c).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg, never by the product package.

* ``run_batch``   — run every instance of a ``Batch`` through the C restatement
                    of run_cluster (cluster.py:65-174) or Engine.run
                    (engine.py:236-265), optionally multi-threaded.
* ``summarize``   — numpy restatement of summarize/percentile
                    (metrics.py:46-99) plus the north-star extras (TPOT,
                    queueing delay) with the same nearest-rank rule.
* ``rng_integers``— the oracle's PCG64 Generator.integers model.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_2410_17840_b200 import _abi  # noqa: E402  (struct layouts only)

ORACLE_DIR = Path(__file__).resolve().parent
LIB = ORACLE_DIR / "libssb_oracle.so"
_lib = None


def build(force: bool = False) -> Path:
    deps = [ORACLE_DIR / "ssb_oracle.c", ROOT / "include" / "ssb.h"]
    if force or not LIB.exists() or any(LIB.stat().st_mtime < d.stat().st_mtime for d in deps):
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR), "-B" if force else "libssb_oracle.so"], check=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        lib = ctypes.CDLL(str(LIB))
        lib.ssb_oracle_run.restype = ctypes.c_int32
        lib.ssb_oracle_run.argtypes = [
            ctypes.c_void_p, _abi.SsbTrace, _abi.SsbRecords, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
        ]
        lib.ssb_oracle_run_many.restype = ctypes.c_int32
        lib.ssb_oracle_run_many.argtypes = [
            ctypes.c_void_p, ctypes.c_int32, _abi.SsbTrace, _abi.SsbRecords, ctypes.c_void_p,
            ctypes.c_int32, ctypes.c_int32,
        ]
        lib.ssb_oracle_set_trail_fast.restype = None
        lib.ssb_oracle_set_trail_fast.argtypes = [ctypes.c_int32]
        lib.ssb_oracle_rng_integers.restype = None
        lib.ssb_oracle_rng_integers.argtypes = [ctypes.c_uint64] * 4 + [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        sizes = np.zeros(len(_abi.STRUCT_ORDER), dtype=np.int64)
        lib.ssb_oracle_struct_sizes(sizes.ctypes.data)
        for name, got in zip(_abi.STRUCT_ORDER, sizes):
            assert int(got) == _abi.STRUCT_SIZES[name], (name, got)
        _lib = lib
    return _lib


class Records:
    """Host SoA of per-request results."""

    def __init__(self, n: int):
        self.first_token = np.full(n, np.nan)
        self.finish = np.full(n, np.nan)
        self.first_dispatch = np.full(n, np.nan)
        self.preempt_count = np.zeros(n, dtype=np.int32)
        self.server = np.full(n, -1, dtype=np.int32)

    def c(self) -> _abi.SsbRecords:
        return _abi.SsbRecords(
            self.first_token.ctypes.data, self.finish.ctypes.data, self.first_dispatch.ctypes.data,
            self.preempt_count.ctypes.data, self.server.ctypes.data,
        )


def _ctrace(trace) -> _abi.SsbTrace:
    return _abi.SsbTrace(trace.arrival.ctypes.data, trace.prompt.ctypes.data, trace.output.ctypes.data)


def run_batch(batch, *, mode: int = 0, threads: int = 1, events: bool = False, event_cap: int | None = None):
    """Run every instance; returns (records, stats[, events list per instance]).

    mode 0 = run_cluster heap loop; mode 1 = Engine.run (only for n_servers == 1)."""
    lib = load()
    inst = np.ascontiguousarray(batch.instances).copy()
    keep = []  # heterogeneous prebuilt engines: per-server parameter sets (h_servers)
    for i, srv in getattr(batch, "servers", {}).items():
        a = np.ascontiguousarray(srv, dtype=_abi.ENGINE_PARAMS)
        keep.append(a)
        inst[i]["h_servers"] = a.ctypes.data
    rec = Records(batch.n_records)
    stats = np.zeros(len(inst), dtype=_abi.STATS)
    tr = _ctrace(batch.trace)
    if not events:
        if threads > 1:
            lib.ssb_oracle_run_many(inst.ctypes.data, len(inst), tr, rec.c(), stats.ctypes.data, threads, mode)
        else:
            for i in range(len(inst)):
                lib.ssb_oracle_run(inst[i:i + 1].ctypes.data, tr, rec.c(), stats[i:i + 1].ctypes.data, None, 0, None,
                                   mode)
        return rec, stats
    evs = []
    for i in range(len(inst)):
        cap = event_cap or int(inst[i]["n_requests"]) * 16 + 64
        buf = np.zeros(cap, dtype=_abi.EVENT)
        cnt = np.zeros(1, dtype=np.int64)
        lib.ssb_oracle_run(inst[i:i + 1].ctypes.data, tr, rec.c(), stats[i:i + 1].ctypes.data, buf.ctypes.data, cap,
                           cnt.ctypes.data, mode)
        evs.append(buf[: min(int(cnt[0]), cap)].copy())
    return rec, stats, evs


def set_trail_fast(on: bool) -> None:
    """Single-engine trail_plus runs (mode 1) use the indexed waiting set (select_trail_fast):
    the same decisions, in time a 1M-request backlog allows (C3 at full size)."""
    load().ssb_oracle_set_trail_fast(1 if on else 0)


def rng_integers(seed_words, highs) -> np.ndarray:
    lib = load()
    highs = np.ascontiguousarray(highs, dtype=np.int64)
    out = np.zeros(len(highs), dtype=np.int64)
    lib.ssb_oracle_rng_integers(*[ctypes.c_uint64(w) for w in seed_words], highs.ctypes.data, len(highs),
                                out.ctypes.data)
    return out


def nearest_rank(n: int, p: float) -> int:
    """metrics.py:53 — Python float arithmetic."""
    return math.ceil(p / 100 * n)


def summarize(arrival, prompt, output, first_token, finish, preempt_count, first_dispatch=None) -> dict:
    """metrics.py:80-99 (+ TPOT / queueing-delay extras, same nearest-rank rule)."""
    n = len(arrival)
    if n == 0:
        raise ValueError("no records to summarize")
    ttft = first_token - arrival
    norm = ttft / prompt.astype(np.float64)
    gen = finish - arrival

    def pct(v, p):
        return float(np.sort(v, kind="stable")[nearest_rank(len(v), p) - 1])

    span = float(np.max(finish)) - float(np.min(arrival))
    preempted = int(np.count_nonzero(preempt_count > 0))
    out = {
        "n_requests": n,
        "ttft_p50": pct(ttft, 50), "ttft_p95": pct(ttft, 95), "ttft_p99": pct(ttft, 99),
        "norm_ttft_p50": pct(norm, 50), "norm_ttft_p95": pct(norm, 95),
        "gen_time_p50": pct(gen, 50), "gen_time_p95": pct(gen, 95),
        "preemption_rate": preempted / n,
        "throughput_rps": n / span if span > 0 else float("inf"),
    }
    m = output > 1
    tp = (finish[m] - first_token[m]) / (output[m] - 1).astype(np.float64)
    out["n_tpot"] = int(m.sum())
    for p in (50, 95, 99):
        out[f"tpot_p{p}"] = float(np.sort(tp)[(p * len(tp) + 99) // 100 - 1]) if len(tp) else float("nan")
    if first_dispatch is not None:
        q = first_dispatch - arrival
        for p in (50, 95, 99):
            out[f"queue_p{p}"] = float(np.sort(q)[(p * n + 99) // 100 - 1])
    return out
