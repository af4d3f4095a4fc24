"""Records, summaries and capacity sweeps (drop-in for metrics.py).

``summarize`` computes the reference's Summary (metrics.py:57-99) exactly on
the device (csrc/ssb_summary.cu: radix-select nearest-rank percentiles);
``summarize_many`` does it for many record groups in one launch and also
returns the north-star extras (TPOT, queueing delay). ``percentile`` keeps the
reference's host helper for small lists. Writers reproduce the reference's
byte-stable CSV/JSON formats (metrics.py:115-165).
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import asdict, dataclass, fields
from pathlib import Path
from typing import Sequence

import numpy as np

from . import _abi


@dataclass(frozen=True)
class MetricsRecord:
    """Completion record for one request (metrics.py:20-43)."""

    request_id: int
    server: int
    arrival_time: float
    first_token_time: float
    finish_time: float
    prompt_len: int
    output_len: int
    preempt_count: int

    @property
    def ttft(self) -> float:
        return self.first_token_time - self.arrival_time

    @property
    def norm_ttft(self) -> float:
        return self.ttft / self.prompt_len

    @property
    def generation_time(self) -> float:
        return self.finish_time - self.arrival_time


def percentile(values: Sequence[float], p: float) -> float:
    """Nearest-rank percentile (metrics.py:46-54)."""
    if not values:
        raise ValueError("percentile of an empty sample")
    if not 0 < p <= 100:
        raise ValueError(f"p must be in (0, 100], got {p}")
    ordered = sorted(values)
    return ordered[math.ceil(p / 100 * len(ordered)) - 1]


@dataclass(frozen=True)
class Summary:
    """metrics.py:57-77 (same fields, same order)."""

    n_requests: int
    ttft_p50: float
    ttft_p95: float
    ttft_p99: float
    norm_ttft_p50: float
    norm_ttft_p95: float
    gen_time_p50: float
    gen_time_p95: float
    preemption_rate: float
    throughput_rps: float

    def to_dict(self) -> dict:
        return asdict(self)

    @staticmethod
    def field_names() -> list[str]:
        return [f.name for f in fields(Summary)]


@dataclass(frozen=True)
class SummaryExtras:
    """North-star metrics the reference does not compute:
    TPOT = (finish - first_token) / (output - 1) over requests with output > 1,
    queueing delay = first dispatch - arrival; nearest rank ceil(p*n/100)."""

    n_tpot: int
    tpot_p50: float
    tpot_p95: float
    tpot_p99: float
    queue_p50: float
    queue_p95: float
    queue_p99: float
    n_preempted: int


class RecordsSoA:
    """Structure-of-arrays records (what the device produces)."""

    def __init__(self, arrival, prompt, output, first_token, finish, preempt_count, server, first_dispatch=None):
        self.arrival = np.ascontiguousarray(arrival, dtype=np.float64)
        self.prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        self.output = np.ascontiguousarray(output, dtype=np.int32)
        self.first_token = np.ascontiguousarray(first_token, dtype=np.float64)
        self.finish = np.ascontiguousarray(finish, dtype=np.float64)
        self.preempt_count = np.ascontiguousarray(preempt_count, dtype=np.int32)
        self.server = np.ascontiguousarray(server, dtype=np.int32)
        self.first_dispatch = (np.full(len(self.arrival), np.nan) if first_dispatch is None
                               else np.ascontiguousarray(first_dispatch, dtype=np.float64))

    def __len__(self):
        return len(self.arrival)

    @classmethod
    def from_records(cls, records: Sequence[MetricsRecord]) -> "RecordsSoA":
        n = len(records)
        return cls(
            np.fromiter((r.arrival_time for r in records), np.float64, n),
            np.fromiter((r.prompt_len for r in records), np.int64, n),
            np.fromiter((r.output_len for r in records), np.int64, n),
            np.fromiter((r.first_token_time for r in records), np.float64, n),
            np.fromiter((r.finish_time for r in records), np.float64, n),
            np.fromiter((r.preempt_count for r in records), np.int64, n),
            np.fromiter((r.server for r in records), np.int64, n),
        )

    def to_records(self) -> list[MetricsRecord]:
        return [
            MetricsRecord(i, int(s), float(a), float(ft), float(fn), int(p), int(o), int(pc))
            for i, (s, a, ft, fn, p, o, pc) in enumerate(zip(self.server, self.arrival, self.first_token, self.finish,
                                                              self.prompt, self.output, self.preempt_count))
        ]


def _summary_from_row(row) -> tuple[Summary, SummaryExtras]:
    s = Summary(int(row["n_requests"]), float(row["ttft_p50"]), float(row["ttft_p95"]), float(row["ttft_p99"]),
                float(row["norm_ttft_p50"]), float(row["norm_ttft_p95"]), float(row["gen_time_p50"]),
                float(row["gen_time_p95"]), float(row["preemption_rate"]), float(row["throughput_rps"]))
    x = SummaryExtras(int(row["n_tpot"]), float(row["tpot_p50"]), float(row["tpot_p95"]), float(row["tpot_p99"]),
                      float(row["queue_p50"]), float(row["queue_p95"]), float(row["queue_p99"]),
                      int(row["n_preempted"]))
    return s, x


def nearest_ranks(n: int) -> tuple[int, int, int]:
    """ceil(p/100*n) in Python float arithmetic, exactly as metrics.py:53."""
    return tuple(math.ceil(p / 100 * n) for p in (50, 95, 99))


def summary_groups(offsets_n, trace_offsets=None, qps=None) -> np.ndarray:
    """ssb_summary_group array for consecutive record groups [(record_offset, n), ...].
    The nearest ranks are ceil(p/100*n) in binary64 exactly as Python computes them
    (metrics.py:53): p/100 and the product round the same way in numpy's float64."""
    on = np.asarray(offsets_n, dtype=np.int64).reshape(-1, 2)
    g = np.zeros(len(on), dtype=_abi.SUMMARY_GROUP)
    g["record_offset"] = on[:, 0]
    g["trace_offset"] = on[:, 0] if trace_offsets is None else np.asarray(trace_offsets, dtype=np.int64)
    g["n"] = on[:, 1]
    g["qps_factor"] = 1.0 if qps is None else np.asarray(qps, dtype=np.float64)
    nf = on[:, 1].astype(np.float64)
    for j, p in enumerate((50, 95, 99)):
        g["rank"][:, j] = np.ceil((p / 100) * nf)
    # TPOT ranks (3:) stay 0: derived on the device from the TPOT sample size
    return g


def instance_groups(inst: np.ndarray) -> np.ndarray:
    """summary_groups for every row of an INSTANCE array (one group per instance)."""
    return summary_groups(np.stack([inst["record_offset"], inst["n_requests"]], 1),
                          trace_offsets=inst["trace_offset"], qps=inst["qps_factor"])


def summarize_device(d_trace: _abi.SsbTrace, d_records: _abi.SsbRecords, groups: np.ndarray, device=None):
    """Run ssb_summarize for `groups` over device-resident trace/records; returns SUMMARY rows."""
    import torch

    lib = _abi.load_library()
    device = device or torch.device("cuda", torch.cuda.current_device())
    groups = np.ascontiguousarray(groups)
    d_groups = torch.from_numpy(groups.view(np.uint8)).to(device)
    wb = int(lib.ssb_summary_work_bytes(groups.ctypes.data, len(groups)))
    d_work = torch.empty(wb, dtype=torch.uint8, device=device)
    d_out = torch.empty(len(groups) * _abi.SUMMARY.itemsize, dtype=torch.uint8, device=device)
    rc = lib.ssb_summarize(d_trace, d_records, groups.ctypes.data, d_groups.data_ptr(), len(groups), d_out.data_ptr(),
                           d_work.data_ptr(), wb, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if rc != 0:
        raise RuntimeError(f"ssb_summarize: {lib.ssb_error_string(rc).decode()}")
    return d_out.cpu().numpy().view(_abi.SUMMARY).copy()


def summarize_many(soa: RecordsSoA, groups_n) -> list[tuple[Summary, SummaryExtras]]:
    """Summaries of consecutive groups of `soa` (one device launch)."""
    import torch

    for _, n in groups_n:
        if n < 1:
            raise ValueError("no records to summarize")
    dev = torch.device("cuda", torch.cuda.current_device())
    t = {k: torch.from_numpy(getattr(soa, k)).to(dev) for k in
         ("arrival", "prompt", "output", "first_token", "finish", "first_dispatch", "preempt_count", "server")}
    d_trace = _abi.SsbTrace(t["arrival"].data_ptr(), t["prompt"].data_ptr(), t["output"].data_ptr())
    d_rec = _abi.SsbRecords(t["first_token"].data_ptr(), t["finish"].data_ptr(), t["first_dispatch"].data_ptr(),
                            t["preempt_count"].data_ptr(), t["server"].data_ptr())
    rows = summarize_device(d_trace, d_rec, summary_groups(groups_n), dev)
    return [_summary_from_row(r) for r in rows]


def summarize(records) -> Summary:
    """Summary of one record set (metrics.py:80-99), computed on the device."""
    if isinstance(records, RecordsSoA):
        soa = records
    else:
        records = list(records)
        if not records:
            raise ValueError("no records to summarize")
        soa = RecordsSoA.from_records(records)
    if len(soa) == 0:
        raise ValueError("no records to summarize")
    return summarize_many(soa, [(0, len(soa))])[0][0]


def capacity_sweep(cluster_settings, trace, factors) -> list[tuple[float, Summary]]:
    """metrics.py:102-112 as ONE batched launch: every factor is an instance
    (scale_qps fused into the kernel's trace read); summaries on the device."""
    from .cluster import simulate_jobs

    jobs = [(cluster_settings, trace, float(f)) for f in factors]
    # per factor the reference's run_cluster raises (StallError / RuntimeError) instead of
    # summarising an incomplete run; scale_qps raises ValueError for factor <= 0 (make_batch)
    res = simulate_jobs(jobs, summaries=True, check=True)
    return [(float(f), r.summary) for f, r in zip(factors, res)]


_RECORD_COLUMNS = ["request_id", "server", "arrival_s", "first_token_s", "finish_s", "prompt_tokens",
                   "output_tokens", "preempt_count"]


def write_records_csv(path, records: Sequence[MetricsRecord]) -> None:
    """metrics.py:127-137 (repr floats: byte-stable reruns)."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    lines = [",".join(_RECORD_COLUMNS)]
    for r in records:
        lines.append(f"{r.request_id},{r.server},{r.arrival_time!r},{r.first_token_time!r},"
                     f"{r.finish_time!r},{r.prompt_len},{r.output_len},{r.preempt_count}")
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")


def write_summary_csv(path, rows: Sequence[dict]) -> None:
    """metrics.py:140-153."""
    if not rows:
        raise ValueError("no summary rows to write")
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    columns = list(rows[0].keys())
    lines = [",".join(columns)]
    for row in rows:
        if list(row.keys()) != columns:
            raise ValueError("summary rows have inconsistent columns")
        lines.append(",".join(repr(row[c]) if isinstance(row[c], float) else str(row[c]) for c in columns))
    path.write_text("\n".join(lines) + "\n", encoding="utf-8")


def write_summary_json(path, rows: Sequence[dict]) -> None:
    """metrics.py:162-165."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(list(rows), indent=2, sort_keys=False) + "\n", encoding="utf-8")
