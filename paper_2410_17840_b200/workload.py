"""Request traces as structure-of-arrays, synthesis and rate scaling.

Host-side input generation (out of the hot path). The
simulator consumes a ``Trace`` — three contiguous arrays (arrival f64,
prompt i32, output i32) — instead of a list of ``TraceEntry`` objects.

``synthesize`` is a vectorised restatement of workload.py:237-279 that is
bit-identical to it: the reference draws gamma gaps one scalar call at a
time until the cumulative time passes ``duration_s``; here the number of
gaps is found on a cloned generator and then exactly that many gammas are
drawn in one vector call (numpy's vector and scalar gamma consume the same
stream), followed by the same two lognormal vector draws. Cumulative sums use
``np.cumsum`` (sequential accumulation == the reference's ``t += g`` loop).
Pinned by tests/test_workload.py against golden trace hashes.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np


@dataclass(frozen=True)
class TraceEntry:
    """One request (workload.py:42-56)."""

    arrival_time: float
    prompt_len: int
    output_len: int

    def __post_init__(self):
        if self.arrival_time < 0:
            raise ValueError(f"arrival_time must be >= 0, got {self.arrival_time}")
        if self.prompt_len < 1:
            raise ValueError(f"prompt_len must be >= 1, got {self.prompt_len}")
        if self.output_len < 1:
            raise ValueError(f"output_len must be >= 1, got {self.output_len}")


@dataclass(frozen=True)
class LengthDist:
    """Log-normal token-length distribution (workload.py:197-206)."""

    location: float
    scale: float

    def __post_init__(self):
        if self.scale < 0:
            raise ValueError(f"scale must be >= 0, got {self.scale}")


@dataclass(frozen=True)
class SynthSpec:
    """Synthetic trace parameters (workload.py:209-234)."""

    duration_s: float
    mean_qps: float
    burstiness: float = 1.0
    prompt_dist: LengthDist = LengthDist(location=6.2, scale=1.1)
    output_dist: LengthDist = LengthDist(location=4.9, scale=0.9)
    max_context: int = 8192
    seed: int = 0

    def __post_init__(self):
        if self.duration_s <= 0:
            raise ValueError(f"duration_s must be > 0, got {self.duration_s}")
        if self.mean_qps <= 0:
            raise ValueError(f"mean_qps must be > 0, got {self.mean_qps}")
        if self.burstiness < 0:
            raise ValueError(f"burstiness must be >= 0, got {self.burstiness}")
        if self.max_context < 2:
            raise ValueError(f"max_context must be >= 2, got {self.max_context}")


class Trace:
    """SoA trace: arrival (f64, seconds, sorted), prompt / output (i32)."""

    __slots__ = ("arrival", "prompt", "output")

    def __init__(self, arrival, prompt, output):
        self.arrival = np.ascontiguousarray(arrival, dtype=np.float64)
        self.prompt = np.ascontiguousarray(prompt, dtype=np.int32)
        self.output = np.ascontiguousarray(output, dtype=np.int32)
        if not (len(self.arrival) == len(self.prompt) == len(self.output)):
            raise ValueError("trace columns differ in length")

    def __len__(self) -> int:
        return len(self.arrival)

    @classmethod
    def from_entries(cls, entries: Iterable[TraceEntry]) -> "Trace":
        if isinstance(entries, Trace):
            return entries
        entries = list(entries)
        return cls(
            np.fromiter((e.arrival_time for e in entries), np.float64, len(entries)),
            np.fromiter((e.prompt_len for e in entries), np.int64, len(entries)),
            np.fromiter((e.output_len for e in entries), np.int64, len(entries)),
        )

    def entries(self) -> list[TraceEntry]:
        return [TraceEntry(float(a), int(p), int(o)) for a, p, o in zip(self.arrival, self.prompt, self.output)]

    def digest(self) -> str:
        h = hashlib.sha256()
        for col in (self.arrival, self.prompt.astype(np.int64), self.output.astype(np.int64)):
            h.update(np.ascontiguousarray(col).tobytes())
        return h.hexdigest()[:32]

    def validate(self) -> None:
        """Same checks as the reference (workload.py:50-56, cluster.py:81-83)."""
        if len(self) == 0:
            return
        if np.any(self.arrival < 0):
            raise ValueError("arrival_time must be >= 0")
        if np.any(self.prompt < 1) or np.any(self.output < 1):
            raise ValueError("prompt_len and output_len must be >= 1")
        if np.any(np.diff(self.arrival) < 0):
            raise ValueError("trace arrivals must be sorted")


def as_trace(trace) -> Trace:
    return trace if isinstance(trace, Trace) else Trace.from_entries(trace)


def _gamma_count(rng_state, shape: float, scale: float, duration: float, hint: int) -> int:
    """Number of gamma draws the reference's loop consumes (gaps incl. the one past duration)."""
    probe = np.random.Generator(np.random.PCG64())
    probe.bit_generator.state = rng_state
    t = 0.0
    total = 0
    chunk = max(1024, hint)
    while True:
        g = probe.gamma(shape, scale, size=chunk)
        c = np.cumsum(np.concatenate(([t], g)))[1:]
        over = np.flatnonzero(c > duration)
        if over.size:
            return total + int(over[0]) + 1
        total += chunk
        t = float(c[-1])


def synthesize(spec: SynthSpec) -> Trace:
    """Bit-identical vectorised restatement of workload.py:237-279."""
    rng = np.random.default_rng(spec.seed)
    mean_gap = 1.0 / spec.mean_qps
    if spec.burstiness == 0:
        n = int(spec.duration_s / mean_gap)
        arrivals = np.array(
            [(i + 1) * mean_gap for i in range(n) if (i + 1) * mean_gap <= spec.duration_s], dtype=np.float64
        )
    else:
        shape = 1.0 / (spec.burstiness**2)
        scale = mean_gap * spec.burstiness**2
        total = _gamma_count(
            rng.bit_generator.state, shape, scale, spec.duration_s, int(spec.duration_s * spec.mean_qps * 1.1) + 16
        )
        gaps = rng.gamma(shape, scale, size=total)
        arrivals = np.cumsum(gaps)[: total - 1]
    n = len(arrivals)
    cap = spec.max_context - 1
    prompts = np.clip(np.rint(rng.lognormal(spec.prompt_dist.location, spec.prompt_dist.scale, n)), 1, cap).astype(
        np.int64
    )
    outputs = np.clip(np.rint(rng.lognormal(spec.output_dist.location, spec.output_dist.scale, n)), 1, cap).astype(
        np.int64
    )
    outputs = np.minimum(outputs, spec.max_context - prompts)
    return Trace(arrivals, prompts, outputs)


def scale_qps(trace, factor: float) -> Trace:
    """Divide arrival times by ``factor`` (workload.py:187-194). IEEE division == Python float division."""
    if factor <= 0:
        raise ValueError(f"factor must be > 0, got {factor}")
    t = as_trace(trace)
    return Trace(t.arrival / float(factor), t.prompt, t.output)


def concat(traces: Sequence[Trace]) -> tuple[Trace, np.ndarray]:
    """Concatenate traces; returns (trace, offsets[len+1])."""
    offs = np.zeros(len(traces) + 1, dtype=np.int64)
    for i, t in enumerate(traces):
        offs[i + 1] = offs[i] + len(t)
    return (
        Trace(
            np.concatenate([t.arrival for t in traces]) if traces else np.zeros(0),
            np.concatenate([t.prompt for t in traces]) if traces else np.zeros(0),
            np.concatenate([t.output for t in traces]) if traces else np.zeros(0),
        ),
        offs,
    )
