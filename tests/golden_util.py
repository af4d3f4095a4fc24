"""Digest helpers shared by the golden generator and the tests."""

from __future__ import annotations

import hashlib
import struct

import numpy as np

FNV_OFF = 0xCBF29CE484222325
FNV_PRIME = 0x100000001B3
MASK = (1 << 64) - 1
EVENT_CODES = {"enqueue": 0, "dispatch": 1, "preempt": 2, "park": 3, "first_token": 4, "finish": 5}


def event_digest(events) -> int:
    """FNV-1a (64-bit words) over (code, request_id, time bits) — DESIGN.md §digest."""
    h = FNV_OFF
    for code, rid, t in events:
        for w in (code, rid, struct.unpack("<Q", struct.pack("<d", t))[0]):
            h ^= w
            h = (h * FNV_PRIME) & MASK
    return h


def fold_digests(ds) -> int:
    h = FNV_OFF
    for d in ds:
        h ^= d
        h = (h * FNV_PRIME) & MASK
    return h


def records_sha(first_token, finish, preempt_count, server) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(first_token, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(finish, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(preempt_count, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(server, dtype=np.int64).tobytes())
    return h.hexdigest()[:32]


def trace_sha(arrival, prompt, output) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(arrival, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(prompt, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(output, dtype=np.int64).tobytes())
    return h.hexdigest()[:32]
