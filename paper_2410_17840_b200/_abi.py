"""numpy mirrors of the C structs in include/ssb.h and the libssb.so loader.

The loader fails loudly: there is no CPU fallback for the simulation path.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libssb.so"

POLICY_IDS = {"fcfs": 0, "nopreempt": 1, "trail_plus": 2, "larry": 3}
BALANCER_IDS = {"rr": 0, "random": 1, "p2c": 2, "sal": 3}
EVENT_NAMES = ("enqueue", "dispatch", "preempt", "park", "first_token", "finish")

SSB_FLAG_GLOBAL_TABLES = 1
SSB_OK, SSB_E_INFEASIBLE, SSB_E_STALL, SSB_E_CAPACITY, SSB_E_INVARIANT, SSB_E_CUDA, SSB_E_ARG = range(7)

ENGINE_PARAMS = np.dtype(
    [
        ("policy", "<i4"),
        ("max_output", "<i4"),
        ("alpha", "<f8"),
        ("c", "<f8"),
        ("block_size", "<i4"),
        ("pool_blocks", "<i4"),
        ("max_tokens_per_batch", "<i4"),
        ("max_running", "<i4"),
        ("max_context", "<i4"),
        ("_pad0", "<i4"),
        ("mem_base_s", "<f8"),
        ("mem_per_kv_token_s", "<f8"),
        ("compute_per_token_s", "<f8"),
        ("overhead_s", "<f8"),
    ],
    align=True,
)

INSTANCE = np.dtype(
    [
        ("engine", ENGINE_PARAMS),
        ("n_servers", "<i4"),
        ("balancer", "<i4"),
        ("poll_interval_s", "<f8"),
        ("beta_prior", "<f8"),
        ("beta_fixed", "<f8"),
        ("pcg_state_hi", "<u8"),
        ("pcg_state_lo", "<u8"),
        ("pcg_inc_hi", "<u8"),
        ("pcg_inc_lo", "<u8"),
        ("qps_factor", "<f8"),
        ("trace_offset", "<i8"),
        ("record_offset", "<i8"),
        ("n_requests", "<i8"),
        ("scratch_offset", "<i8"),
        ("wait_cap", "<i4"),
        ("run_cap", "<i4"),
        ("est_cost", "<i4"),
        ("flags", "<i4"),
        ("route_cap", "<i4"),
        ("_pad1", "<i4"),
        ("h_servers", "<u8"),
        ("d_servers", "<u8"),
        ("server_stride", "<i8"),
    ],
    align=True,
)

STATS = np.dtype(
    [
        ("iterations", "<i8"),
        ("request_steps", "<i8"),
        ("batch_tokens", "<i8"),
        ("dispatches", "<i8"),
        ("preempts", "<i8"),
        ("parks", "<i8"),
        ("finished", "<i8"),
        ("peak_batch_tokens", "<i8"),
        ("digest", "<u8"),
        ("status", "<i4"),
        ("_pad", "<i4"),
        ("device_cycles", "<i8"),
    ],
    align=True,
)

ENGINE_STATS = np.dtype(
    [
        ("iterations", "<i8"),
        ("request_steps", "<i8"),
        ("batch_tokens", "<i8"),
        ("dispatches", "<i8"),
        ("preempts", "<i8"),
        ("parks", "<i8"),
        ("finished", "<i8"),
        ("peak_batch_tokens", "<i8"),
        ("digest", "<u8"),
        ("event_count", "<i8"),
        ("clock", "<f8"),
        ("status", "<i4"),
        ("_pad", "<i4"),
    ],
    align=True,
)

EVENT = np.dtype([("time", "<f8"), ("request_id", "<i4"), ("server", "<i2"), ("code", "<i2")], align=True)

SUMMARY = np.dtype(
    [
        ("n_requests", "<i8"),
        ("ttft_p50", "<f8"),
        ("ttft_p95", "<f8"),
        ("ttft_p99", "<f8"),
        ("norm_ttft_p50", "<f8"),
        ("norm_ttft_p95", "<f8"),
        ("gen_time_p50", "<f8"),
        ("gen_time_p95", "<f8"),
        ("preemption_rate", "<f8"),
        ("throughput_rps", "<f8"),
        ("n_tpot", "<i8"),
        ("tpot_p50", "<f8"),
        ("tpot_p95", "<f8"),
        ("tpot_p99", "<f8"),
        ("queue_p50", "<f8"),
        ("queue_p95", "<f8"),
        ("queue_p99", "<f8"),
        ("n_preempted", "<i8"),
        ("max_finish", "<f8"),
        ("min_arrival", "<f8"),
    ],
    align=True,
)

SUMMARY_GROUP = np.dtype(
    [
        ("record_offset", "<i8"),
        ("trace_offset", "<i8"),
        ("n", "<i8"),
        ("qps_factor", "<f8"),
        ("rank", "<i8", (6,)),
    ],
    align=True,
)

STRUCT_SIZES = {
    "ssb_engine_params": ENGINE_PARAMS.itemsize,
    "ssb_instance": INSTANCE.itemsize,
    "ssb_stats": STATS.itemsize,
    "ssb_event": EVENT.itemsize,
    "ssb_summary": SUMMARY.itemsize,
    "ssb_summary_group": SUMMARY_GROUP.itemsize,
    "ssb_engine_stats": ENGINE_STATS.itemsize,
}
STRUCT_ORDER = ["ssb_engine_params", "ssb_instance", "ssb_stats", "ssb_event", "ssb_summary", "ssb_summary_group",
                "ssb_engine_stats"]
ABI_VERSION = 3


class SsbTrace(ctypes.Structure):
    _fields_ = [("arrival", ctypes.c_void_p), ("prompt", ctypes.c_void_p), ("output", ctypes.c_void_p)]


class SsbRecords(ctypes.Structure):
    _fields_ = [
        ("first_token", ctypes.c_void_p),
        ("finish", ctypes.c_void_p),
        ("first_dispatch", ctypes.c_void_p),
        ("preempt_count", ctypes.c_void_p),
        ("server", ctypes.c_void_p),
    ]


# exported C symbols (include/ssb.h) and their ctypes signatures
EXPORTS = {
    "ssb_abi_version": (ctypes.c_int32, []),
    "ssb_error_string": (ctypes.c_char_p, [ctypes.c_int32]),
    "ssb_prepare": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int32]),
    "ssb_simulate": (
        ctypes.c_int32,
        [
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            SsbTrace,
            SsbRecords,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
            ctypes.c_int64,
            ctypes.c_void_p,
            ctypes.c_void_p,
        ],
    ),
    "ssb_summary_work_bytes": (ctypes.c_size_t, [ctypes.c_void_p, ctypes.c_int32]),
    "ssb_summarize": (
        ctypes.c_int32,
        [
            SsbTrace,
            SsbRecords,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "ssb_pool_hist": (
        ctypes.c_int32,
        [
            SsbTrace,
            SsbRecords,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_int32,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_void_p,
            ctypes.c_size_t,
            ctypes.c_void_p,
        ],
    ),
    "ssb_struct_sizes": (ctypes.c_int32, [ctypes.c_void_p]),
    "ssb_engine_stats_gather": (
        ctypes.c_int32,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, SsbRecords,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
}

_LIB = None


class NativeLibraryMissing(RuntimeError):
    """libssb.so is not built: the simulation path has no CPU fallback."""


def load_library(path: os.PathLike | None = None) -> ctypes.CDLL:
    """Load libssb.so (in-tree). Raises NativeLibraryMissing if absent."""
    global _LIB
    if _LIB is not None and path is None:
        return _LIB
    p = Path(path) if path is not None else Path(os.environ.get("SSB_LIB", LIB_PATH))
    if not p.exists():
        raise NativeLibraryMissing(
            f"{p} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 simulation path has no CPU fallback)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ssb_abi_version() != ABI_VERSION:
        raise NativeLibraryMissing(f"{p}: ABI version mismatch")
    sizes = np.zeros(len(STRUCT_ORDER), dtype=np.int64)
    lib.ssb_struct_sizes(sizes.ctypes.data)
    for name, got in zip(STRUCT_ORDER, sizes):
        if int(got) != STRUCT_SIZES[name]:
            raise NativeLibraryMissing(f"{p}: sizeof({name}) = {got}, numpy mirror = {STRUCT_SIZES[name]}")
    if path is None:
        _LIB = lib
    return lib
