"""Resident-buffer sweep runner: the batched public API used for policy/config
sweeps (BASELINE config 4, capacity_sweep).

``SweepRunner(jobs)`` plans the instances once, keeps pinned host copies of
the inputs and device buffers for everything, and ``run()`` performs one full
sweep: host->device copy of the trace and instance table, the simulation
kernels, the device summaries of every instance, device->host copy of the
per-instance stats and summaries. ``run(copy_inputs=False,
read_results=False)`` is the kernel-only form (inputs already in HBM).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _abi
from . import instances as I
from .metrics import instance_groups
from .simulate import DeviceBatch, SimulationError, estimate_cost, retry_overflows

SUMMARY_LAUNCHES = 18  # radix path: k_init + 8 x (k_hist + k_select) + k_finish
SMALL_GROUP_MAX = 4096  # every group this small: one k_small_summary launch (ssb_summary.cu)


class SweepRunner:
    def __init__(self, jobs, *, device=None, validate: bool = True):
        import torch

        if not torch.cuda.is_available():
            raise SimulationError("the B200 simulator needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.lib = _abi.load_library()
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.batch = I.make_batch(jobs, validate=validate)
        b = self.batch
        h_inst = np.ascontiguousarray(b.instances.copy())
        h_inst["est_cost"] = estimate_cost(b)
        self.scratch_bytes = int(self.lib.ssb_prepare(h_inst.ctypes.data, len(h_inst)))
        self.h_inst = h_inst
        n = b.n_records
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        self.p_arrival, self.p_prompt, self.p_output = pin(b.trace.arrival), pin(b.trace.prompt), pin(b.trace.output)
        self.p_inst = pin(h_inst.view(np.uint8))
        dev = self.device
        self.d_arrival = torch.empty_like(self.p_arrival, device=dev)
        self.d_prompt = torch.empty_like(self.p_prompt, device=dev)
        self.d_output = torch.empty_like(self.p_output, device=dev)
        self.d_inst = torch.empty_like(self.p_inst, device=dev)
        self.db = DeviceBatch(
            batch=b, h_inst=h_inst, d_inst=self.d_inst, d_arrival=self.d_arrival, d_prompt=self.d_prompt,
            d_output=self.d_output,
            d_ft=torch.empty(n, dtype=torch.float64, device=dev), d_fin=torch.empty(n, dtype=torch.float64, device=dev),
            d_fd=torch.empty(n, dtype=torch.float64, device=dev), d_pc=torch.empty(n, dtype=torch.int32, device=dev),
            d_srv=torch.empty(n, dtype=torch.int32, device=dev),
            d_stats=torch.zeros(len(h_inst) * _abi.STATS.itemsize, dtype=torch.uint8, device=dev),
            d_scratch=torch.empty(max(self.scratch_bytes, 256), dtype=torch.uint8, device=dev),
            scratch_bytes=self.scratch_bytes)
        g = instance_groups(h_inst)
        self.h_groups = np.ascontiguousarray(g)
        self.d_groups = torch.from_numpy(self.h_groups.view(np.uint8)).to(dev)
        wb = int(self.lib.ssb_summary_work_bytes(self.h_groups.ctypes.data, len(g)))
        self.d_work = torch.empty(wb, dtype=torch.uint8, device=dev)
        self.work_bytes = wb
        self.d_summary = torch.empty(len(g) * _abi.SUMMARY.itemsize, dtype=torch.uint8, device=dev)
        self.p_stats = torch.empty(len(h_inst) * _abi.STATS.itemsize, dtype=torch.uint8).pin_memory()
        self.p_summary = torch.empty(len(g) * _abi.SUMMARY.itemsize, dtype=torch.uint8).pin_memory()
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in (self.p_arrival, self.p_prompt, self.p_output,
                                                                     self.p_inst))
        self.d2h_bytes = self.p_stats.numel() + self.p_summary.numel()
        self.n_singles = int((h_inst["n_servers"] == 1).sum())
        self.n_multis = len(h_inst) - self.n_singles
        self.sim_launches = (int(self.n_singles > 0) + int(self.n_multis > 0)
                             + int(bool((h_inst["qps_factor"] != 1.0).any())))  # + k_scale_arrivals
        self.copy_inputs()
        torch.cuda.synchronize()

    @property
    def launches_per_run(self) -> int:
        small = len(self.h_groups) > 0 and int(self.h_groups["n"].max()) <= SMALL_GROUP_MAX
        return self.sim_launches + (1 if small else SUMMARY_LAUNCHES)

    def copy_inputs(self):
        for d, h in ((self.d_arrival, self.p_arrival), (self.d_prompt, self.p_prompt), (self.d_output, self.p_output),
                     (self.d_inst, self.p_inst)):
            d.copy_(h, non_blocking=True)

    def simulate(self, stream=None):
        stream = stream or self.torch.cuda.current_stream()
        db = self.db
        rc = self.lib.ssb_simulate(self.h_inst.ctypes.data, db.d_inst.data_ptr(), len(self.h_inst), db.trace_c(),
                                   db.records_c(), db.d_stats.data_ptr(), db.d_scratch.data_ptr(), db.scratch_bytes,
                                   None, 0, None, ctypes.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise SimulationError(f"ssb_simulate: {self.lib.ssb_error_string(rc).decode()}")

    def summarize(self, stream=None):
        stream = stream or self.torch.cuda.current_stream()
        db = self.db
        rc = self.lib.ssb_summarize(db.trace_c(), db.records_c(), self.h_groups.ctypes.data, self.d_groups.data_ptr(),
                                    len(self.h_groups), self.d_summary.data_ptr(), self.d_work.data_ptr(),
                                    self.work_bytes, ctypes.c_void_p(stream.cuda_stream))
        if rc != 0:
            raise SimulationError(f"ssb_summarize: {self.lib.ssb_error_string(rc).decode()}")

    def read_results(self):
        self.p_stats.copy_(self.db.d_stats, non_blocking=True)
        self.p_summary.copy_(self.d_summary, non_blocking=True)

    def run(self, *, copy_inputs: bool = True, read_results: bool = True):
        if copy_inputs:
            self.copy_inputs()
        self.simulate()
        self.summarize()
        if read_results:
            self.read_results()

    def results(self):
        """(stats, summaries) as numpy after synchronising."""
        self.torch.cuda.synchronize()
        return (self.p_stats.numpy().view(_abi.STATS).copy(), self.p_summary.numpy().view(_abi.SUMMARY).copy())

    def adopt_measured_schedule(self, stats) -> None:
        """Use the measured cost of each instance (simulate.measured_cost: iterations x its
        policy's mean device cycles per iteration) as its scheduling hint for later runs of
        this sweep: per-policy SM shares, the SMs reserved for the longest instances, and
        longest-first queue order. Work is unchanged; only the placement adapts."""
        from .simulate import measured_cost

        c = measured_cost(self.h_inst, stats)
        if c is not None:
            self.h_inst["est_cost"] = c

    def fix_overflows(self) -> int:
        """Re-run instances whose shared running table overflowed (then re-summarize)."""
        n = retry_overflows(self.db)
        if n:
            self.p_inst.copy_(self.torch.from_numpy(self.db.h_inst.view(np.uint8)))
            self.h_inst = self.db.h_inst
            self.summarize()
            self.read_results()
            self.torch.cuda.synchronize()
        return n
