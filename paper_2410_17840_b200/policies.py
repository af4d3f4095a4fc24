"""Scheduler-policy registry (drop-in for policies.py).

The reference's plugin surface is the registry: ``make_policy(name, alpha=,
c=, max_output=)`` over ``POLICY_NAMES`` (policies.py:279-298), plus
``check_feasible`` (policies.py:56-68, 119-131). Here each policy object is a
*descriptor* that is compiled into the device instance table; ``select`` runs
only inside the sm_100a engine-step kernel (csrc/ssb_kernels.cu). A Python
subclass that overrides ``select`` cannot be executed on the device and is
rejected with NotImplementedError (no CPU fallback).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .settings import blocks_needed


class InfeasibleRequestError(ValueError):
    """A request that can never run under the given engine configuration (policies.py:18-19)."""


@dataclass(frozen=True)
class EngineLimits:
    """policies.py:22-36."""

    max_tokens_per_batch: int
    max_running: int | None
    max_context: int

    def __post_init__(self):
        if self.max_tokens_per_batch < 1:
            raise ValueError(f"max_tokens_per_batch must be >= 1, got {self.max_tokens_per_batch}")
        if self.max_running is not None and self.max_running < 1:
            raise ValueError(f"max_running must be >= 1, got {self.max_running}")
        if self.max_context < 1:
            raise ValueError(f"max_context must be >= 1, got {self.max_context}")


class SchedulerPolicy:
    """Base descriptor. ``policy_id`` selects the device implementation."""

    name = "base"
    policy_id = -1

    def select(self, waiting, running, pool, clock, limits):
        raise NotImplementedError(
            "policy decisions run inside the sm_100a engine-step kernel; "
            "custom Python policies are not supported by the B200 simulator"
        )

    # -- feasibility (vectorised restatement of policies.py:56-68) ----------
    def _infeasible_mask(self, prompt, output, block_size, pool_blocks, limits):
        peak = prompt.astype(np.int64) + output
        bad_ctx = peak > limits.max_context
        bad_pool = (-(-peak // block_size)) > pool_blocks
        return bad_ctx, bad_pool

    def feasible_by_max(self, maxes, block_size, pool_blocks, limits) -> bool:
        """Every request is feasible, decided from the trace's maxima alone (max prompt +
        output, max prompt, max output): each check of policies.py:56-68,119-131 is monotone
        in the request's lengths, so the largest one passing means all pass. False = run the
        per-request check (which names the first failing request)."""
        peak, _, _ = maxes
        return peak <= limits.max_context and -(-peak // block_size) <= pool_blocks

    def check_feasible_many(self, prompt, output, block_size, pool_blocks, limits, maxes=None) -> None:
        """Raise InfeasibleRequestError for the first infeasible request (request-id order).
        maxes: (max prompt+output, max prompt, max output) of the trace, when known."""
        if maxes is not None and self.feasible_by_max(maxes, block_size, pool_blocks, limits):
            return
        masks = self._infeasible_mask(np.asarray(prompt), np.asarray(output), block_size, pool_blocks, limits)
        any_bad = np.zeros(len(prompt), dtype=bool)
        for m in masks:
            any_bad |= m
        if not any_bad.any():
            return
        i = int(np.flatnonzero(any_bad)[0])
        self.check_feasible_one(i, int(prompt[i]), int(output[i]), block_size, pool_blocks, limits)
        raise AssertionError("vectorised feasibility disagrees with the scalar check")  # pragma: no cover

    def check_feasible_one(self, rid, prompt, output, block_size, pool_blocks, limits) -> None:
        peak = prompt + output
        if peak > limits.max_context:
            raise InfeasibleRequestError(
                f"request {rid}: prompt {prompt} + output {output} exceeds the {limits.max_context}-token context window"
            )
        if blocks_needed(peak, block_size) > pool_blocks:
            raise InfeasibleRequestError(
                f"request {rid}: needs {blocks_needed(peak, block_size)} blocks at peak, pool holds {pool_blocks}"
            )

    def params(self) -> dict:
        return {}


class FcfsPolicy(SchedulerPolicy):
    """Strict FCFS with head-of-line blocking (policies.py:76-97)."""

    name = "fcfs"
    policy_id = 0


class NoPreemptPolicy(SchedulerPolicy):
    """FIFO admission with worst-case reservations (policies.py:100-146)."""

    name = "nopreempt"
    policy_id = 1

    def __init__(self, max_output: int = 1024):
        if max_output < 1:
            raise ValueError(f"max_output must be >= 1, got {max_output}")
        self.max_output = max_output

    def reservation_tokens(self, prompt: int, limits: EngineLimits) -> int:
        return min(limits.max_context, prompt + self.max_output)

    def _infeasible_mask(self, prompt, output, block_size, pool_blocks, limits):
        a, b = super()._infeasible_mask(prompt, output, block_size, pool_blocks, limits)
        res = np.minimum(limits.max_context, prompt.astype(np.int64) + self.max_output)
        return a, b, output > self.max_output, (-(-res // block_size)) > pool_blocks

    def feasible_by_max(self, maxes, block_size, pool_blocks, limits) -> bool:
        _, pmax, omax = maxes
        res = min(limits.max_context, pmax + self.max_output)
        return (super().feasible_by_max(maxes, block_size, pool_blocks, limits) and omax <= self.max_output
                and -(-res // block_size) <= pool_blocks)

    def check_feasible_one(self, rid, prompt, output, block_size, pool_blocks, limits) -> None:
        super().check_feasible_one(rid, prompt, output, block_size, pool_blocks, limits)
        if output > self.max_output:
            raise InfeasibleRequestError(
                f"request {rid}: output {output} exceeds the promised max_output {self.max_output}"
            )
        reservation = blocks_needed(self.reservation_tokens(prompt, limits), block_size)
        if reservation > pool_blocks:
            raise InfeasibleRequestError(
                f"request {rid}: reservation of {reservation} blocks exceeds the pool ({pool_blocks})"
            )

    def params(self) -> dict:
        return {"max_output": self.max_output}


class ShortestRemainingPolicy(SchedulerPolicy):
    """TRAIL+: shortest remaining output first, greedy skip, optional preemption (policies.py:149-212)."""

    name = "trail_plus"
    policy_id = 2

    def __init__(self, c: float = 0.0):
        if not 0.0 <= c <= 1.0:
            raise ValueError(f"c must be in [0, 1], got {c}")
        self.c = c

    def params(self) -> dict:
        return {"c": self.c}


def larry_score(request, clock: float, queue_len: int, alpha: float) -> float:
    """Eq. 1 (policies.py:215-224): alpha*(clock-enqueue_time) - queue_len*pending_prefill.

    Host formula for documentation/KATs; the device evaluates the same
    expression with the same binary64 rounding (no FMA)."""
    wait = clock - request.enqueue_time
    return alpha * wait - queue_len * request.pending_prefill


class LoadAdaptivePolicy(SchedulerPolicy):
    """LARRY: score-ordered admission under the iteration token budget (policies.py:227-276)."""

    name = "larry"
    policy_id = 3

    def __init__(self, alpha: float = 1.0):
        if alpha < 0:
            raise ValueError(f"alpha must be >= 0, got {alpha}")
        self.alpha = alpha

    def params(self) -> dict:
        return {"alpha": self.alpha}


POLICY_NAMES = ("fcfs", "nopreempt", "trail_plus", "larry")
_POLICY_CLASSES = (FcfsPolicy, NoPreemptPolicy, ShortestRemainingPolicy, LoadAdaptivePolicy)


def make_policy(name: str, *, alpha: float = 1.0, c: float = 0.0, max_output: int = 1024) -> SchedulerPolicy:
    """Registry (policies.py:282-298)."""
    if name == "fcfs":
        return FcfsPolicy()
    if name == "nopreempt":
        return NoPreemptPolicy(max_output=max_output)
    if name == "trail_plus":
        return ShortestRemainingPolicy(c=c)
    if name == "larry":
        return LoadAdaptivePolicy(alpha=alpha)
    raise ValueError(f"unknown policy {name!r}; expected one of {POLICY_NAMES}")


def policy_descriptor(policy: SchedulerPolicy) -> tuple[int, float, float, int]:
    """(policy_id, alpha, c, max_output) for the device; rejects custom subclasses."""
    if type(policy) not in _POLICY_CLASSES:
        raise NotImplementedError(
            f"{type(policy).__name__}: only the registry policies {POLICY_NAMES} run on the B200 simulator"
        )
    alpha = float(getattr(policy, "alpha", 1.0))
    c = float(getattr(policy, "c", 0.0))
    max_output = int(getattr(policy, "max_output", 1024))
    return policy.policy_id, alpha, c, max_output
