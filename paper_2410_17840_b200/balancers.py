"""Load-balancer registry (drop-in for balancers.py).

The reference routes each arrival with ``LoadBalancer.route(prompt)`` over a
stale ``BalancerView`` (balancers.py:29-64) and feeds completions back with
``on_finish`` (balancers.py:128-129, 214-216). On the B200 path routing runs
inside the cluster kernel (csrc/ssb_kernels.cu): rr, random and p2c draw
from a device restatement of numpy's PCG64 ``Generator.integers`` seeded with
``np.random.PCG64(seed).state``; sal evaluates Eq. 2 (``sal_load``) for every
replica with a warp argmin. The classes here are descriptors plus the small
pure functions (``sal_load``, ``BetaEstimator``) whose host restatements the
tests use as known-answer checks.
"""

from __future__ import annotations

from dataclasses import dataclass

import functools

import numpy as np


@dataclass
class ServerStats:
    """balancers.py:20-26."""

    queued_tokens: int
    free_mem_tokens: int
    in_flight: int


class BetaEstimator:
    """(mean_in + mean_out) / mean_out over finished requests (balancers.py:67-100)."""

    def __init__(self, prior: float = 2.0):
        if prior < 1:
            raise ValueError(f"prior must be >= 1, got {prior}")
        self.prior = prior
        self.count = 0
        self._sum_in = 0
        self._sum_out = 0

    def update(self, prompt_tokens: int, output_tokens: int) -> None:
        if prompt_tokens < 1 or output_tokens < 1:
            raise ValueError("token counts must be >= 1")
        self.count += 1
        self._sum_in += prompt_tokens
        self._sum_out += output_tokens

    @property
    def beta(self) -> float:
        if self.count == 0:
            return self.prior
        return (self._sum_in + self._sum_out) / self._sum_out


def sal_load(stats: ServerStats, prompt_tokens: int, beta: float, max_tokens_per_batch: int) -> float:
    """Eq. 2 (balancers.py:103-112)."""
    memory_term = beta * (prompt_tokens - stats.free_mem_tokens)
    queue_term = (stats.queued_tokens + prompt_tokens) / max_tokens_per_batch
    return max(memory_term, queue_term)


class LoadBalancer:
    name = "base"
    balancer_id = -1

    def __init__(self, n_servers: int):
        if n_servers < 1:
            raise ValueError(f"n_servers must be >= 1, got {n_servers}")
        self.n_servers = n_servers

    def route(self, prompt_tokens: int) -> int:
        raise NotImplementedError(
            "routing runs inside the sm_100a cluster kernel; custom Python balancers are not supported"
        )


class RoundRobinBalancer(LoadBalancer):
    name = "rr"
    balancer_id = 0


class RandomBalancer(LoadBalancer):
    name = "random"
    balancer_id = 1


class PowerOfTwoBalancer(LoadBalancer):
    name = "p2c"
    balancer_id = 2


class ServerAwareBalancer(LoadBalancer):
    name = "sal"
    balancer_id = 3

    def __init__(self, n_servers: int, max_tokens_per_batch: int = 1024, beta_prior: float = 2.0,
                 beta_fixed: float | None = None):
        super().__init__(n_servers)
        BetaEstimator(prior=beta_prior)  # same validation
        self.max_tokens_per_batch = max_tokens_per_batch
        self.beta_prior = beta_prior
        self.beta_fixed = beta_fixed


BALANCER_NAMES = ("rr", "random", "p2c", "sal")


def make_balancer(name: str, n_servers: int, *, max_tokens_per_batch: int = 1024, beta_prior: float = 2.0,
                  beta_fixed: float | None = None) -> LoadBalancer:
    """Registry (balancers.py:222-253); the rng/view wiring lives on the device."""
    if name == "rr":
        return RoundRobinBalancer(n_servers)
    if name == "random":
        return RandomBalancer(n_servers)
    if name == "p2c":
        return PowerOfTwoBalancer(n_servers)
    if name == "sal":
        return ServerAwareBalancer(n_servers, max_tokens_per_batch, beta_prior, beta_fixed)
    raise ValueError(f"unknown balancer {name!r}; expected one of {BALANCER_NAMES}")


def pcg64_words(seed) -> tuple[int, int, int, int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of np.random.default_rng(seed) (cluster.py:94)."""
    if isinstance(seed, int) and seed >= 0:
        return _pcg64_words_int(seed)
    return _pcg64_words(seed)


@functools.lru_cache(maxsize=4096)
def _pcg64_words_int(seed: int) -> tuple[int, int, int, int]:
    return _pcg64_words(seed)


def _pcg64_words(seed) -> tuple[int, int, int, int]:
    st = np.random.PCG64(seed).state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m
