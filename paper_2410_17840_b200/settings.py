"""Engine / balancer / cluster settings and the static model tables.

Host-side mirror of the reference's configuration surface, so that a caller
of the reference's simulation path constructs exactly the same objects:

* ``EngineSettings`` / ``BalancerSettings`` / ``ClusterSettings``
  — config.py:26-56 (same field names, defaults and meaning)
* ``ModelProfile`` / ``PROFILES`` / ``pool_blocks_for`` / ``blocks_needed``
  — kvmem.py:15-71
* ``CostParams`` / ``default_params`` — costmodel.py:22-94

These are plain host data; nothing here simulates. The simulation itself is
the CUDA path in ``simulate.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

DEFAULT_BLOCK_SIZE = 16  # kvmem.py:12


def blocks_needed(tokens: int, block_size: int) -> int:
    """ceil(tokens / block_size) (kvmem.py:15-21)."""
    if tokens < 0:
        raise ValueError(f"token count must be >= 0, got {tokens}")
    if block_size < 1:
        raise ValueError(f"block_size must be >= 1, got {block_size}")
    return -(-tokens // block_size)


@dataclass(frozen=True)
class ModelProfile:
    """Per-model constants for KV sizing (kvmem.py:24-31)."""

    name: str
    kv_bytes_per_token: int
    max_context: int
    weights_bytes: int


# kv bytes/token = layers * kv_heads * head_dim * 2 (K,V) * 2 (fp16) (kvmem.py:34-48)
PROFILES = {
    "llama3-8b": ModelProfile("llama3-8b", 32 * 8 * 128 * 2 * 2, 8192, 16_000_000_000),
    "llama3-70b": ModelProfile("llama3-70b", 80 * 8 * 128 * 2 * 2, 8192, 70_000_000_000),
}


def pool_blocks_for(gpu_mem_bytes: float, profile: ModelProfile, block_size: int = DEFAULT_BLOCK_SIZE) -> int:
    """KV pool capacity in blocks left after the weights (kvmem.py:58-71)."""
    spare = gpu_mem_bytes - profile.weights_bytes
    if spare <= 0:
        raise ValueError(
            f"{profile.name} weights ({profile.weights_bytes} B) do not fit in {gpu_mem_bytes} B of device memory"
        )
    return int(spare // (profile.kv_bytes_per_token * block_size))


@dataclass(frozen=True)
class CostParams:
    """latency = overhead + max(mem_base + mem_per_kv*resident, compute*tokens) (costmodel.py:22-47)."""

    mem_base_s: float
    mem_per_kv_token_s: float
    compute_per_token_s: float
    overhead_s: float

    def __post_init__(self):
        if self.mem_base_s <= 0:
            raise ValueError(f"mem_base_s must be > 0, got {self.mem_base_s}")
        for name in ("mem_per_kv_token_s", "compute_per_token_s", "overhead_s"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0, got {getattr(self, name)}")


_COST_DEFAULTS = {  # costmodel.py:62-75
    ("llama3-8b", "a100"): CostParams(1.03e-2, 8.4e-8, 1.0e-4, 5e-4),
    ("llama3-70b", "h100x2"): CostParams(1.05e-2, 4.9e-8, 1.4e-4, 5e-4),
}


def default_params(profile_name: str, hardware: str, **overrides: float) -> CostParams:
    """Cost parameters for a (profile, hardware) pair (costmodel.py:78-94): the known
    pairs' defaults with per-field overrides; an unknown pair needs all four fields."""
    fields_ = ("mem_base_s", "mem_per_kv_token_s", "compute_per_token_s", "overhead_s")
    base = _COST_DEFAULTS.get((profile_name, hardware))
    if base is None and set(overrides) != set(fields_):
        raise KeyError(
            f"no default cost parameters for {profile_name!r} on {hardware!r}; known pairs: {sorted(_COST_DEFAULTS)}"
        )
    if base is None or overrides:
        vals = {f: overrides.get(f, getattr(base, f) if base is not None else None) for f in fields_}
        unknown = set(overrides) - set(fields_)
        if unknown:
            raise TypeError(f"unknown cost parameter(s): {sorted(unknown)}")
        return CostParams(**vals)
    return base


@dataclass
class EngineSettings:
    """config.py:26-39."""

    policy: str = "fcfs"
    alpha: float = 1.0
    c: float = 0.0
    max_output: int = 8191
    profile: str = "llama3-8b"
    hardware: str = "a100"
    block_size: int = DEFAULT_BLOCK_SIZE
    pool_blocks: int | None = None
    gpu_mem_bytes: float = 40e9
    max_tokens_per_batch: int = 1024
    max_running: int | None = None
    cost: dict = field(default_factory=dict)


@dataclass
class BalancerSettings:
    """config.py:42-47."""

    name: str = "random"
    poll_interval_s: float = 0.1
    beta_prior: float = 2.0
    beta_fixed: float | None = None


@dataclass
class ClusterSettings:
    """config.py:50-55."""

    n_servers: int = 1
    engine: EngineSettings = field(default_factory=EngineSettings)
    balancer: BalancerSettings = field(default_factory=BalancerSettings)
    seed: int = 0


class KvBlockPool:
    """Pool descriptor for ``Engine(KvBlockPool(total_blocks, block_size), ...)``
    construction (kvmem.py:74-104 constructor and validation). The block
    accounting itself (try_allocate / try_grow / free, kvmem.py:106-154) runs on
    the device as one free-block counter per engine plus each running request's
    prompt+generated token count (csrc/ssb_engine.cuh); there is no host copy."""

    def __init__(self, total_blocks: int, block_size: int = DEFAULT_BLOCK_SIZE):
        if total_blocks < 0:
            raise ValueError(f"total_blocks must be >= 0, got {total_blocks}")
        if block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {block_size}")
        self.total_blocks = int(total_blocks)
        self.block_size = int(block_size)
        self.free_blocks = self.total_blocks  # a fresh pool; engines are run once (engine.py:238-239)

    def __repr__(self) -> str:
        return f"KvBlockPool(total_blocks={self.total_blocks}, block_size={self.block_size})"
