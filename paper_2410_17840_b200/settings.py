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
    """Cost parameters for a (profile, hardware) pair (costmodel.py:78-94)."""
    key = (profile_name, hardware)
    if key in _COST_DEFAULTS:
        base = _COST_DEFAULTS[key]
        return replace(base, **overrides) if overrides else base
    required = {"mem_base_s", "mem_per_kv_token_s", "compute_per_token_s", "overhead_s"}
    if set(overrides) == required:
        return CostParams(**overrides)
    raise KeyError(
        f"no default cost parameters for {profile_name!r} on {hardware!r}; known pairs: {sorted(_COST_DEFAULTS)}"
    )


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
    """Host-side KV block accounting object (kvmem.py:74-154), kept for API parity
    (Engine(pool, ...) construction, unit checks). The simulation itself keeps
    the pool on the device as a free-block counter plus per-request
    prompt+generated token counts (csrc/ssb_engine.cuh)."""

    def __init__(self, total_blocks: int, block_size: int = DEFAULT_BLOCK_SIZE):
        if total_blocks < 0:
            raise ValueError(f"total_blocks must be >= 0, got {total_blocks}")
        if block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {block_size}")
        self.total_blocks = total_blocks
        self.block_size = block_size
        self.free_blocks = total_blocks
        self._tokens: dict[int, int] = {}

    def allocated_tokens(self, request_id: int) -> int:
        return self._tokens[request_id]

    def allocated_blocks(self, request_id: int) -> int:
        return blocks_needed(self._tokens[request_id], self.block_size)

    def try_allocate(self, request_id: int, tokens: int) -> bool:
        if request_id in self._tokens:
            raise ValueError(f"request {request_id} already holds an allocation")
        need = blocks_needed(tokens, self.block_size)
        if need > self.free_blocks:
            return False
        self._tokens[request_id] = tokens
        self.free_blocks -= need
        return True

    def try_grow(self, request_id: int, new_total_tokens: int) -> bool:
        if request_id not in self._tokens:
            raise KeyError(f"request {request_id} holds no allocation")
        current = self._tokens[request_id]
        if new_total_tokens < current:
            raise ValueError(f"allocation for request {request_id} cannot shrink")
        extra = blocks_needed(new_total_tokens, self.block_size) - blocks_needed(current, self.block_size)
        if extra > self.free_blocks:
            return False
        self._tokens[request_id] = new_total_tokens
        self.free_blocks -= extra
        return True

    def free(self, request_id: int) -> int:
        if request_id not in self._tokens:
            raise KeyError(f"request {request_id} holds no allocation")
        released = self.allocated_blocks(request_id)
        del self._tokens[request_id]
        self.free_blocks += released
        return released

    def conserved(self) -> bool:
        held = sum(blocks_needed(t, self.block_size) for t in self._tokens.values())
        return self.free_blocks + held == self.total_blocks and self.free_blocks >= 0
