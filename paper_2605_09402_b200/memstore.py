"""Hot-slot budget and policy names (oocgnn/memstore.py:276-330).

The memory manager itself is the device engine (csrc/engine.cu): pending
counters, lifecycle states, the hot set and the min-pending / LRU / random
victim selection all live in HBM and are replayed bit-exactly. This module
keeps the host-side pieces of the reference's interface: the budget
arithmetic and the policy registry.
"""

from dataclasses import dataclass

from .errors import ConfigError

POLICIES = ("minpend", "lru", "rnd")


def make_policy(name: str, max_pending: int = 0, seed: int = 0) -> str:
    """Validates a policy name (oocgnn/memstore.py:276-283); the policy
    state machine runs on the device."""
    if name not in POLICIES:
        raise ConfigError(f"unknown eviction policy {name!r}")
    return name


@dataclass
class MemoryBudget:
    slot_count: int
    slot_dim: int

    @property
    def slot_bytes(self) -> int:
        return self.slot_dim * 4

    @classmethod
    def from_bytes(cls, budget_bytes: int, slot_dim: int) -> "MemoryBudget":
        slots = budget_bytes // (slot_dim * 4)
        if slots < 1:
            raise ConfigError(
                f"budget {budget_bytes} B holds no {slot_dim}-wide slot")
        return cls(slots, slot_dim)


def default_evict_batch(slot_count: int) -> int:
    return max(1, slot_count // 100)


class MemoryFacade:
    """What ``ctx.memory`` exposes in the reference: slot_count, the
    evict batch and close()."""

    def __init__(self, budget: MemoryBudget, evict_batch, layer):
        self.slot_count = budget.slot_count
        self.slot_dim = budget.slot_dim
        self.evict_batch = evict_batch or default_evict_batch(budget.slot_count)
        self._layer = layer

    @property
    def unique_reloaded(self):
        raise AttributeError("unique reloads are reported by finalize_layer")

    def hot_population(self) -> int:
        _, st, _, _ = self._layer.state_arrays()
        return int((st == 1).sum())

    def close(self, delete_cold: bool = True) -> None:
        self._layer.close()
