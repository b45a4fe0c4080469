"""Sharding plan: world W, sharding factor F, host size G.

Mirrors `collectives.py:37-106` (ShardingPlan / build_plan): sharded groups
are W/F consecutive blocks of F ranks, replicated groups are F strided groups
{j, j+F, ...}.  Strategy: F == 1 replicate (NO_SHARD), F == W full
(FULL_SHARD / SHARD_GRAD_OP), otherwise hybrid (HYBRID_SHARD).

On the device a group is the (size, stride) pair the C ABI takes: sharded
group = (F, 1), replicated group = (W/F, F), world = (W, 1).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence


class CollectiveError(ValueError):
    """Contract violation at a collective call site (uneven input, bad group...)."""


class DeadlockError(RuntimeError):
    """A cross-GPU wait timed out: some member never entered the collective."""


@dataclass(frozen=True)
class ShardingPlan:
    world_size: int
    shard_factor: int
    host_size: int

    def __post_init__(self) -> None:
        w, f, g = self.world_size, self.shard_factor, self.host_size
        if w < 1:
            raise CollectiveError(f"world_size must be >= 1, got {w}")
        if not 1 <= f <= w or w % f != 0:
            raise CollectiveError(f"shard_factor {f} must divide world_size {w} (1 <= F <= W)")
        if not 1 <= g <= w or w % g != 0:
            raise CollectiveError(f"host_size {g} must divide world_size {w}")

    @property
    def sharded_groups(self) -> list[tuple[int, ...]]:
        f = self.shard_factor
        return [tuple(range(b, b + f)) for b in range(0, self.world_size, f)]

    @property
    def replicated_groups(self) -> list[tuple[int, ...]]:
        f = self.shard_factor
        return [tuple(range(j, self.world_size, f)) for j in range(f)]

    @property
    def replica_count(self) -> int:
        return self.world_size // self.shard_factor

    @property
    def num_hosts(self) -> int:
        return self.world_size // self.host_size

    @property
    def strategy(self) -> str:
        if self.shard_factor == 1:
            return "replicate"
        return "full" if self.shard_factor == self.world_size else "hybrid"

    def host_of(self, rank: int) -> int:
        return rank // self.host_size

    def sharded_group_of(self, rank: int) -> tuple[int, ...]:
        base = rank - rank % self.shard_factor
        return tuple(range(base, base + self.shard_factor))

    def replicated_group_of(self, rank: int) -> tuple[int, ...]:
        return tuple(range(rank % self.shard_factor, self.world_size, self.shard_factor))

    def shard_index(self, rank: int) -> int:
        return rank % self.shard_factor

    def spans_hosts(self, group: Sequence[int]) -> bool:
        return len({self.host_of(r) for r in group}) > 1

    # device-side group descriptors (size, stride)
    @property
    def sharded_desc(self) -> tuple[int, int]:
        return self.shard_factor, 1

    @property
    def replicated_desc(self) -> tuple[int, int]:
        return self.replica_count, self.shard_factor

    @property
    def world_desc(self) -> tuple[int, int]:
        return self.world_size, 1


def build_plan(world_size: int, shard_factor: int, host_size: int | None = None) -> ShardingPlan:
    """Validate and build a ShardingPlan; host_size defaults to one host."""
    return ShardingPlan(world_size, shard_factor, world_size if host_size is None else host_size)


def group_desc_of(group: Sequence[int], world_size: int) -> tuple[int, int]:
    """(size, stride) of a sorted rank group the device can address, or raise."""
    g = tuple(sorted(group))
    n = len(g)
    if n == 0:
        raise CollectiveError("empty group")
    stride = 1 if n == 1 else g[1] - g[0]
    if any(b - a != stride for a, b in zip(g, g[1:])) or stride < 1:
        raise CollectiveError(f"group {g} is not an arithmetic progression")
    if stride == 1:
        if world_size % n or g[0] % n:
            raise CollectiveError(f"group {g} is not a consecutive block of size {n}")
    else:
        if g[0] >= stride or n * stride != world_size:
            raise CollectiveError(f"group {g} is not a replicated group of stride {stride}")
    return n, stride
