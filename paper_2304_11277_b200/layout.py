"""FlatParameter geometry — host side, integer only.

Mirrors the reference's `flatparam.py` interface (names, argument meaning,
error classes and messages) so code written against shardsim's layout API
runs unchanged:

* `build_unit_layouts(param_shapes, unit_param_names, F)` — flatparam.py:63-96:
  every parameter in exactly one unit (SharedParameterError naming the
  SHARD_GRAD_OP / NRAF workaround, FlatParamError for unknown or uncovered
  names), offsets = cumulative numel in declaration order, psi = ceil(raw/F)*F,
  padding = psi - raw <= F-1, shard_numel = psi/F (rank r owns chunk r % F).
* `dump_plan_lines` — flatparam.py:238-247 golden line format.
* `peak_param_memory` — flatparam.py:198-235 closed forms.

The device-side counterparts (flatten / unflatten / shard copy of these
layouts) are CUDA kernels behind the C ABI (include/fsdp_b200.h).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import Iterable, Sequence


class FlatParamError(ValueError):
    pass


class SharedParameterError(FlatParamError):
    """A parameter assigned to two units — rejected, with the workaround named."""


@dataclass(frozen=True)
class OriginalParam:
    name: str
    shape: tuple
    offset: int

    @property
    def numel(self) -> int:
        return math.prod(self.shape)


@dataclass(frozen=True)
class UnitLayout:
    """Rank-independent geometry of one FlatParameter."""

    unit_id: int
    originals: tuple
    psi: int
    padding: int
    shard_factor: int

    @property
    def raw_numel(self) -> int:
        return self.psi - self.padding

    @property
    def shard_numel(self) -> int:
        return self.psi // self.shard_factor

    def shard_range(self, shard_index: int) -> tuple[int, int]:
        b = self.shard_numel
        return shard_index * b, (shard_index + 1) * b

    @property
    def offsets(self) -> list[int]:
        return [o.offset for o in self.originals]

    @property
    def numels(self) -> list[int]:
        return [o.numel for o in self.originals]


def _owner_map(unit_param_names: Sequence[Sequence[str]], known: dict) -> dict:
    owner: dict[str, int] = {}
    for uid, names in enumerate(unit_param_names):
        for name in names:
            prev = owner.get(name)
            if prev is not None:
                raise SharedParameterError(
                    f"parameter '{name}' is assigned to units {prev} and {uid}; sharing a "
                    f"parameter across units is unsupported — merge the sharing layers into "
                    f"one unit, or keep parameters materialized through backward with "
                    f"grad-op sharding (reshard_after_forward=NRAF, ShardingStrategy."
                    f"SHARD_GRAD_OP)")
            if name not in known:
                raise FlatParamError(f"unknown parameter '{name}'")
            owner[name] = uid
    uncovered = [n for n in known if n not in owner]
    if uncovered:
        raise FlatParamError(f"unit boundaries do not cover parameters: {uncovered}")
    return owner


def build_unit_layouts(param_shapes: Iterable[tuple[str, tuple]],
                       unit_param_names: Sequence[Sequence[str]],
                       shard_factor: int) -> list[UnitLayout]:
    """Assign every parameter to exactly one unit and lay out flat buffers."""
    if shard_factor < 1:
        raise FlatParamError(f"shard_factor must be >= 1, got {shard_factor}")
    shapes = {name: tuple(shape) for name, shape in param_shapes}
    _owner_map(unit_param_names, shapes)
    layouts = []
    for uid, names in enumerate(unit_param_names):
        cursor = 0
        originals = []
        for name in names:
            originals.append(OriginalParam(name, shapes[name], cursor))
            cursor += math.prod(shapes[name])
        psi = ((cursor + shard_factor - 1) // shard_factor) * shard_factor
        layouts.append(UnitLayout(uid, tuple(originals), psi, psi - cursor, shard_factor))
    return layouts


def dump_plan_lines(layouts: Sequence[UnitLayout]) -> list[str]:
    """`unit=<id> ψ=<n> padding=<k> originals=[name:AxB ...]` per unit."""
    out = []
    for lay in layouts:
        shapes = " ".join(f"{o.name}:{'x'.join(map(str, o.shape))}" for o in lay.originals)
        out.append(f"unit={lay.unit_id} ψ={lay.psi} padding={lay.padding} originals=[{shapes}]")
    return out


def peak_param_memory(psis: Sequence[int], shard_factor: int, k_full: int = 4,
                      k_low: int | None = None, variant: str = "serialized") -> dict:
    """Predicted peak parameter memory (flatparam.py:198-235); the B200 build's
    widths are k_full = 4 (fp32 master) and k_low = 2 (bf16 gathered)."""
    if not psis:
        return {"elements": Fraction(0), "bytes": Fraction(0)}
    if variant not in ("serialized", "two_inflight"):
        raise FlatParamError(f"unknown variant '{variant}'")
    total = sum(psis)
    if shard_factor == 1:
        return {"elements": Fraction(total), "bytes": Fraction(total * k_full)}
    largest = sorted(psis, reverse=True)[: 1 if variant == "serialized" else 2]
    shards = Fraction(total, shard_factor)
    elements = shards + sum(largest)
    if k_low is None:
        nbytes = elements * k_full
    else:
        nbytes = shards * k_full + sum(largest) * k_low
    return {"elements": elements, "bytes": nbytes}
