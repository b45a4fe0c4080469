"""The reference's model zoo and data semantics, so a Session on B200 sees
bit-identical inputs and initial parameters to a shardsim Session.

* `named_stream(seed, name)` — numerics.py:73-78 (sha256-keyed SeedSequence)
* `batch_stream(...)`        — numerics.py:303-321 ("integer" / "uniform")
* `ModelSpec`                — numerics.py:81-127 (Linear + ReLU/Tanh units)
* `init_values(spec, seed)`  — deferred_init.py:63-143 replay of the
                               dyadic / scaled_uniform / normal / zeros styles
Host-side numpy only (float64, cast to fp32 when loaded on device).
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np


class NumericsError(ValueError):
    pass


def named_stream(seed: int, name: str) -> np.random.Generator:
    key = int.from_bytes(hashlib.sha256(name.encode("utf-8")).digest()[:8], "big")
    return np.random.default_rng(np.random.SeedSequence([seed, key]))


def batch_stream(seed: int, steps: int, batch: int, dim_in: int, dim_out: int,
                 regime: str = "integer"):
    rng = named_stream(seed, "data")
    for _ in range(steps):
        if regime == "integer":
            x = rng.integers(-3, 4, size=(batch, dim_in)).astype(np.float64)
            y = rng.integers(-3, 4, size=(batch, dim_out)).astype(np.float64)
        elif regime == "uniform":
            x = rng.uniform(-1.0, 1.0, size=(batch, dim_in))
            y = rng.uniform(-1.0, 1.0, size=(batch, dim_out))
        else:
            raise NumericsError(f"unknown data regime '{regime}'")
        yield x, y


@dataclass(frozen=True)
class ModelSpec:
    dims: tuple = (4, 8, 8, 2)
    activation: str = "relu"
    unit_sizes: tuple | None = None
    init: str = "dyadic"
    bias: bool = True

    @property
    def num_linears(self) -> int:
        return len(self.dims) - 1

    @property
    def units(self) -> list[list[int]]:
        sizes = self.unit_sizes or tuple(1 for _ in range(self.num_linears))
        if sum(sizes) != self.num_linears:
            raise NumericsError(f"unit_sizes {sizes} must cover {self.num_linears} linears")
        out, nxt = [], 0
        for s in sizes:
            out.append(list(range(nxt, nxt + s)))
            nxt += s
        return out

    def param_shapes(self) -> list[tuple[str, tuple]]:
        shapes = []
        for i in range(self.num_linears):
            shapes.append((f"linear{i}.weight", (self.dims[i + 1], self.dims[i])))
            if self.bias:
                shapes.append((f"linear{i}.bias", (self.dims[i + 1],)))
        return shapes

    def unit_param_names(self) -> list[list[str]]:
        per: dict[int, list[str]] = {}
        for name, _ in self.param_shapes():
            per.setdefault(int(name.split(".")[0][len("linear"):]), []).append(name)
        return [[n for li in unit for n in per[li]] for unit in self.units]


_SHIFT = 3.0 * 2.0 ** 51   # deferred_init.py:26-27 round-to-integer trick


def init_values(spec: ModelSpec, seed: int) -> dict[str, np.ndarray]:
    return init_values_for(spec, seed, None)


def init_values_for(spec: ModelSpec, seed: int, names) -> dict[str, np.ndarray]:
    """Replay of the named parameters only (all when `names` is None): the
    PRNG stream of each parameter is keyed by (seed, name), so a subset
    replays to the same values as the whole model (deferred_init.py:63-143)."""
    out = {}
    keep = None if names is None else set(names)
    for name, shape in spec.param_shapes():
        if keep is not None and name not in keep:
            continue
        n = math.prod(shape)
        fan_in = shape[-1] if len(shape) > 1 else shape[0]
        rng = named_stream(seed, name)
        if spec.init == "zeros":
            v = np.zeros(n)
        elif spec.init == "dyadic":
            v = rng.uniform(0.0, 1.0, size=n)
            v *= 8.0
            v += _SHIFT
            v += -_SHIFT
            v *= 0.125
            v += -0.5
        elif spec.init == "scaled_uniform":
            v = rng.uniform(-1.0, 1.0, size=n)
            v *= 1.0 / math.sqrt(max(fan_in, 1))
        elif spec.init == "normal":
            v = rng.normal(0.0, 1.0, size=n)
            v *= 1.0 / math.sqrt(max(fan_in, 1))
        else:
            raise NumericsError(f"unknown init style '{spec.init}'")
        out[name] = v.reshape(shape)
    return out
