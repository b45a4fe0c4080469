"""ORACLE (test infrastructure only) — numpy restatement of the shardsim
sharded-training hot path.  See `oracle/__init__.py` for who may import it.

Citations are `file:line` into the reference's `pkg/src/shardsim/`.

Dtypes.  The reference runs full = float64, low = float32
(`numerics.py:17-18`).  Every function here takes the dtypes as arguments so
the same code
  * reproduces shardsim bit-for-bit with (full=float64, low=float32) — pinned
    against golden vectors produced by the real reference, and
  * defines the B200 build's expected bits with (full=float32, low="bf16").
bf16 arrays are carried as float32 arrays holding bf16-representable values
(`round_to_bf16`); the build never does arithmetic *in* bf16, only casts.

One deliberate, documented difference for the B200 build: the reference
accumulates collective sums in the payload dtype (`collectives.py:273-278`,
`acc = np.zeros_like(arrays[0])`).  The B200 reduce-scatter accumulates bf16
payloads in fp32 (BASELINE north star).  `acc_dtype` selects this: None =
reference behaviour, np.float32 = the build's.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from .bf16 import round_to_bf16

BF16 = "bf16"


def _np_dtype(dt):
    return np.float32 if dt == BF16 else dt


def cast(x: np.ndarray, dt) -> np.ndarray:
    """Cast to a dtype of this module (float64 / float32 / "bf16")."""
    if dt == BF16:
        return round_to_bf16(np.asarray(x, dtype=np.float32))
    return np.asarray(x).astype(dt)


# ---------------------------------------------------------------------------
# layout  (flatparam.py:33-96)
# ---------------------------------------------------------------------------

class FlatParamError(ValueError):
    pass


class SharedParameterError(FlatParamError):
    pass


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


def build_unit_layouts(param_shapes, unit_param_names, shard_factor):
    """flatparam.py:63-96 — declaration-order offsets, psi = ceil(raw/F)*F."""
    shapes = dict(param_shapes)
    owner = {}
    for uid, names in enumerate(unit_param_names):
        for n in names:
            if n in owner:                                   # :70-77
                raise SharedParameterError(
                    f"parameter '{n}' is assigned to units {owner[n]} and {uid}")
            if n not in shapes:                              # :78-79
                raise FlatParamError(f"unknown parameter '{n}'")
            owner[n] = uid
    missing = [n for n, _ in param_shapes if n not in owner]  # :81-84
    if missing:
        raise FlatParamError(f"unit boundaries do not cover parameters: {missing}")
    out = []
    for uid, names in enumerate(unit_param_names):
        origs, off = [], 0
        for n in names:                                      # :88-92
            origs.append(OriginalParam(n, tuple(shapes[n]), off))
            off += math.prod(shapes[n])
        psi = -(-off // shard_factor) * shard_factor if off else 0   # :93
        out.append(UnitLayout(uid, tuple(origs), psi, psi - off, shard_factor))
    return out


def dump_plan_lines(layouts):
    """flatparam.py:238-247 golden line format."""
    lines = []
    for l in layouts:
        shapes = " ".join(f"{o.name}:{'x'.join(str(d) for d in o.shape)}"
                          for o in l.originals)
        lines.append(f"unit={l.unit_id} ψ={l.psi} padding={l.padding} "
                     f"originals=[{shapes}]")
    return lines


# ---------------------------------------------------------------------------
# plan  (collectives.py:37-106)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Plan:
    world_size: int
    shard_factor: int

    def __post_init__(self):
        w, f = self.world_size, self.shard_factor
        if w < 1 or not 1 <= f <= w or w % f:
            raise ValueError(f"shard_factor {f} must divide world_size {w}")

    @property
    def sharded_groups(self):                                # :63-66
        f = self.shard_factor
        return [tuple(range(i * f, (i + 1) * f)) for i in range(self.world_size // f)]

    @property
    def replicated_groups(self):                             # :68-71
        f = self.shard_factor
        return [tuple(range(j, self.world_size, f)) for j in range(f)]

    def sharded_group_of(self, r):                           # :89-92
        b = (r // self.shard_factor) * self.shard_factor
        return tuple(range(b, b + self.shard_factor))

    def replicated_group_of(self, r):                        # :94-96
        return tuple(range(r % self.shard_factor, self.world_size, self.shard_factor))


# ---------------------------------------------------------------------------
# flat parameter values  (flatparam.py:113-164, deferred_init.py:156-176)
# ---------------------------------------------------------------------------

def flatten(values: dict, layout: UnitLayout, dtype) -> np.ndarray:
    """Unsharded flat buffer: originals at their offsets, pad = 0
    (deferred_init.py:167-171 replays into zero-initialised views)."""
    buf = np.zeros(layout.psi, dtype=_np_dtype(dtype))
    for o in layout.originals:
        buf[o.offset:o.offset + o.numel] = cast(np.asarray(values[o.name]).reshape(-1), dtype)
    return buf


def shard_index(plan: Plan, rank: int) -> int:
    return rank % plan.shard_factor                          # flatparam.py:113


def shard(flat: np.ndarray, layout: UnitLayout, index: int) -> np.ndarray:
    """flatparam.py:124-126 / :139-147 — copy chunk `index` of psi."""
    b = layout.shard_numel
    return flat[index * b:(index + 1) * b].copy()


def unflatten(flat: np.ndarray, layout: UnitLayout) -> dict:
    """Views of flatparam.py:159-164 materialised as copies
    (what gather_full_params does, engine.py:824-834)."""
    return {o.name: flat[o.offset:o.offset + o.numel].reshape(o.shape).copy()
            for o in layout.originals}


# ---------------------------------------------------------------------------
# collective values  (collectives.py:273-301, :377-397)
# ---------------------------------------------------------------------------

def fabric_reduce(arrays: Sequence[np.ndarray], acc_dtype=None) -> np.ndarray:
    """collectives.py:273-278: acc = zeros; acc = acc + a, ascending rank.
    acc_dtype None = the payload dtype (reference); else upcast first."""
    if acc_dtype is None:
        acc = np.zeros_like(arrays[0])
        for a in arrays:
            acc = acc + a
        return acc
    acc = np.zeros(arrays[0].shape, dtype=acc_dtype)
    for a in arrays:
        acc = acc + np.asarray(a).astype(acc_dtype)
    return acc


def all_gather(inputs: Sequence[np.ndarray]) -> np.ndarray:
    """collectives.py:288-291 — ascending-rank concatenation."""
    return np.concatenate(list(inputs))


def reduce_scatter(inputs: Sequence[np.ndarray], acc_dtype=None) -> list:
    """collectives.py:292-297 — position k gets chunk k of the sum."""
    n = len(inputs)
    if inputs[0].size % n:
        raise ValueError("reduce_scatter: length not divisible by group size")
    acc = fabric_reduce(inputs, acc_dtype)
    c = acc.size // n
    return [acc[k * c:(k + 1) * c].copy() for k in range(n)]


def all_reduce(inputs: Sequence[np.ndarray], acc_dtype=None) -> np.ndarray:
    """collectives.py:298-301."""
    return fabric_reduce(inputs, acc_dtype)


def hybrid_reduce(grads: Sequence[np.ndarray], plan: Plan, acc_dtype=None, stage2_dtype=None) -> list:
    """collectives.py:377-397 (Eq. 1): RS in the sharded group, then AR in
    the replicated group; degenerates to RS at F=W and AR at F=1.

    stage2_dtype: the partial is cast to it before the all-reduce (the
    reference's flow: the reduce-scatter output, in the payload dtype, is the
    all-reduce payload, engine.py:798-810); None keeps the acc_dtype partial."""
    w, f = plan.world_size, plan.shard_factor
    out = [None] * w
    if f == 1:
        total = all_reduce([grads[r] for r in range(w)], acc_dtype)
        return [total.copy() for _ in range(w)]
    partial = [None] * w
    for g in plan.sharded_groups:
        res = reduce_scatter([grads[r] for r in g], acc_dtype)
        for pos, r in enumerate(g):
            partial[r] = res[pos] if stage2_dtype is None or f == w else cast(res[pos], stage2_dtype)
    if f == w:
        return partial
    for g in plan.replicated_groups:
        total = all_reduce([partial[r] for r in g], acc_dtype)
        for r in g:
            out[r] = total.copy()
    return out


# ---------------------------------------------------------------------------
# gradient write-back and the per-unit reduction  (flatparam.py:167-191,
# engine.py:771-820)
# ---------------------------------------------------------------------------

def writeback_grad(layout: UnitLayout, grads: dict, dtype, out=None):
    """flatparam.py:167-191 — grads at offsets; pad and missing grads = 0."""
    if out is None:
        out = np.zeros(layout.psi, dtype=_np_dtype(dtype))
    else:
        out[:] = 0.0
    warnings = []
    for o in layout.originals:
        g = grads.get(o.name)
        if g is None:
            warnings.append(f"unit {layout.unit_id}: no gradient for '{o.name}', zero-filled")
            continue
        if tuple(np.shape(g)) != o.shape:
            raise FlatParamError(f"gradient shape {np.shape(g)} != parameter shape {o.shape}")
        out[o.offset:o.offset + o.numel] = cast(np.asarray(g).reshape(-1), dtype)
    return out, warnings


def reduce_unit(flat_grads: Sequence[np.ndarray], plan: Plan, *, reduce_dtype,
                full_dtype, acc_dtype=None, mean: bool = True,
                accum: Sequence[np.ndarray] | None = None, stage2_dtype=None) -> list:
    """engine.py:787-820 for every rank at once: payload = grad in the reduce
    dtype (:789-790); RS in the sharded group then AR in the replicated group
    (:798-816); astype(full) (:817); / W when the loss is a mean (:818-819);
    accum += (:820; a fresh accumulator starts at zeros, :791-796)."""
    w = plan.world_size
    payload = [cast(g, reduce_dtype) for g in flat_grads]
    reduced = hybrid_reduce(payload, plan, acc_dtype, stage2_dtype)
    out = []
    for r in range(w):
        red = np.asarray(reduced[r]).astype(full_dtype)
        if mean:
            red = red / full_dtype(w)
        base = np.zeros(red.shape, dtype=full_dtype) if accum is None or accum[r] is None \
            else accum[r]
        out.append(base + red)
    return out


# ---------------------------------------------------------------------------
# optimizers on shards  (numerics.py:239-296)
# ---------------------------------------------------------------------------

def sgd_step(param: np.ndarray, grad: np.ndarray, lr: float = 0.03125) -> None:
    """numerics.py:248-253: param -= lr * grad (python-float lr is weak)."""
    param -= lr * grad


def adam_init(n: int, dtype) -> dict:
    """numerics.py:268-271."""
    return {"m": np.zeros(n, dtype=dtype), "v": np.zeros(n, dtype=dtype), "t": 0}


def adam_step(param, grad, state, lr=1e-3, betas=(0.9, 0.999), eps=1e-8) -> None:
    """numerics.py:273-285, operation for operation (NEP 50: python floats
    are weak scalars, so float32 arrays compute in float32)."""
    b1, b2 = betas
    state["t"] += 1
    t = state["t"]
    state["m"] = b1 * state["m"] + (1.0 - b1) * grad
    state["v"] = b2 * state["v"] + (1.0 - b2) * grad * grad
    m_hat = state["m"] / (1.0 - b1 ** t)
    v_hat = state["v"] / (1.0 - b2 ** t)
    param -= lr * m_hat / (np.sqrt(v_hat) + eps)


# ---------------------------------------------------------------------------
# sharded gradient scaler  (engine.py:109-145, :563-576)
# ---------------------------------------------------------------------------

@dataclass
class Scaler:
    init_scale: float = 65536.0
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    growth_interval: int = 2000
    scale: float = field(default=None)
    tracker: int = 0
    skipped: int = 0

    def __post_init__(self):
        if self.scale is None:
            self.scale = float(self.init_scale)

    def update(self, found_inf: bool) -> None:              # engine.py:133-145
        if found_inf:
            self.scale *= self.backoff_factor
            self.tracker = 0
            self.skipped += 1
        else:
            self.tracker += 1
            if self.tracker >= self.growth_interval:
                self.scale *= self.growth_factor
                self.tracker = 0


def unscale_and_check(accums: Sequence[np.ndarray], scale: float) -> bool:
    """engine.py:566-571 for one rank: accum *= 1/scale in place; flag if any
    non-finite.  The world verdict is the all-reduced sum of flags > 0
    (:572-576)."""
    inv = 1.0 / scale
    flag = False
    for a in accums:
        a *= inv
        if not np.isfinite(a).all():
            flag = True
    return flag


# ---------------------------------------------------------------------------
# model + data used by the reference (numerics.py:73-232, :303-321,
# deferred_init.py:63-143) — only for pinning the composed step against
# shardsim's Session / local_train outputs.
# ---------------------------------------------------------------------------

def named_stream(seed: int, name: str) -> np.random.Generator:
    """numerics.py:73-78 (sha256-keyed SeedSequence)."""
    key = int.from_bytes(hashlib.sha256(name.encode("utf-8")).digest()[:8], "big")
    return np.random.default_rng(np.random.SeedSequence([seed, key]))


def batch_stream(seed, steps, batch, dim_in, dim_out, regime="integer"):
    """numerics.py:303-321."""
    rng = named_stream(seed, "data")
    for _ in range(steps):
        if regime == "integer":
            x = rng.integers(-3, 4, size=(batch, dim_in)).astype(np.float64)
            y = rng.integers(-3, 4, size=(batch, dim_out)).astype(np.float64)
        elif regime == "uniform":
            x = rng.uniform(-1.0, 1.0, size=(batch, dim_in))
            y = rng.uniform(-1.0, 1.0, size=(batch, dim_out))
        else:
            raise ValueError(regime)
        yield x, y


@dataclass(frozen=True)
class MLPSpec:
    """numerics.py:81-127 (ModelSpec), restated."""
    dims: tuple = (4, 8, 8, 2)
    activation: str = "relu"
    unit_sizes: tuple | None = None
    init: str = "dyadic"
    bias: bool = True

    @property
    def num_linears(self):
        return len(self.dims) - 1

    @property
    def units(self):
        sizes = self.unit_sizes or tuple(1 for _ in range(self.num_linears))
        out, nxt = [], 0
        for s in sizes:
            out.append(list(range(nxt, nxt + s)))
            nxt += s
        return out

    def param_shapes(self):
        shapes = []
        for i in range(self.num_linears):
            shapes.append((f"linear{i}.weight", (self.dims[i + 1], self.dims[i])))
            if self.bias:
                shapes.append((f"linear{i}.bias", (self.dims[i + 1],)))
        return shapes

    def unit_param_names(self):
        per = {}
        for n, _ in self.param_shapes():
            per.setdefault(int(n.split(".")[0][6:]), []).append(n)
        return [[n for li in u for n in per[li]] for u in self.units]


_ROUND_SHIFT = 3.0 * 2.0 ** 51


def eager_param_values(spec: MLPSpec, seed: int) -> dict:
    """deferred_init.py:63-143 replay semantics for the styles the model zoo
    uses (float64, keyed by (seed, name))."""
    out = {}
    for name, shape in spec.param_shapes():
        n = math.prod(shape)
        fan_in = shape[-1] if len(shape) > 1 else shape[0]
        rng = named_stream(seed, name)
        if spec.init == "zeros":
            buf = np.zeros(n)
        elif spec.init == "dyadic":                          # :69-77
            buf = rng.uniform(0.0, 1.0, size=n)
            buf *= 8.0
            buf += _ROUND_SHIFT
            buf += -_ROUND_SHIFT
            buf *= 0.125
            buf += -0.5
        elif spec.init == "scaled_uniform":
            buf = rng.uniform(-1.0, 1.0, size=n)
            buf *= 1.0 / math.sqrt(max(fan_in, 1))
        elif spec.init == "normal":
            buf = rng.normal(0.0, 1.0, size=n)
            buf *= 1.0 / math.sqrt(max(fan_in, 1))
        else:
            raise ValueError(spec.init)
        out[name] = buf.reshape(shape)
    return out


def _act(kind, z):
    return z * (z > 0) if kind == "relu" else np.tanh(z)


def _act_bwd(kind, z, d):
    if kind == "relu":
        return d * (z > 0)
    t = np.tanh(z)
    return d * (1.0 - t * t)


def forward_unit(spec: MLPSpec, params: dict, unit: int, x):
    """numerics.py:160-170."""
    cache = []
    for i in spec.units[unit]:
        w = params[f"linear{i}.weight"]
        z = x @ w.T
        if spec.bias:
            z = z + params[f"linear{i}.bias"]
        last = i == spec.num_linears - 1
        a = z if last else _act(spec.activation, z)
        cache.append((i, x, z, last))
        x = a
    return x, cache


def backward_unit(spec: MLPSpec, params: dict, cache, dout):
    """numerics.py:172-185."""
    grads = {}
    for i, x, z, last in reversed(cache):
        dz = dout if last else _act_bwd(spec.activation, z, dout)
        grads[f"linear{i}.weight"] = dz.T @ x
        if spec.bias:
            grads[f"linear{i}.bias"] = dz.sum(axis=0)
        dout = dz @ params[f"linear{i}.weight"]
    return dout, grads


def mse_loss(pred, target, reduction="mean"):
    """numerics.py:222-232."""
    diff = pred - target
    if reduction == "mean":
        return float((diff * diff).mean()), (2.0 / diff.size) * diff
    return float((diff * diff).sum()), 2.0 * diff


def sharded_train(spec: MLPSpec, plan: Plan, seed: int, steps: int, batch: int, *,
                  regime="integer", optimizer="sgd", lr=None, mixed=False,
                  reduce_in_low=True, accumulation="off", accumulation_steps=1,
                  loss_reduction="mean", use_scaler=False, scaler_kw=None,
                  forwards_per_micro=1, inject_inf=(), order=None,
                  full=np.float64, low=np.float32, acc_dtype=None):
    """Value-level restatement of `Session.run` (engine.py:376-597): the
    scheduling (prefetch, limiter, RAF/NRAF, threads) never changes values, so
    only the arithmetic is restated.  Returns (full params dict, per-step
    losses, per-step stepped flags, scales)."""
    w, f = plan.world_size, plan.shard_factor
    layouts = build_unit_layouts(spec.param_shapes(), spec.unit_param_names(), f)
    nu = len(layouts)
    order = list(range(nu)) if order is None else list(order)
    init = eager_param_values(spec, seed)
    # shards[r][u] full precision (engine.py:324-338 via materialize_by_unit)
    shards = [[shard(flatten(init, lay, full), lay, shard_index(plan, r)) for lay in layouts]
              for r in range(w)]
    lr_ = lr
    opt_states = [[adam_init(lay.shard_numel, full) for lay in layouts] for _ in range(w)]
    scaler = Scaler(**(scaler_kw or {})) if use_scaler else None
    compute = low if mixed else full
    reduce_dt = low if (mixed and reduce_in_low) else full
    stream = batch_stream(seed, steps * accumulation_steps, batch, spec.dims[0],
                          spec.dims[-1], regime)
    losses, stepped_l, scales = [], [], []
    for step in range(steps):
        micros = [next(stream) for _ in range(accumulation_steps)]
        per = batch // w
        accum = [[None] * nu for _ in range(w)]
        accum_unsh = [[None] * nu for _ in range(w)]
        rank_losses = []
        # gathered (unsharded) params in compute dtype, per sharded group
        full_params = []
        for r in range(w):
            g = plan.sharded_group_of(r)
            vals = {}
            for u, lay in enumerate(layouts):
                payload = [cast(shards[q][u], compute) if mixed else shards[q][u] for q in g]
                flat = all_gather(payload) if f > 1 else (
                    cast(shards[r][u], compute) if mixed else shards[r][u])
                vals.update(unflatten(flat, lay))
            full_params.append(vals)
        for m, (x, y) in enumerate(micros):
            final = m == accumulation_steps - 1
            flat_grads = [[None] * nu for _ in range(w)]
            for r in range(w):
                xs, ys = x[r * per:(r + 1) * per], y[r * per:(r + 1) * per]
                passes, lsum = [], 0.0
                for _ in range(forwards_per_micro):
                    h = xs.astype(compute)
                    caches = {}
                    for u in order:
                        h, caches[u] = forward_unit(spec, full_params[r], u, h)
                    loss, dpred = mse_loss(h.astype(np.float64), ys, loss_reduction)
                    if scaler is not None:
                        dpred = dpred * scaler.scale
                    lsum += loss
                    passes.append((caches, dpred))
                rank_losses.append((r, m, lsum))
                for caches, dpred in reversed(passes):
                    dout = dpred.astype(compute)
                    for u in reversed(order):
                        dout, ug = backward_unit(spec, full_params[r], caches[u], dout)
                        fl, _ = writeback_grad(layouts[u], ug, compute)
                        flat_grads[r][u] = fl if flat_grads[r][u] is None else flat_grads[r][u] + fl
            for u in range(nu):
                if (final and u == 0):
                    for r in range(w):
                        if (r, step) in inject_inf:
                            flat_grads[r][u][0] = np.inf
                if accumulation == "no_comm":
                    for r in range(w):
                        a = accum_unsh[r][u]
                        accum_unsh[r][u] = (np.zeros(layouts[u].psi, dtype=np.float64)
                                            if a is None else a) + flat_grads[r][u]
                    if final:
                        res = reduce_unit([accum_unsh[r][u] for r in range(w)], plan,
                                          reduce_dtype=reduce_dt, full_dtype=full,
                                          acc_dtype=acc_dtype,
                                          mean=loss_reduction == "mean",
                                          accum=[accum[r][u] for r in range(w)])
                        for r in range(w):
                            accum[r][u] = res[r]
                else:
                    res = reduce_unit([flat_grads[r][u] for r in range(w)], plan,
                                      reduce_dtype=reduce_dt, full_dtype=full,
                                      acc_dtype=acc_dtype,
                                      mean=loss_reduction == "mean",
                                      accum=[accum[r][u] for r in range(w)])
                    for r in range(w):
                        accum[r][u] = res[r]
        found = False
        if scaler is not None:
            flags = [unscale_and_check(accum[r], scaler.scale) for r in range(w)]
            found = sum(1.0 if fl else 0.0 for fl in flags) > 0.0
        if not found:
            for r in range(w):
                for u in range(nu):
                    if optimizer == "sgd":
                        sgd_step(shards[r][u], accum[r][u], 0.03125 if lr_ is None else lr_)
                    else:
                        adam_step(shards[r][u], accum[r][u], opt_states[r][u],
                                  lr=1e-3 if lr_ is None else lr_)
        if scaler is not None:
            scaler.update(found)
        per_rank = {}
        for r, m, l in rank_losses:
            per_rank.setdefault(r, []).append(l)
        losses.append(float(np.mean([float(np.mean(per_rank[r])) for r in range(w)])))
        stepped_l.append(not found)
        scales.append(scaler.scale if scaler else None)
    out = {}
    for u, lay in enumerate(layouts):
        flat = np.concatenate([shards[r][u] for r in plan.sharded_groups[0]])
        out.update(unflatten(flat, lay))
    return out, losses, stepped_l, scales


def fsdp_reduce_and_step(flat_grads_by_rank, shards_by_rank, plan: Plan, *,
                         optimizer="adam", opt_states=None, lr=None,
                         betas=(0.9, 0.999), eps=1e-8, mean=True,
                         reduce_dtype=BF16, full=np.float32, acc_dtype=np.float32,
                         scale: float | None = None, stage2_dtype=None):
    """The B200 build's epilogue for one unit and one step, every rank:
    payload cast -> RS(+AR) with fp32 accumulation -> / W -> unscale ->
    world verdict -> optimizer on the shard.  (engine.py:771-820, :563-589.)
    Mutates shards/opt_states in place; returns (accums, found_inf)."""
    w = plan.world_size
    accums = reduce_unit(flat_grads_by_rank, plan, reduce_dtype=reduce_dtype,
                         full_dtype=full, acc_dtype=acc_dtype, mean=mean,
                         stage2_dtype=stage2_dtype)
    found = False
    if scale is not None:
        flags = [unscale_and_check([accums[r]], scale) for r in range(w)]
        found = any(flags)
    if not found:
        for r in range(w):
            if optimizer == "sgd":
                sgd_step(shards_by_rank[r], accums[r], 0.03125 if lr is None else lr)
            else:
                adam_step(shards_by_rank[r], accums[r], opt_states[r],
                          lr=1e-3 if lr is None else lr, betas=betas, eps=eps)
    return accums, found


def tree_sum(parts: Iterable[dict], block: int) -> dict:
    """engine.py:899-917."""
    parts = list(parts)
    total = None
    for i in range(0, len(parts), block):
        group = parts[i:i + block]
        partial = {k: v.copy() for k, v in group[0].items()}
        for p in group[1:]:
            for k in partial:
                partial[k] += p[k]
        if total is None:
            total = partial
        else:
            for k in total:
                total[k] += partial[k]
    return total
