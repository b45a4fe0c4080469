"""shardsim-shaped front end on the B200 runtime.

Mirrors the reference engine's public API (`engine.py:60-882`): RAF / NRAF,
ACCUM_*, PrecisionPolicy, ScalerConfig, ShardedGradScaler, EngineConfig (with
the same validation errors), StepResult and Session (`train_step`, `run`,
`gather_full_params`, `replica_divergence`, `check_reduction_ordering`,
`order_hook`, `inject_inf`).  Differences are the ones a real system has:

* one Session per process = per rank (the reference simulates all W ranks in
  one process); the plan's world size must equal torch.distributed's;
* full precision is fp32 (master / optimizer / reduced grads) and low
  precision is bf16 (reference: float64 / float32, numerics.py:17-18);
* time is real: `sim_time` is the step's device time in ms.

The model is the reference's layered MLP (ModelSpec) with the reference's
initial values and data stream (data.py), computed by torch on the GPU.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import torch
import torch.nn.functional as F

from .data import ModelSpec, batch_stream, init_values, init_values_for  # noqa: F401  (re-exported)
from . import kernels
from .layout import build_unit_layouts
from .plan import ShardingPlan
from .runtime import (ACCUM_NO_COMM, ACCUM_OFF, ACCUM_WITH_COMM, NRAF, PREFETCH_POST, RAF,
                      EngineError, FSDPRuntime, PreBackward, RuntimeConfig, StaticOrderError,
                      UnitViews)

__all__ = ["RAF", "NRAF", "ACCUM_OFF", "ACCUM_WITH_COMM", "ACCUM_NO_COMM", "EngineError",
           "StaticOrderError", "PrecisionPolicy", "ScalerConfig", "ShardedGradScaler",
           "EngineConfig", "StepResult", "Session", "ModelSpec", "ExecutionOrder"]


@dataclass(frozen=True)
class PrecisionPolicy:
    """engine.py:80-106: mixed = compute/communicate bf16, master fp32."""
    mixed: bool = False
    reduce_in_low: bool = True

    @property
    def compute_dtype(self) -> str:
        return "low" if self.mixed else "full"

    @property
    def reduce_dtype(self) -> str:
        return "low" if (self.mixed and self.reduce_in_low) else "full"

    @property
    def k_full(self) -> int:
        return 4

    @property
    def k_low(self) -> int:
        return 2


@dataclass
class ScalerConfig:
    init_scale: float = 65536.0
    growth_factor: float = 2.0
    backoff_factor: float = 0.5
    growth_interval: int = 2000


class ShardedGradScaler:
    """engine.py:118-145: every rank takes the identical step/skip decision
    from the world all-reduced found_inf flag."""

    def __init__(self, cfg: ScalerConfig | None = None):
        self.cfg = cfg or ScalerConfig()
        self.scale = float(self.cfg.init_scale)
        self._growth_tracker = 0
        self.steps_skipped = 0

    def update(self, found_inf: bool) -> None:
        if found_inf:
            self.scale *= self.cfg.backoff_factor
            self._growth_tracker = 0
            self.steps_skipped += 1
        else:
            self._growth_tracker += 1
            if self._growth_tracker >= self.cfg.growth_interval:
                self.scale *= self.cfg.growth_factor
                self._growth_tracker = 0
        if not math.isfinite(self.scale) or self.scale <= 0.0:
            raise EngineError(f"gradient scale became non-positive or non-finite: {self.scale}")


class ExecutionOrder:
    """engine.py:148-162."""

    def __init__(self) -> None:
        self.order: list[int] = []
        self._seen: set[int] = set()

    def record(self, unit: int) -> None:
        if unit in self._seen:
            raise EngineError(f"unit {unit} materialized twice in one forward")
        self._seen.add(unit)
        self.order.append(unit)

    def backward_order(self) -> list[int]:
        return list(reversed(self.order))


@dataclass
class EngineConfig:
    plan: ShardingPlan
    reshard_after_forward: str = RAF
    backward_prefetch: bool = True
    forward_prefetch: bool = False
    rate_limit: int | None = 2
    precision: PrecisionPolicy = field(default_factory=PrecisionPolicy)
    accumulation: str = ACCUM_OFF
    accumulation_steps: int = 1
    keep_outermost_unsharded: bool = True
    loss_reduction: str = "mean"
    optimizer: str = "sgd"
    lr: float | None = None
    use_scaler: bool = False
    scaler: ScalerConfig = field(default_factory=ScalerConfig)
    forwards_per_micro: int = 1
    init_path: str = "deferred"
    capacity_bytes: int | None = None
    deterministic: bool = True
    comm_backend: str = "ipc"

    def __post_init__(self) -> None:              # engine.py:187-206
        if self.reshard_after_forward not in (RAF, NRAF):
            raise EngineError(f"reshard_after_forward must be {RAF} or {NRAF}, got "
                              f"{self.reshard_after_forward!r}")
        if self.accumulation not in (ACCUM_OFF, ACCUM_WITH_COMM, ACCUM_NO_COMM):
            raise EngineError(f"accumulation must be one of off/with_comm/no_comm, got "
                              f"{self.accumulation!r}")
        if self.accumulation == ACCUM_OFF and self.accumulation_steps != 1:
            raise EngineError("accumulation off requires accumulation_steps=1")
        if self.accumulation_steps < 1:
            raise EngineError("accumulation_steps must be >= 1")
        if self.rate_limit is not None and self.rate_limit < 1:
            raise EngineError("rate_limit must be >= 1 (or None for no limit)")
        if self.forwards_per_micro < 1:
            raise EngineError("forwards_per_micro must be >= 1")
        if self.init_path not in ("deferred", "device", "streamed"):
            raise EngineError(f"unknown init_path {self.init_path!r}")
        if self.loss_reduction not in ("mean", "sum"):
            raise EngineError(f"unknown loss_reduction {self.loss_reduction!r}")
        if self.optimizer not in ("sgd", "adam"):
            raise EngineError(f"unknown optimizer {self.optimizer!r}")


@dataclass
class StepResult:
    step: int
    loss: float
    rank_losses: list[float]
    stepped: bool
    found_inf: bool
    scale: float | None
    sim_time: float             # device ms of this step (rank max)
    makespan: float             # cumulative device ms
    event_counts: dict[str, int]


def _act(kind: str, z: torch.Tensor) -> torch.Tensor:
    if kind == "relu":
        return F.relu(z)
    if kind == "tanh":
        return torch.tanh(z)
    raise EngineError(f"unknown activation '{kind}'")


class Session:
    """One rank of a sharded training world on a B200."""

    def __init__(self, spec: ModelSpec, config: EngineConfig, seed: int = 0):
        import torch.distributed as dist
        self.spec, self.config, self.seed = spec, config, seed
        self.plan = config.plan
        W = self.plan.world_size
        on = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank() if on else 0
        if (dist.get_world_size() if on else 1) != W:
            raise EngineError(f"plan.world_size {W} != number of processes "
                              f"{dist.get_world_size() if on else 1} (one Session per GPU)")
        self.layouts = build_unit_layouts(spec.param_shapes(), spec.unit_param_names(),
                                          self.plan.shard_factor)
        self.num_units = len(self.layouts)
        lr = config.lr if config.lr is not None else (0.03125 if config.optimizer == "sgd" else 1e-3)
        rcfg = RuntimeConfig(
            mixed=config.precision.mixed, reduce_in_low=config.precision.reduce_in_low,
            reshard_after_forward=config.reshard_after_forward,
            backward_prefetch=PREFETCH_POST if config.backward_prefetch else None,
            forward_prefetch=config.forward_prefetch, rate_limit=config.rate_limit,
            keep_outermost_unsharded=config.keep_outermost_unsharded,
            accumulation=config.accumulation, accumulation_steps=config.accumulation_steps,
            loss_mean=config.loss_reduction == "mean", optimizer=config.optimizer, lr=lr,
            comm_backend=config.comm_backend)
        comm, pgs = None, {}
        if W > 1 and config.comm_backend == "ipc":
            from .comm import DeviceComm
            comm = DeviceComm.create(FSDPRuntime.pool_bytes_for(self.layouts, self.plan, rcfg))
        elif W > 1:
            from .fsdp import _nccl_groups
            pgs = _nccl_groups(self.plan, self.rank)
        self.comm = comm
        self.rt = FSDPRuntime(self.layouts, self.plan, self.rank, rcfg, comm=comm,
                              process_groups=pgs)
        self.init_stats = self._materialise(config.init_path)
        self.scaler = ShardedGradScaler(config.scaler) if config.use_scaler else None
        self.device = self.rt.device
        self._anchors = [torch.zeros((), device=self.device, requires_grad=True)
                         for _ in self.layouts]
        self.step_count = 0
        self.order_hook: Callable[[int], Sequence[int]] | None = None
        self.inject_inf: set[tuple[int, int]] = set()
        self.results: list[StepResult] = []
        self._makespan = 0.0
        self.compute_dtype = torch.bfloat16 if config.precision.mixed else torch.float32
        torch.cuda.synchronize()

    # -- initialisation (deferred_init.py:156-263) ---------------------------
    def _materialise(self, path: str) -> dict:
        """The reference's three materialisation paths, on the device.

        Values come from the same replay (`init_values`: PRNG streams keyed
        by (seed, name)), so every path yields bit-identical shards
        (test_acceptance.py:402-433).  They differ in what is resident:
          deferred : one unit at a time — host replay of the unit, H2D,
                     flatten into an unsharded psi buffer, shard, free
                     (materialize_by_unit, :156-176);
          device   : every unit's unsharded buffer first, then shard them all
                     (init_unsharded_on_device, :179-208) — peaks at the full
                     unsharded model;
          streamed : the whole model replayed into one pinned host arena
                     (raw, unpadded), then each unit copied H2D into a padded
                     device buffer and sharded (init_streamed_from_host,
                     :227-263) — host holds the model, device one unit.
        Returns device peak bytes above the pre-init level and the host
        arena's element peak."""
        rt, spec = self.rt, self.spec
        dev = rt.device
        torch.cuda.synchronize(dev)
        base = torch.cuda.memory_allocated(dev)
        torch.cuda.reset_peak_memory_stats(dev)
        host_peak = 0
        shard_k = self.plan.shard_index(self.rank)

        def finish(uid: int, flat: torch.Tensor) -> None:
            u = rt.units[uid]
            kernels.shard_copy(flat, u.master, shard_k)
            if u.low is not None:
                kernels.cast(u.master, u.low)

        def flatten_unit(uid: int, vals: dict) -> torch.Tensor:
            lay = self.layouts[uid]
            srcs = [torch.from_numpy(np.ascontiguousarray(vals[o.name], dtype=np.float32)).to(dev)
                    for o in lay.originals]
            flat = torch.empty(lay.psi, dtype=torch.float32, device=dev)
            kernels.flatten(srcs, lay.offsets, flat)
            return flat

        if path == "deferred":
            for uid, lay in enumerate(self.layouts):
                vals = init_values_for(spec, self.seed, [o.name for o in lay.originals])
                finish(uid, flatten_unit(uid, vals))
                torch.cuda.synchronize(dev)      # the unit's buffers die here
        elif path == "device":
            vals = init_values(spec, self.seed)
            flats = [flatten_unit(uid, vals) for uid in range(len(self.layouts))]
            for uid, flat in enumerate(flats):
                finish(uid, flat)
            torch.cuda.synchronize(dev)
            del flats
        else:   # streamed
            raws = [lay.raw_numel for lay in self.layouts]
            arena = torch.empty(sum(raws), dtype=torch.float32).pin_memory()
            host_peak = arena.numel()
            vals = init_values(spec, self.seed)
            cur = 0
            for lay in self.layouts:
                for o in lay.originals:
                    n = int(np.prod(o.shape))
                    arena[cur: cur + n] = torch.from_numpy(
                        np.ascontiguousarray(vals[o.name], dtype=np.float32).reshape(-1))
                    cur += n
            cur = 0
            for uid, lay in enumerate(self.layouts):
                flat = torch.empty(lay.psi, dtype=torch.float32, device=dev)
                flat[: lay.raw_numel].copy_(arena[cur: cur + lay.raw_numel], non_blocking=True)
                if lay.psi > lay.raw_numel:
                    flat[lay.raw_numel:].zero_()
                finish(uid, flat)
                cur += lay.raw_numel
                torch.cuda.synchronize(dev)
            del arena
        torch.cuda.synchronize(dev)
        return {"path": path, "device_peak_bytes": torch.cuda.max_memory_allocated(dev) - base,
                "host_arena_peak_elements": host_peak}

    # -- ordering -----------------------------------------------------------
    def _order_for(self, step: int) -> list[int]:
        if self.order_hook is not None:
            order = list(self.order_hook(step))
            if sorted(order) != list(range(self.num_units)):
                raise EngineError(f"order hook returned {order}, not a permutation of "
                                  f"{self.num_units} units")
            return order
        return list(range(self.num_units))

    @property
    def trace(self) -> list[tuple[str, int | None]]:
        return self.rt.trace

    # -- the unit computations ----------------------------------------------
    def _forward_unit(self, u: int, h: torch.Tensor, pos: int, outermost: int) -> torch.Tensor:
        rt = self.rt
        rt.record_forward(u)
        flat = rt.ensure_unsharded(u)
        rt.forward_prefetch_after(pos)
        rt.trace.append(("compute_begin", u))
        views = UnitViews.apply(self._anchors[u], flat, rt, u)
        p = {o.name: v for o, v in zip(self.layouts[u].originals, views)}
        for i in self.spec.units[u]:
            z = F.linear(h, p[f"linear{i}.weight"], p.get(f"linear{i}.bias"))
            h = z if i == self.spec.num_linears - 1 else _act(self.spec.activation, z)
        rt.post_order.append(u)
        rt.close_window(u)
        if torch.is_grad_enabled():
            (h,) = PreBackward.apply(rt, u, h)
        rt.release_use(u, "forward", outermost)
        return h

    def _local_loss(self, pred: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        d = pred.float() - y
        return (d * d).mean() if self.config.loss_reduction == "mean" else (d * d).sum()

    # -- public driving -----------------------------------------------------
    def train_step(self, micro_batches, threaded: bool = False) -> StepResult:
        import torch.distributed as dist
        cfg = self.config
        if len(micro_batches) != cfg.accumulation_steps:
            raise EngineError(f"expected {cfg.accumulation_steps} micro-batches per step "
                              f"(accumulation {cfg.accumulation}), got {len(micro_batches)}")
        W = self.plan.world_size
        for x, _ in micro_batches:
            if x.shape[0] % W != 0:
                raise EngineError(f"batch size {x.shape[0]} not divisible by world size {W}")
        step = self.step_count
        order = self._order_for(step)
        rt = self.rt
        rt.inject_inf = {s for (r, s) in self.inject_inf if r == self.rank}
        trace0 = len(rt.trace)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        rt.begin_step()
        micro_losses = []
        k = len(micro_batches)
        per = micro_batches[0][0].shape[0] // W
        for m, (x, y) in enumerate(micro_batches):
            rt.begin_micro(final=(m == k - 1))
            xs = torch.from_numpy(np.ascontiguousarray(x[self.rank * per:(self.rank + 1) * per]))
            ys = torch.from_numpy(np.ascontiguousarray(y[self.rank * per:(self.rank + 1) * per]))
            xs = xs.to(self.device, self.compute_dtype)
            ys = ys.to(self.device, torch.float32)
            total = None
            loss_sum = 0.0
            with rt.saved_tensor_hooks():
                for _ in range(cfg.forwards_per_micro):
                    rt.begin_forward_pass()
                    h = xs
                    for pos, u in enumerate(order):
                        h = self._forward_unit(u, h, pos, order[-1])
                    loss = self._local_loss(h, ys)
                    loss_sum = loss_sum + loss.detach()
                    scaled = loss * self.scaler.scale if self.scaler is not None else loss
                    total = scaled if total is None else total + scaled
            total.backward()
            micro_losses.append(loss_sum)
        found = False
        scale = self.scaler.scale if self.scaler is not None else None
        rt.optimizer_step(scale)
        if self.scaler is not None:
            found = bool(rt.found_inf_world.item() > 0.0)     # host reads the verdict
            if found:
                rt.undo_adam_t()
            self.scaler.update(found)
        rt.trace.append(("step", None))
        t1.record()
        rank_loss = torch.stack(micro_losses).float().mean()
        losses = torch.zeros(W, device=self.device)
        losses[self.rank] = rank_loss
        counts: dict[str, int] = {}
        for kind, _ in rt.trace[trace0:]:
            if kind.endswith("_issue"):
                counts[kind[:-6]] = counts.get(kind[:-6], 0) + 1
        cvec = torch.tensor([counts.get(c, 0) for c in ("AG", "RS", "AR")], device=self.device,
                            dtype=torch.float32)
        torch.cuda.synchronize()
        rt.raise_if_aborted(sync=True)          # DeadlockError (collectives.py:476-482)
        ms = torch.tensor([t0.elapsed_time(t1)], device=self.device)
        if W > 1:
            from .dist_util import all_reduce_
            all_reduce_(losses)
            all_reduce_(cvec)
            all_reduce_(ms, op=dist.ReduceOp.MAX)
        self._makespan += ms.item()
        rl = losses.tolist()
        counts = {c: int(v) for c, v in zip(("AG", "RS", "AR"), cvec.tolist()) if v > 0}
        res = StepResult(step=step, loss=float(np.mean(rl)), rank_losses=rl, stepped=not found,
                         found_inf=found, scale=self.scaler.scale if self.scaler else None,
                         sim_time=ms.item(), makespan=self._makespan, event_counts=counts)
        self.results.append(res)
        self.step_count += 1
        return res

    def run(self, steps: int, batch: int, regime: str = "integer",
            threaded: bool = False) -> list[StepResult]:
        k = self.config.accumulation_steps
        stream = batch_stream(self.seed, steps * k, batch, self.spec.dims[0], self.spec.dims[-1],
                              regime)
        return [self.train_step([next(stream) for _ in range(k)]) for _ in range(steps)]

    # -- inspection ---------------------------------------------------------
    def _all_gather_shard(self, t: torch.Tensor, group_ranks) -> torch.Tensor:
        from .dist_util import all_gather
        if len(group_ranks) == 1:
            return t.clone()
        out = all_gather(t)
        return torch.cat([out[r] for r in group_ranks])

    def gather_full_params(self) -> dict[str, np.ndarray]:
        """engine.py:824-834: reassemble fp32 parameters from sharded group 0
        (unflatten kernel into the original shapes)."""
        from . import kernels
        g0 = self.plan.sharded_groups[0]
        out = {}
        for u, lay in enumerate(self.layouts):
            flat = self._all_gather_shard(self.rt.units[u].master, g0)
            ts = [torch.empty(o.shape, dtype=torch.float32, device=self.device) for o in lay.originals]
            kernels.unflatten(flat, ts, lay.offsets)
            for o, t in zip(lay.originals, ts):
                out[o.name] = t.cpu().numpy()
        return out

    def replica_divergence(self) -> float:
        """engine.py:836-846: max |shard difference| across replicas."""
        from .dist_util import all_gather
        if self.plan.world_size == 1:
            return 0.0
        worst = 0.0
        for u in range(self.num_units):
            t = self.rt.units[u].master
            allv = all_gather(t)
            for grp in self.plan.replicated_groups:
                for r in grp[1:]:
                    if t.numel():
                        worst = max(worst, float((allv[grp[0]] - allv[r]).abs().max()))
        return worst

    def check_reduction_ordering(self) -> list[str]:
        """engine.py:848-878 on this rank's event log."""
        problems = []
        finalized: dict = {}
        reduced: dict = {}
        last_reduce: dict = {}
        opt: dict = {}
        for i, (step, kind, unit) in enumerate(self.rt.events):
            if kind == "grad_finalized":
                finalized[(step, unit)] = finalized.get((step, unit), 0) + 1
            elif kind == "reduce_issue":
                if reduced.get((step, unit), 0) >= finalized.get((step, unit), 0):
                    problems.append(f"rank {self.rank} step {step}: reduce of unit {unit} before "
                                    f"gradient finalized")
                reduced[(step, unit)] = reduced.get((step, unit), 0) + 1
                last_reduce[step] = i
            elif kind == "reduce_stage2":
                last_reduce[step] = i
            elif kind == "opt_step":
                opt[step] = i
        for step, i in opt.items():
            if last_reduce.get(step, -1) > i:
                problems.append(f"rank {self.rank} step {step}: optimizer step before the last reduction")
        return problems

    def close(self) -> None:
        if self.comm is not None:
            self.comm.close()
            self.comm = None
