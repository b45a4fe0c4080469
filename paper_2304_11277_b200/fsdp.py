"""torch-FSDP-v1-shaped wrapper over the B200 runtime.

    model = FullyShardedDataParallel(
        module, sharding_strategy=ShardingStrategy.FULL_SHARD,
        auto_wrap_policy=ModuleWrapPolicy({Block}),
        backward_prefetch=BackwardPrefetch.BACKWARD_PRE,
        mixed_precision=MixedPrecision(param_dtype=torch.bfloat16,
                                       reduce_dtype=torch.bfloat16),
        forward_prefetch=False, limit_all_gathers=True)
    opt = model.optimizer(lr=1e-4)           # sharded Adam over the rank's arena
    loss = model(x).loss; loss.backward(); opt.step()

Mapping to the reference engine (`engine.py:165-207`, EngineConfig):

  ShardingStrategy.FULL_SHARD       F = W, RAF
  ShardingStrategy.SHARD_GRAD_OP    F = W, NRAF
  ShardingStrategy.NO_SHARD         F = 1
  ShardingStrategy.HYBRID_SHARD     1 < F < W (hybrid_shard_size = F), RAF
  ShardingStrategy._HYBRID_SHARD_ZERO2  hybrid, NRAF
  BackwardPrefetch.BACKWARD_PRE     prefetch at the unit's pre-backward
  BackwardPrefetch.BACKWARD_POST    prefetch before the unit's reduce-scatter
                                    (the reference's point, engine.py:544-545)
  backward_prefetch=None            backward_prefetch=False
  forward_prefetch                  forward_prefetch
  limit_all_gathers                 rate_limit = 2 (else None); rate_limit=k overrides
  keep_outermost_unsharded=         keep_outermost_unsharded (default True, as torch)
  MixedPrecision(param_dtype=bf16)  PrecisionPolicy(mixed=True)
  MixedPrecision(reduce_dtype=fp32) PrecisionPolicy(reduce_in_low=False)
  hybrid_stage2="reduce" (default)  HYBRID's replica all-reduce moves the
                                    reduce-scatter's partial in the reduce dtype
                                    (as torch FSDP and engine.py:798-810; sums
                                    in fp32); "fp32" keeps fp32 partials (the
                                    Session / RuntimeConfig default)
  no_sync()                         accumulation = no_comm (engine.py:547-556)
  (root unit kept after forward)    keep_outermost_unsharded = True

Auto-wrap: every submodule the policy accepts becomes a unit (a
FlatParameter); the root keeps the remaining parameters (`flatparam.py:63-96`
assignment; a parameter reachable from two units raises
SharedParameterError).
"""
from __future__ import annotations

import contextlib
import enum
import functools
import warnings
from dataclasses import dataclass
from typing import Any, Callable, Iterable

import torch
import torch.nn as nn

from .comm import DeviceComm
from .layout import SharedParameterError, build_unit_layouts
from .plan import build_plan
from .runtime import (ACCUM_OFF, NRAF, PREFETCH_POST, PREFETCH_PRE, RAF, FSDPRuntime,
                      PreBackward, RuntimeConfig, UnitViews)


class ShardingStrategy(enum.Enum):
    FULL_SHARD = enum.auto()
    SHARD_GRAD_OP = enum.auto()
    NO_SHARD = enum.auto()
    HYBRID_SHARD = enum.auto()
    _HYBRID_SHARD_ZERO2 = enum.auto()


class BackwardPrefetch(enum.Enum):
    BACKWARD_PRE = enum.auto()
    BACKWARD_POST = enum.auto()


@dataclass
class MixedPrecision:
    param_dtype: torch.dtype | None = None
    reduce_dtype: torch.dtype | None = None
    buffer_dtype: torch.dtype | None = None


@dataclass
class CPUOffload:
    offload_params: bool = False


class ModuleWrapPolicy:
    """Wrap every submodule whose type is in `module_classes` (torch's
    ModuleWrapPolicy / transformer_auto_wrap_policy)."""

    def __init__(self, module_classes: Iterable[type]):
        self.classes = tuple(module_classes)

    def __call__(self, module: nn.Module) -> bool:
        return isinstance(module, self.classes)


def transformer_auto_wrap_policy(module: nn.Module, recurse: bool = False, nonwrapped_numel: int = 0,
                                 transformer_layer_cls: Iterable[type] = ()) -> bool:
    """torch-compatible functional policy (use with functools.partial)."""
    return isinstance(module, tuple(transformer_layer_cls))


def _policy_fn(policy) -> Callable[[nn.Module], bool] | None:
    if policy is None:
        return None
    if isinstance(policy, ModuleWrapPolicy):
        return policy
    if isinstance(policy, (set, list, tuple)):
        return ModuleWrapPolicy(policy)
    return lambda m: bool(policy(module=m, recurse=False, nonwrapped_numel=0))




def _map_tensors(fn, obj):
    if isinstance(obj, torch.Tensor):
        return fn([obj])[0]
    if isinstance(obj, (tuple, list)):
        ts = [o for o in obj if isinstance(o, torch.Tensor) and o.requires_grad]
        if not ts:
            return obj
        mapped = iter(fn(ts))
        out = [next(mapped) if (isinstance(o, torch.Tensor) and o.requires_grad) else o for o in obj]
        return type(obj)(out) if not hasattr(obj, "_fields") else type(obj)(*out)
    if isinstance(obj, dict):
        keys = [k for k, v in obj.items() if isinstance(v, torch.Tensor) and v.requires_grad]
        if not keys:
            return obj
        mapped = fn([obj[k] for k in keys])
        out = dict(obj)
        out.update(zip(keys, mapped))
        return type(obj)(out) if type(obj) is not dict else out
    return obj


class FullyShardedDataParallel(nn.Module):
    def __init__(self, module: nn.Module, process_group=None,
                 sharding_strategy: ShardingStrategy = ShardingStrategy.FULL_SHARD,
                 cpu_offload: CPUOffload | None = None, auto_wrap_policy=None,
                 backward_prefetch: BackwardPrefetch | None = BackwardPrefetch.BACKWARD_PRE,
                 mixed_precision: MixedPrecision | None = None, ignored_modules=None,
                 param_init_fn: Callable[[nn.Module], None] | None = None, device_id=None,
                 sync_module_states: bool = False, forward_prefetch: bool = False,
                 limit_all_gathers: bool = True, use_orig_params: bool = False,
                 ignored_states=None, device_mesh=None, *, hybrid_shard_size: int | None = None,
                 comm_backend: str = "ipc", num_slots: int | None = None, ag_ctas: int = 32, rs_ctas: int = 64,
                 optimizer: str = "adam", lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 optimizer_in_backward: bool = False, ag_engine: str = "ce", rs_engine: str = "ce",
                 tail_engine: str = "sm", ll_max_bytes: int = 6 << 20, opt_split_first: int = 2,
                 rate_limit: int | None | str = "auto", keep_outermost_unsharded: bool = True,
                 fused_cast_ag: bool = False, ar_in_pool: bool = True, w1_bf16_grad: bool = True,
                 opt_split_geom: bool | None = None, hybrid_stage2: str = "reduce"):
        super().__init__()
        if cpu_offload is not None and cpu_offload.offload_params:
            raise NotImplementedError("CPU offload is out of scope for the B200 runtime")
        if use_orig_params:
            warnings.warn("use_orig_params=True: the original parameters are exposed as views of "
                          "the unit's unsharded flat buffer during forward/backward (as with "
                          "use_orig_params); between steps only the flat shards exist "
                          "(flat_shards(), full_state_dict())")
        import torch.distributed as dist
        dist_on = dist.is_available() and dist.is_initialized()
        hybrid = sharding_strategy in (ShardingStrategy.HYBRID_SHARD, ShardingStrategy._HYBRID_SHARD_ZERO2)
        F_req = _shard_factor_from(process_group, device_mesh, hybrid_shard_size, hybrid, dist_on)
        pg = None if isinstance(process_group, tuple) else process_group
        world = dist.get_world_size(pg) if dist_on else 1
        rank = dist.get_rank(pg) if dist_on else 0
        if device_id is not None:
            torch.cuda.set_device(device_id)
        device = torch.device("cuda", torch.cuda.current_device())
        if sharding_strategy in (ShardingStrategy.FULL_SHARD, ShardingStrategy.SHARD_GRAD_OP):
            F = world
            if F_req is not None and F_req != world:
                raise ValueError(f"{sharding_strategy.name} shards over the whole world ({world}); the "
                                 f"device_mesh / process_group asks for groups of {F_req} (use HYBRID_SHARD)")
        elif sharding_strategy == ShardingStrategy.NO_SHARD:
            F = 1
        else:
            if F_req is None:
                raise ValueError("HYBRID_SHARD needs the shard-group size: pass hybrid_shard_size=F, a 2-D "
                                 "device_mesh (replicate, shard), or process_group=(shard_group, "
                                 "replicate_group) (collectives.py:63-72: shard groups of F consecutive "
                                 "ranks, replica groups strided by F)")
            F = F_req
        plan = build_plan(world, F)
        if isinstance(process_group, tuple) and dist_on:
            _check_group_tuple(process_group, plan, rank)
        raf = NRAF if sharding_strategy in (ShardingStrategy.SHARD_GRAD_OP,
                                            ShardingStrategy._HYBRID_SHARD_ZERO2) else RAF
        mp = mixed_precision
        mixed = mp is not None and mp.param_dtype == torch.bfloat16
        if mp is not None and mp.param_dtype not in (None, torch.bfloat16, torch.float32):
            raise ValueError("param_dtype must be bf16 or fp32 on the B200 runtime")
        reduce_low = mixed and (mp.reduce_dtype in (None, torch.bfloat16))
        bp = {None: None, BackwardPrefetch.BACKWARD_PRE: PREFETCH_PRE,
              BackwardPrefetch.BACKWARD_POST: PREFETCH_POST}[backward_prefetch]
        cfg = RuntimeConfig(mixed=mixed, reduce_in_low=reduce_low, reshard_after_forward=raf,
                            backward_prefetch=bp, forward_prefetch=forward_prefetch,
                            rate_limit=(2 if limit_all_gathers else None) if rate_limit == "auto" else rate_limit,
                            keep_outermost_unsharded=keep_outermost_unsharded, accumulation=ACCUM_OFF,
                            comm_backend=comm_backend, num_slots=num_slots, ag_ctas=ag_ctas, rs_ctas=rs_ctas,
                            optimizer=optimizer, lr=lr, betas=tuple(betas), eps=eps,
                            optimizer_in_backward=optimizer_in_backward,
                            ag_engine=ag_engine, rs_engine=rs_engine, tail_engine=tail_engine,
                            ll_max_bytes=ll_max_bytes, opt_split_first=opt_split_first,
                            fused_cast_ag=fused_cast_ag, ar_in_pool=ar_in_pool, w1_bf16_grad=w1_bf16_grad,
                            opt_split_geom=opt_split_geom, hybrid_stage2=hybrid_stage2)
        self.module = module
        self.plan = plan
        self.rank = rank
        policy = _policy_fn(auto_wrap_policy)
        ignored = set(ignored_modules or [])
        # ---- units: root + policy-accepted submodules, pre-order ----------
        unit_mods: list[nn.Module] = [module]
        for name, m in module.named_modules():
            if m is not module and policy is not None and m not in ignored and policy(m):
                unit_mods.append(m)
        owner_of: dict[int, int] = {id(m): 0 for m in module.modules()}
        for uid, um in enumerate(unit_mods[1:], start=1):
            for m in um.modules():
                owner_of[id(m)] = uid
        # parameter refs per unit in declaration order; shared params rejected
        names: list[list[str]] = [[] for _ in unit_mods]
        refs: list[list[tuple[nn.Module, str]]] = [[] for _ in unit_mods]
        shapes: list[tuple[str, tuple]] = []
        seen: dict[int, str] = {}
        for mname, m in module.named_modules(remove_duplicate=False):
            uid = owner_of[id(m)]
            for pname, p in list(m.named_parameters(recurse=False)):
                fq = f"{mname}.{pname}" if mname else pname
                if id(p) in seen:
                    first = seen[id(p)]
                    if owner_of_name(first, module, owner_of) != uid:
                        raise SharedParameterError(
                            f"parameter '{fq}' is shared with '{first}' across units; sharing a "
                            f"parameter across units is unsupported — merge the sharing layers "
                            f"into one unit, or use SHARD_GRAD_OP (NRAF)")
                    refs[uid].append((m, pname))      # alias within a unit: same view
                    continue
                seen[id(p)] = fq
                names[uid].append(fq)
                refs[uid].append((m, pname))
                shapes.append((fq, tuple(p.shape)))
        self._refs = refs
        self._alias: list[list[int]] = []
        for uid in range(len(unit_mods)):
            idx, amap = {}, []
            for (m, pname) in refs[uid]:
                p = m._parameters[pname]
                if id(p) not in idx:
                    idx[id(p)] = len(idx)
                amap.append(idx[id(p)])
            self._alias.append(amap)
        layouts = build_unit_layouts(shapes, names, F)
        self.layouts = layouts
        # ---- communicator + runtime ---------------------------------------
        comm = None
        pgs = {}
        if world > 1 and comm_backend == "ipc":
            comm = DeviceComm.create(FSDPRuntime.pool_bytes_for(layouts, plan, cfg), max_ctas=max(ag_ctas, rs_ctas),
                                     group=pg,
                                     nvls_group=plan.shard_factor if ag_engine == "nvls" else None)
        elif world > 1:
            pgs = _nccl_groups(plan, rank)
        self.comm = comm
        self.rt = FSDPRuntime(layouts, plan, rank, cfg, comm=comm, process_groups=pgs, device=device)
        # ---- materialise unit by unit: flatten + shard, then drop originals
        for uid, um in enumerate(unit_mods):
            params = []
            for (m, pname), a in zip(refs[uid], self._alias[uid]):
                if a < len(params):
                    continue
                p = m._parameters[pname]
                if p.is_meta:
                    mods = [mm for mm in um.modules() if owner_of[id(mm)] == uid]
                    for mm in mods:
                        mm.to_empty(device=device, recurse=False)
                        if param_init_fn is not None:
                            param_init_fn(mm)
                        elif hasattr(mm, "reset_parameters"):
                            mm.reset_parameters()
                    p = m._parameters[pname]
                params.append(p)
            if params:
                self.rt.load_unit_values(uid, params, sync_src=0 if sync_module_states else None)
            for (m, pname) in refs[uid]:
                if pname in m._parameters:
                    del m._parameters[pname]
        module.to(device)
        if sync_module_states and world > 1:
            from .dist_util import broadcast_
            for b in module.buffers():
                broadcast_(b.data, src=0)
        if mixed and (mp.buffer_dtype is not None):
            for m in module.modules():
                for bn, b in list(m._buffers.items()):
                    if b is not None and b.is_floating_point():
                        m._buffers[bn] = b.to(mp.buffer_dtype)
        torch.cuda.synchronize()
        self._unit_mods = unit_mods
        self._anchors = [torch.zeros((), device=device, requires_grad=True) for _ in unit_mods]
        self._handles = []
        for uid, um in enumerate(unit_mods):
            self._handles.append(um.register_forward_pre_hook(functools.partial(self._pre_fwd, uid)))
            self._handles.append(um.register_forward_hook(functools.partial(self._post_fwd, uid)))
        self._defer = False
        self._new_micro = True
        self.rt.on_end_backward = self._end_backward
        self.mixed = mixed

    # ------------------------------------------------------------ hooks ---
    def _install(self, uid: int, flat: torch.Tensor) -> None:
        if flat.numel() == 0 or not self._refs[uid]:
            return
        views = UnitViews.apply(self._anchors[uid], flat, self.rt, uid)
        for (m, pname), a in zip(self._refs[uid], self._alias[uid]):
            setattr(m, pname, views[a])

    def _pre_fwd(self, uid, module, args):
        rt = self.rt
        if uid == 0:
            if self._new_micro:
                self._new_micro = False
                rt.begin_micro(final=not self._defer)
                rt.defer_reduce = self._defer
            rt.begin_forward_pass()
        pos = rt.record_forward(uid)
        flat = rt.ensure_unsharded(uid)
        rt.forward_prefetch_after(pos)
        self._install(uid, flat)
        return None

    def _post_fwd(self, uid, module, args, output):
        rt = self.rt
        rt.post_order.append(uid)
        rt.close_window(uid)
        rt.sample_activations()
        if torch.is_grad_enabled():
            output = _map_tensors(lambda ts: PreBackward.apply(rt, uid, *ts), output)
            rt.release_use(uid, "forward", 0)
        else:
            # no backward will follow (eval / no_grad): nothing is kept unsharded
            rt.release_use(uid, "backward", None)
            if uid == 0:
                self._new_micro = True
        return output

    def _end_backward(self) -> None:
        self._new_micro = True

    # -------------------------------------------------------------- api ---
    def forward(self, *args, **kwargs):
        with self.rt.saved_tensor_hooks():
            return self.module(*args, **kwargs)

    @contextlib.contextmanager
    def no_sync(self):
        """Accumulate unsharded gradients locally without communication; the
        first backward outside the context reduces them (engine.py:547-556)."""
        prev = self._defer
        self._defer = True
        try:
            yield
        finally:
            self._defer = prev

    def optimizer(self, lr: float | None = None, betas=None, eps: float | None = None):
        return ShardedOptimizer(self, lr, betas, eps)

    def step(self, scale: float | None = None) -> None:
        self.rt.optimizer_step(scale)
        self.rt.begin_step()

    def check_errors(self) -> None:
        """Synchronise and raise DeadlockError if a cross-GPU collective wait
        timed out on this rank or a peer aborted (collectives.py:461-483).
        Without this call the runtime raises at the next optimizer step; the
        optimizer never applies an update once the error word is set."""
        self.rt.raise_if_aborted(sync=True)

    def close(self) -> None:
        """Release the communicator's pool and IPC mappings."""
        for h in self._handles:
            h.remove()
        self._handles = []
        if self.comm is not None:
            self.comm.close()
            self.comm = None

    def flat_shards(self) -> list[torch.Tensor]:
        return [u.master for u in self.rt.units]

    def full_state_dict(self) -> dict[str, torch.Tensor]:
        """Gather fp32 parameters (engine.py:824-834 gather_full_params):
        all-gather every unit's master shard within the sharded group, then
        unflatten into the original shapes (kernels)."""
        from . import kernels
        out = {}
        for uid, lay in enumerate(self.layouts):
            flat = self.rt.gather_master(uid)     # this library's all-gather (ipc backend)
            tensors = [torch.empty(o.shape, dtype=torch.float32, device=flat.device) for o in lay.originals]
            kernels.unflatten(flat, tensors, lay.offsets)
            for o, t in zip(lay.originals, tensors):
                out[o.name] = t
        return out


    def load_full_state_dict(self, sd: dict[str, torch.Tensor]) -> None:
        """Inverse of full_state_dict: flatten each unit's original tensors and
        keep this rank's shard (the init path, deferred_init.py:156-176);
        the bf16 copy is refreshed.  Optimizer state is left unchanged."""
        for uid, lay in enumerate(self.layouts):
            if lay.psi:
                self.rt.load_unit_values(uid, [sd[o.name] for o in lay.originals])
        torch.cuda.synchronize()

    def sharded_state_dict(self) -> dict:
        """This rank's shards + optimizer state (a checkpoint that needs no
        gather); restore with load_sharded_state_dict on the same plan."""
        rt = self.rt
        out = {"world_size": self.plan.world_size, "shard_factor": self.plan.shard_factor,
               "rank": self.rank, "adam_steps": rt.adam_steps,
               "psi": [lay.psi for lay in self.layouts], "units": []}
        for u in rt.units:
            d = {"master": u.master.detach().clone().cpu()}
            if u.exp_avg is not None:
                d["exp_avg"] = u.exp_avg.detach().clone().cpu()
                d["exp_avg_sq"] = u.exp_avg_sq.detach().clone().cpu()
            out["units"].append(d)
        return out

    def load_sharded_state_dict(self, sd: dict) -> None:
        rt = self.rt
        if (sd["world_size"], sd["shard_factor"], sd["rank"]) != \
                (self.plan.world_size, self.plan.shard_factor, self.rank) or \
                sd["psi"] != [lay.psi for lay in self.layouts]:
            raise ValueError("sharded state dict was saved with a different plan/layout/rank")
        from . import kernels
        for u, d in zip(rt.units, sd["units"]):
            u.master.copy_(d["master"])
            if u.exp_avg is not None and "exp_avg" in d:
                u.exp_avg.copy_(d["exp_avg"])
                u.exp_avg_sq.copy_(d["exp_avg_sq"])
            if u.low is not None:
                kernels.cast(u.master, u.low)
        rt.adam_steps = int(sd["adam_steps"])
        torch.cuda.synchronize()

    def memory_ledger(self) -> dict:
        """Per-category residency and peaks of this rank (memsim.py:113-185),
        with torch's allocator statistics and the symmetric pool size beside it."""
        st = torch.cuda.memory_stats(self.rt.device)
        out = self.rt.ledger.snapshot()
        out["torch"] = {"allocated_peak_bytes": int(st.get("allocated_bytes.all.peak", 0)),
                        "reserved_peak_bytes": int(st.get("reserved_bytes.all.peak", 0)),
                        "num_alloc_retries": int(st.get("num_alloc_retries", 0))}
        out["symmetric_pool_bytes"] = self.comm.pool_bytes if self.comm is not None else 0
        return out

    def inject_fault(self, kind: str, step: int | None = None) -> None:
        """Verify-sensitivity faults (cli.py:568-574): "misordered-reduction"
        hands every reduce-scatter member the neighbouring chunk
        (collectives.py:296); "inf-grad" writes inf into unit 0's gradient on
        this rank at optimizer step `step` (engine.py:541-543)."""
        if kind == "misordered-reduction":
            if self.comm is not None:
                self.comm.set_fault(True)
            elif self.plan.shard_factor > 1:
                raise NotImplementedError("misordered-reduction needs the ipc backend")
        elif kind == "inf-grad":
            self.rt.inject_inf.add(self.rt.step_count if step is None else int(step))
        else:
            raise ValueError(f"unknown fault {kind!r} (misordered-reduction, inf-grad)")

    def trace_lines(self) -> list[str]:
        """The reference's trace format (memsim.py:50-61) for this rank."""
        return self.rt.trace.lines(self.rank)


def owner_of_name(fq: str, root: nn.Module, owner_of: dict) -> int:
    mod_name, _, _ = fq.rpartition(".")
    m = root.get_submodule(mod_name) if mod_name else root
    return owner_of[id(m)]


_GROUP_CACHE: dict = {}


def _nccl_groups(plan, rank):
    import torch.distributed as dist
    key = (plan.world_size, plan.shard_factor)
    if key not in _GROUP_CACHE:
        shard = {g: dist.new_group(list(g)) for g in plan.sharded_groups}
        rep = {g: dist.new_group(list(g)) for g in plan.replicated_groups}
        _GROUP_CACHE[key] = (shard, rep)
    shard, rep = _GROUP_CACHE[key]
    return {"shard": shard[plan.sharded_group_of(rank)], "replicate": rep[plan.replicated_group_of(rank)]}


def _shard_factor_from(process_group, device_mesh, hybrid_shard_size, hybrid: bool, dist_on: bool):
    """Shard-group size F requested by torch-FSDP's ways of naming it:
    hybrid_shard_size, a DeviceMesh (1-D: shard over it; 2-D: (replicate,
    shard), mesh_dim_names honoured) or a (shard_group, replicate_group)
    process-group tuple.  None if nothing names it.  Only the reference's
    group convention is accepted (collectives.py:63-72, :89-96): shard groups
    of F consecutive ranks, replica groups strided by F."""
    cands = []
    if hybrid_shard_size is not None:
        cands.append(int(hybrid_shard_size))
    if device_mesh is not None:
        mesh = device_mesh.mesh if hasattr(device_mesh, "mesh") else torch.as_tensor(device_mesh)
        mesh = torch.as_tensor(mesh).cpu()
        names = tuple(getattr(device_mesh, "mesh_dim_names", None) or ())
        if mesh.dim() == 1:
            F = mesh.numel()
            canon = torch.arange(F)
        elif mesh.dim() == 2:
            if names and names[0] == "shard":      # (shard, replicate) order: transpose
                mesh = mesh.t()
            R, F = mesh.shape
            canon = torch.arange(R * F).view(R, F)
        else:
            raise ValueError("device_mesh must be 1-D (shard) or 2-D (replicate, shard)")
        if not torch.equal(mesh.to(torch.int64), canon):
            raise ValueError(f"device_mesh {mesh.tolist()} does not follow the shard-group convention "
                             f"(rows of consecutive ranks = shard groups): collectives.py:89-96")
        cands.append(int(F))
    if isinstance(process_group, tuple):
        if len(process_group) != 2:
            raise ValueError("process_group tuple must be (shard_group, replicate_group)")
        if dist_on:
            import torch.distributed as dist
            cands.append(dist.get_world_size(process_group[0]))
    if len(set(cands)) > 1:
        raise ValueError(f"inconsistent shard-group sizes {cands} (hybrid_shard_size / device_mesh / "
                         f"process_group)")
    if cands and not hybrid and device_mesh is None and not isinstance(process_group, tuple):
        return None                               # hybrid_shard_size is ignored by FULL/NO_SHARD
    return cands[0] if cands else None


def _check_group_tuple(groups, plan, rank) -> None:
    import torch.distributed as dist
    shard = tuple(dist.get_process_group_ranks(groups[0]))
    rep = tuple(dist.get_process_group_ranks(groups[1]))
    if shard != tuple(plan.sharded_group_of(rank)) or rep != tuple(plan.replicated_group_of(rank)):
        raise ValueError(f"process groups {shard} / {rep} do not match the shard/replica convention "
                         f"{plan.sharded_group_of(rank)} / {plan.replicated_group_of(rank)} "
                         f"(collectives.py:89-96)")


class ShardedGradScaler:
    """torch.distributed.fsdp.ShardedGradScaler-shaped loss scaler over the
    runtime's device-side verdict (engine.py:118-145, :563-589):

        scaler.scale(loss).backward(); scaler.step(opt); scaler.update()

    step() unscales every rank's gradient shard, all-reduces the found_inf
    flag across the world and runs the optimizer with an on-device skip (no
    host sync); update() reads the verdict once and backs off / grows the
    scale exactly like the reference."""

    def __init__(self, init_scale: float = 65536.0, growth_factor: float = 2.0,
                 backoff_factor: float = 0.5, growth_interval: int = 2000, enabled: bool = True):
        self.scale_value = float(init_scale)
        self.growth_factor, self.backoff_factor = growth_factor, backoff_factor
        self.growth_interval = growth_interval
        self.enabled = enabled
        self._tracker = 0
        self._pending: FullyShardedDataParallel | None = None
        self.steps_skipped = 0

    def scale(self, loss: torch.Tensor) -> torch.Tensor:
        return loss * self.scale_value if self.enabled else loss

    def step(self, optimizer: "ShardedOptimizer") -> None:
        if not self.enabled:
            optimizer.step()
            return
        optimizer.step(scale=self.scale_value)
        self._pending = optimizer.fsdp

    def update(self) -> bool:
        """Returns True if the last step was skipped (non-finite gradients)."""
        if not self.enabled or self._pending is None:
            return False
        rt = self._pending.rt
        found = bool(rt.found_inf_world.item() > 0.0)
        if found:
            # an aborted communicator also forces the verdict: surface it as
            # DeadlockError (collectives.py:476-482), not as an inf step
            rt.raise_if_aborted(sync=True)
            rt.undo_adam_t()
            self.scale_value *= self.backoff_factor
            self._tracker = 0
            self.steps_skipped += 1
        else:
            self._tracker += 1
            if self._tracker >= self.growth_interval:
                self.scale_value *= self.growth_factor
                self._tracker = 0
        self._pending = None
        return found


class ShardedOptimizer:
    """torch.optim-like handle: step() runs the fused sharded optimizer."""

    def __init__(self, fsdp: FullyShardedDataParallel, lr=None, betas=None, eps=None):
        cfg = fsdp.rt.cfg
        if lr is not None:
            cfg.lr = lr
        if betas is not None:
            cfg.betas = tuple(betas)
        if eps is not None:
            cfg.eps = eps
        self.fsdp = fsdp

    def step(self, scale: float | None = None) -> None:
        self.fsdp.step(scale)

    def zero_grad(self, set_to_none: bool = True) -> None:
        pass   # reduced grads are overwritten by the first reduce of a step
