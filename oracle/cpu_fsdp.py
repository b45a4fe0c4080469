"""ORACLE (test infrastructure only) — the reference's FSDP step on the CPU,
for bench.py's `cpu_baseline` leg and the `--impl reference` arm.

The shardsim algorithm (shardsim_port.py) applied to a GPT-style module:
flat buffers per unit (numpy, flatparam.py:63-96), the module's parameters
installed as zero-copy views of those buffers (flatparam.py:159-164), one
forward/backward on the CPU (torch, fp32 — shardsim's own model is a numpy
MLP, so the model math here is plain torch CPU), gradient write-back
(flatparam.py:167-191), the W-rank reduction (collectives.py:273-297 via
`reduce_unit`, engine.py:771-820) and Adam on the shards (numerics.py:273-285).
For W > 1 the ranks are simulated in one process exactly as shardsim does
(`pkg/README.md:11-14`): every rank's slice is computed in turn.
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import shardsim_port as sp

_CHUNK = 1 << 22      # elements per thread-pool task of the elementwise numpy work


def adam_step_threaded(pool, param, grad, state, lr) -> None:
    """sp.adam_step (numerics.py:273-285) applied chunk by chunk on a thread
    pool: every element's arithmetic is the same numpy expression, so the
    result is bit-identical to one call over the whole shard; numpy releases
    the GIL inside the ufuncs, so the chunks run on all host cores."""
    n = param.size
    t = state["t"]
    m, v = state["m"], state["v"]

    def one(a):
        b = min(n, a + _CHUNK)
        st = {"m": m[a:b], "v": v[a:b], "t": t}
        sp.adam_step(param[a:b], grad[a:b], st, lr=lr)
        m[a:b] = st["m"]
        v[a:b] = st["v"]

    list(pool.map(one, range(0, n, _CHUNK)))
    state["t"] = t + 1


def _units_of(model, block_cls):
    """Root + every `block_cls` submodule, declaration order (auto-wrap)."""
    names = [[]]
    unit_of_mod = {}
    blocks = [m for m in model.modules() if isinstance(m, block_cls)]
    for i, b in enumerate(blocks, start=1):
        for m in b.modules():
            unit_of_mod[id(m)] = i
        names.append([])
    shapes = []
    for mname, m in model.named_modules():
        for pname, p in m.named_parameters(recurse=False):
            fq = f"{mname}.{pname}" if mname else pname
            names[unit_of_mod.get(id(m), 0)].append(fq)
            shapes.append((fq, tuple(p.shape)))
    return shapes, names


class CPUFSDP:
    """shardsim-style W-rank FSDP over one CPU process for a torch module."""

    def __init__(self, model, block_cls, world: int = 1, shard_factor: int | None = None,
                 lr: float = 1e-3, threads: int | None = None):
        import torch
        self.torch = torch
        self.threads = threads or os.cpu_count() or 1
        torch.set_num_threads(self.threads)
        self.pool = ThreadPoolExecutor(max_workers=self.threads)
        self.model = model
        self.plan = sp.Plan(world, shard_factor or world)
        shapes, names = _units_of(model, block_cls)
        self.layouts = sp.build_unit_layouts(shapes, names, self.plan.shard_factor)
        params = dict(model.named_parameters())
        values = {k: v.detach().float().numpy() for k, v in params.items()}
        self.shards = [[sp.shard(sp.flatten(values, lay, np.float32), lay, sp.shard_index(self.plan, r))
                        for lay in self.layouts] for r in range(world)]
        self.states = [[sp.adam_init(lay.shard_numel, np.float32) for lay in self.layouts]
                       for _ in range(world)]
        self.lr = lr
        self._mods = {}
        for mname, m in model.named_modules():
            for pname, _ in m.named_parameters(recurse=False):
                self._mods[f"{mname}.{pname}" if mname else pname] = (m, pname)

    def _install(self, rank: int):
        """Unshard every unit (all-gather of the group's shards) and point the
        module's parameters at views of the gathered flat buffers."""
        torch = self.torch
        g = self.plan.sharded_group_of(rank)
        for u, lay in enumerate(self.layouts):
            flat = sp.all_gather([self.shards[q][u] for q in g])
            for o in lay.originals:
                m, pname = self._mods[o.name]
                t = torch.from_numpy(flat[o.offset:o.offset + o.numel]).view(o.shape)
                m._parameters[pname] = torch.nn.Parameter(t)

    def step(self, batches_per_rank) -> float:
        """One optimizer step; batches_per_rank[r] = (x, y) torch CPU tensors.

        The W-rank reduction is accumulated while the simulated ranks run, in
        exactly the fabric's order (collectives.py:273-297 ascending within
        each sharded group, engine.py:899-917 ascending across groups), so
        only one partial sum per group is resident instead of W gradients."""
        W, F = self.plan.world_size, self.plan.shard_factor
        nu = len(self.layouts)
        partial = {}                       # (group index, unit) -> running fp32 sum
        losses = []
        for r in range(W):
            self._install(r)
            x, y = batches_per_rank[r]
            self.model.zero_grad(set_to_none=True)
            loss = self.model(x, y)
            loss.backward()
            losses.append(float(loss.detach()))
            grads = {n: p.grad.numpy() for n, p in self.model.named_parameters()
                     if p.grad is not None}
            gi = r // F
            for u, lay in enumerate(self.layouts):
                flat = sp.writeback_grad(lay, grads, np.float32)[0]
                key = (gi, u)
                partial[key] = (np.zeros_like(flat) if key not in partial else partial[key]) + flat
        for u, lay in enumerate(self.layouts):
            total = None
            for gi in range(W // F):                       # ascending across groups
                p = partial.pop((gi, u))
                total = (np.zeros_like(p) + p) if total is None else total + p
            red = total / np.float32(W)
            for r in range(W):
                k = sp.shard_index(self.plan, r)
                g = red[k * lay.shard_numel:(k + 1) * lay.shard_numel]
                adam_step_threaded(self.pool, self.shards[r][u], np.zeros_like(g) + g, self.states[r][u],
                                   self.lr)
        return float(np.mean(losses))


def time_cpu_steps(model, block_cls, batches_fn, steps: int, warmup: int, world: int = 1,
                   threads: int | None = None) -> dict:
    """Time `steps` CPU FSDP steps after `warmup`; returns seconds per step."""
    runner = CPUFSDP(model, block_cls, world=world, threads=threads)
    for i in range(warmup):
        runner.step(batches_fn(i))
    t0 = time.perf_counter()
    for i in range(steps):
        runner.step(batches_fn(warmup + i))
    dt = (time.perf_counter() - t0) / max(1, steps)
    return {"sec_per_step": dt, "threads": runner.threads}
