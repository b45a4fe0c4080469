"""World-size-2 CPU/gloo restatement of the FSDP step:
two real processes, each holding its flat shard, all-gather / reduce-scatter
over gloo, forward/backward of the tiny GPT on its slice, write-back, / W,
Adam on the shard.  Checked bit-for-bit against the oracle's single-process
multi-rank simulation (oracle/cpu_fsdp.py) — for W = 2 the sum order is
irrelevant (a + b), so gloo's unspecified order cannot break exactness.
Also exercises the plan's group descriptors across real ranks."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(2)
    try:
        from oracle import shardsim_port as sp
        from oracle.cpu_fsdp import _units_of
        from paper_2304_11277_b200.layout import build_unit_layouts
        from paper_2304_11277_b200.plan import build_plan
        from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_
        cfg = CONFIGS["tiny"]
        model = init_gpt_(GPT(cfg), seed=0)
        shapes, names = _units_of(model, Block)
        plan = build_plan(world, world)
        assert plan.sharded_group_of(rank) == tuple(range(world))
        lays = build_unit_layouts(shapes, names, world)
        vals = {k: v.detach().numpy().copy() for k, v in model.named_parameters()}
        shards = [torch.from_numpy(sp.shard(sp.flatten(vals, l, np.float32), l, rank)) for l in lays]
        # all-gather every unit, install views
        mods = {}
        for mn, m in model.named_modules():
            for pn, _ in m.named_parameters(recurse=False):
                mods[f"{mn}.{pn}" if mn else pn] = (m, pn)
        for l, s in zip(lays, shards):
            flat = torch.empty(l.psi)
            dist.all_gather_into_tensor(flat, s)
            for o in l.originals:
                m, pn = mods[o.name]
                m._parameters[pn] = torch.nn.Parameter(flat[o.offset:o.offset + o.numel].view(o.shape))
        g = torch.Generator().manual_seed(7)
        xs = [(torch.randint(0, cfg.vocab, (1, 64), generator=g),
               torch.randint(0, cfg.vocab, (1, 64), generator=g)) for _ in range(world)]
        loss = model(*xs[rank])
        loss.backward()
        grads = {n: p.grad.numpy() for n, p in model.named_parameters()}
        out = []
        for l, s in zip(lays, shards):
            fg = torch.from_numpy(sp.writeback_grad(l, grads, np.float32)[0])
            red = torch.empty(l.shard_numel)
            dist.reduce_scatter_tensor(red, fg)
            acc = red.numpy() / np.float32(world)
            p = s.numpy().copy()
            sp.adam_step(p, np.zeros_like(p) + acc, sp.adam_init(p.size, np.float32))
            out.append(p)
        q.put((rank, [o.tobytes() for o in out], float(loss)))
    finally:
        dist.destroy_process_group()


def test_gloo_w2_step_matches_oracle_simulation():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        r, shards, loss = q.get(timeout=300)
        got[r] = shards
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # oracle: both ranks simulated in one process
    sys.path.insert(0, ROOT)
    from oracle.cpu_fsdp import CPUFSDP
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_
    cfg = CONFIGS["tiny"]
    torch.set_num_threads(2)
    sim = CPUFSDP(init_gpt_(GPT(cfg), seed=0), Block, world=world, threads=2)
    g = torch.Generator().manual_seed(7)
    xs = [(torch.randint(0, cfg.vocab, (1, 64), generator=g),
           torch.randint(0, cfg.vocab, (1, 64), generator=g)) for _ in range(world)]
    sim.step(xs)
    for r in range(world):
        for u, b in enumerate(got[r]):
            assert sim.shards[r][u].tobytes() == b, (r, u)
