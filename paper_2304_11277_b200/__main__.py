"""Command line front end (the reference's `shardsim run/verify/dump-plan`,
cli.py:428-731, driving the GPU runtime).

    python -m paper_2304_11277_b200 dump-plan --model gpt1.3b --shard-factor 8
    torchrun --nproc-per-node 8 -m paper_2304_11277_b200 run --model gpt1.3b --steps 20
    torchrun --nproc-per-node 2 -m paper_2304_11277_b200 verify --steps 3

`run` prints one JSON record per step (schema: step, loss, ms, tflops_per_gpu).
`verify` trains the tiny GPT sharded (fp32, FULL_SHARD) and, on every rank,
an unsharded torch copy with torch.optim.Adam on the global batch, and checks
the gathered parameters agree (exit 1 if they do not: the analogue of
shardsim verify's tolerance check, cli.py:469-519).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time


def _models():
    from .workloads import CONFIGS, GPT, T5, T5_CONFIGS, Block, T5DecoderBlock, T5EncoderBlock
    out = {k: (lambda c=c: GPT(c), {Block}, c) for k, c in CONFIGS.items()}
    out.update({k: (lambda c=c: T5(c), {T5EncoderBlock, T5DecoderBlock}, c)
                for k, c in T5_CONFIGS.items()})
    return out


def cmd_dump_plan(a) -> int:
    import torch
    from .layout import build_unit_layouts, dump_plan_lines
    make, wrap, _ = _models()[a.model]
    with torch.device("meta"):
        m = make()
    units, owner = [[]], {}
    blocks = [x for x in m.modules() if isinstance(x, tuple(wrap))]
    for i, b in enumerate(blocks, start=1):
        units.append([])
        for sub in b.modules():
            owner[id(sub)] = i
    shapes = []
    for mn, mod in m.named_modules():
        for pn, p in mod.named_parameters(recurse=False):
            fq = f"{mn}.{pn}" if mn else pn
            units[owner.get(id(mod), 0)].append(fq)
            shapes.append((fq, tuple(p.shape)))
    for line in dump_plan_lines(build_unit_layouts(shapes, units, a.shard_factor)):
        print(line)
    return 0


def _dist():
    from .dist_util import init_from_env
    rank, world, _ = init_from_env()
    return rank, world


def cmd_run(a) -> int:
    import torch
    from .fsdp import (BackwardPrefetch, FullyShardedDataParallel, MixedPrecision,
                       ModuleWrapPolicy, ShardingStrategy)
    from .workloads import param_init_fn
    rank, world = _dist()
    make, wrap, cfg = _models()[a.model]
    torch.manual_seed(a.seed)
    with torch.device("meta"):
        m = make()
    fsdp = FullyShardedDataParallel(
        m, sharding_strategy=ShardingStrategy[a.strategy], auto_wrap_policy=ModuleWrapPolicy(wrap),
        backward_prefetch=BackwardPrefetch[a.backward_prefetch] if a.backward_prefetch else None,
        mixed_precision=MixedPrecision(param_dtype=torch.bfloat16) if a.mixed else None,
        forward_prefetch=a.forward_prefetch, limit_all_gathers=not a.no_limiter,
        param_init_fn=param_init_fn, hybrid_shard_size=a.hybrid_shard_size, lr=a.lr)
    opt = fsdp.optimizer()
    g = torch.Generator().manual_seed(a.seed + 1 + rank)
    if hasattr(cfg, "seq"):
        inputs = lambda: tuple(torch.randint(0, cfg.vocab, (a.micro, cfg.seq), generator=g).cuda()  # noqa: E731
                               for _ in range(2))
        flops = cfg.flops_per_token() * a.micro * cfg.seq
    else:
        inputs = lambda: (torch.randint(0, cfg.vocab, (a.micro, cfg.enc_seq), generator=g).cuda(),  # noqa: E731
                          torch.randint(0, cfg.vocab, (a.micro, cfg.dec_seq), generator=g).cuda(),
                          torch.randint(0, cfg.vocab, (a.micro, cfg.dec_seq), generator=g).cuda())
        flops = cfg.flops_per_sample() * a.micro
    for step in range(a.steps):
        t0 = time.perf_counter()
        loss = fsdp(*inputs())
        loss.backward()
        opt.step()
        lv = loss.item()
        dt = time.perf_counter() - t0
        if rank == 0:
            print(json.dumps({"schema": 1, "step": step, "loss": lv, "ms": round(dt * 1e3, 3),
                              "tflops_per_gpu": round(flops / dt / 1e12, 2)}), flush=True)
    fsdp.close()
    return 0


def cmd_verify(a) -> int:
    import torch
    import torch.distributed as dist
    from .fsdp import FullyShardedDataParallel, ModuleWrapPolicy
    from .workloads import CONFIGS, GPT, Block, init_gpt_
    rank, world = _dist()
    torch.backends.cuda.matmul.allow_tf32 = False
    cfg = CONFIGS["tiny"]
    fsdp = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=a.seed),
                                    auto_wrap_policy=ModuleWrapPolicy({Block}), lr=a.lr)
    ref = init_gpt_(GPT(cfg), seed=a.seed).cuda()
    opt_ref = torch.optim.Adam(ref.parameters(), lr=a.lr, foreach=False)
    opt = fsdp.optimizer()
    g = torch.Generator().manual_seed(a.seed + 7)
    worst = 0.0
    for step in range(a.steps):
        xs = torch.randint(0, cfg.vocab, (world * a.micro, 64), generator=g).cuda()
        ys = torch.randint(0, cfg.vocab, (world * a.micro, 64), generator=g).cuda()
        sl = slice(rank * a.micro, (rank + 1) * a.micro)
        fsdp(xs[sl], ys[sl]).backward()
        opt.step()
        opt_ref.zero_grad()
        # the global mean of per-rank means == the FSDP gradient (÷ W post-reduction)
        loss = sum(ref(xs[r * a.micro:(r + 1) * a.micro], ys[r * a.micro:(r + 1) * a.micro])
                   for r in range(world)) / world
        loss.backward()
        opt_ref.step()
        sd = fsdp.full_state_dict()
        d = max(float((sd[n] - p.detach()).abs().max()) for n, p in ref.named_parameters())
        worst = max(worst, d)
        if rank == 0:
            print(json.dumps({"step": step, "max_param_delta": d}), flush=True)
    ok = worst <= a.tol
    if rank == 0:
        print(json.dumps({"verify": "PASS" if ok else "FAIL", "max_param_delta": worst, "tol": a.tol}))
    fsdp.close()
    if world > 1:
        dist.barrier()
    return 0 if ok else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2304_11277_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("dump-plan")
    p.add_argument("--model", default="tiny")
    p.add_argument("--shard-factor", type=int, default=1)
    p = sub.add_parser("run")
    p.add_argument("--model", default="tiny")
    p.add_argument("--strategy", default="FULL_SHARD")
    p.add_argument("--hybrid-shard-size", type=int, default=None)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--micro", type=int, default=4)
    p.add_argument("--lr", type=float, default=1e-4)
    p.add_argument("--seed", type=int, default=int(os.environ.get("FSDP_SEED", 0)))
    p.add_argument("--mixed", action="store_true", default=True)
    p.add_argument("--backward-prefetch", default="BACKWARD_PRE")
    p.add_argument("--forward-prefetch", action="store_true")
    p.add_argument("--no-limiter", action="store_true")
    p = sub.add_parser("verify")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--micro", type=int, default=2)
    p.add_argument("--lr", type=float, default=1e-3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--tol", type=float, default=1e-4)
    a = ap.parse_args(argv)
    return {"dump-plan": cmd_dump_plan, "run": cmd_run, "verify": cmd_verify}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
