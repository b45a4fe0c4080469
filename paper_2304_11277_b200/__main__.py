"""Command line front end (the reference's `shardsim run/verify/dump-plan`,
cli.py:428-731, driving the GPU runtime).

    python -m paper_2304_11277_b200 dump-plan --model gpt1.3b --shard-factor 8
    torchrun --nproc-per-node 8 -m paper_2304_11277_b200 run --model gpt1.3b --steps 20
    torchrun --nproc-per-node 2 -m paper_2304_11277_b200 verify --steps 3

    torchrun --nproc-per-node 4 -m paper_2304_11277_b200 sweep --axis F=1,2,4 --axis raf=RAF,NRAF

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


EXIT_VERIFY_FAIL, EXIT_CONFIG = 1, 2          # cli.py:40-42


def _verify_fsdp(a, seed, **kw):
    from .fsdp import BackwardPrefetch, FullyShardedDataParallel, ModuleWrapPolicy, ShardingStrategy
    from .workloads import CONFIGS, GPT, Block, init_gpt_
    cfg = CONFIGS["tiny"]
    strat = ShardingStrategy[a.strategy]
    extra = {}
    if a.serialized:
        # one unit materialised at a time: rate_limit 1, no prefetch, RAF,
        # no keep-outermost (the peak formula's premise, cli.py:538-551)
        extra = dict(backward_prefetch=None, forward_prefetch=False, rate_limit=1,
                     keep_outermost_unsharded=False)
    return FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=seed), sharding_strategy=strat,
                                    auto_wrap_policy=ModuleWrapPolicy({Block}), lr=a.lr,
                                    hybrid_shard_size=a.hybrid_shard_size, **extra, **kw), cfg


def cmd_verify(a) -> int:
    """cli.py:469-590: sharded training vs a local (unsharded) oracle, exit 1
    on any parameter or loss delta beyond tolerance, or on a skip
    divergence; --inject-fault corrupts the sharded run to show the check is
    sensitive (misordered-reduction: collectives.py:296; inf-grad:
    engine.py:541-543 at step min(1, steps-1) on rank 0).  --serialized adds
    the peak-parameter-memory formula check (flatparam.py:198-235)."""
    import math

    import torch
    from .dist_util import all_reduce_
    from .ledger import peak_param_bytes
    from .workloads import CONFIGS, GPT, init_gpt_
    rank, world = _dist()
    torch.backends.cuda.matmul.allow_tf32 = False
    fsdp, cfg = _verify_fsdp(a, a.seed)
    if a.inject_fault == "misordered-reduction":
        fsdp.inject_fault("misordered-reduction")
    elif a.inject_fault == "inf-grad" and rank == 0:
        fsdp.inject_fault("inf-grad", step=min(1, a.steps - 1))
    ref = init_gpt_(GPT(cfg), seed=a.seed).cuda()
    opt_ref = torch.optim.Adam(ref.parameters(), lr=a.lr, foreach=False)
    opt = fsdp.optimizer()
    g = torch.Generator().manual_seed(a.seed + 7)
    ok = True
    worst = 0.0
    fsdp.rt.ledger.reset_peaks()
    for step in range(a.steps):
        xs = torch.randint(0, cfg.vocab, (world * a.micro, 64), generator=g).cuda()
        ys = torch.randint(0, cfg.vocab, (world * a.micro, 64), generator=g).cuda()
        sl = slice(rank * a.micro, (rank + 1) * a.micro)
        loss = fsdp(xs[sl], ys[sl])
        loss.backward()
        opt.step()
        opt_ref.zero_grad()
        # the global mean of per-rank means == the FSDP gradient (÷ W post-reduction)
        lref = sum(ref(xs[r * a.micro:(r + 1) * a.micro], ys[r * a.micro:(r + 1) * a.micro])
                   for r in range(world)) / world
        lref.backward()
        opt_ref.step()
        lsh = loss.detach().float().reshape(1).clone()
        if world > 1:
            all_reduce_(lsh)
            lsh /= world
        sd = fsdp.full_state_dict()
        d = max(float((sd[n] - p.detach()).abs().max()) for n, p in ref.named_parameters())
        dl = abs(float(lsh.item()) - float(lref.item()))
        good = math.isfinite(d) and math.isfinite(dl) and d <= a.tol and dl <= max(a.tol, 1e-5)
        ok = ok and good
        worst = d if not math.isfinite(d) else max(worst, d)
        if rank == 0:
            print(json.dumps({"step": step, "loss_sharded": float(lsh.item()), "loss_local": float(lref.item()),
                              "max_param_delta": d, "ok": good}), flush=True)
    mem = None
    if a.serialized and fsdp.plan.shard_factor > 1:
        lays = fsdp.layouts
        pred = peak_param_bytes([l.psi for l in lays], [l.shard_numel for l in lays], fsdp.plan.shard_factor,
                                k_full=4, k_low=2 if fsdp.mixed else None, low_copy=fsdp.mixed,
                                nested_root=True)
        meas = fsdp.rt.ledger.peak_param_bytes
        mem = {"peak_param_bytes": meas, "predicted": pred, "ok": meas == pred}
        ok = ok and meas == pred
    flag = torch.tensor([0.0 if ok else 1.0], device="cuda")
    if world > 1:
        all_reduce_(flag)
    ok = flag.item() == 0.0
    if rank == 0:
        print(json.dumps({"verify": "PASS" if ok else "FAIL", "max_param_delta": worst, "tol": a.tol,
                          "inject_fault": a.inject_fault, **({"memory": mem} if mem else {})}), flush=True)
    fsdp.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    return 0 if ok else EXIT_VERIFY_FAIL


_SWEEP_AXES = ("world_size", "sharding_factor", "rate_limit", "raf", "prefetch")


def _parse_axis(spec: str, world: int):
    """cli.py:626-654: name=v1,v2,... (aliases W, F)."""
    if "=" not in spec:
        raise ValueError(f"axis: expected name=v1,v2,..., got {spec!r}")
    name, _, values = spec.partition("=")
    name = {"W": "world_size", "F": "sharding_factor"}.get(name.strip(), name.strip().replace("-", "_"))
    if name not in _SWEEP_AXES:
        raise ValueError(f"axis: {name!r} not sweepable; choose from {_SWEEP_AXES}")
    out = []
    for v in values.split(","):
        v = v.strip()
        if name in ("world_size", "sharding_factor"):
            out.append(int(v))
        elif name == "rate_limit":
            out.append(None if v.lower() in ("none", "inf") else int(v))
        elif name == "raf":
            if v not in ("RAF", "NRAF"):
                raise ValueError(f"axis: raf value {v!r}")
            out.append(v)
        else:
            if v not in ("on", "off"):
                raise ValueError(f"axis: prefetch value {v!r} (on/off)")
            out.append(v)
    if name == "world_size" and any(x != world for x in out):
        raise ValueError(f"axis: world_size must equal the launched world ({world}); "
                         f"launch one sweep per world size")
    if name == "sharding_factor" and any(world % x for x in out):
        raise ValueError(f"axis: sharding_factor values must divide the world ({world})")
    return name, out


def cmd_sweep(a) -> int:
    """cli.py:656-706 on the GPU runtime: Cartesian sweep over F / rate_limit
    / RAF / prefetch; one tab-separated row per point with the final loss,
    AG/RS/AR counts, allocator retries, peak parameter and total bytes from
    the ledger, and the measured step time."""
    import itertools

    import torch
    from .fsdp import BackwardPrefetch, FullyShardedDataParallel, MixedPrecision, ModuleWrapPolicy, ShardingStrategy
    from .workloads import param_init_fn
    rank, world = _dist()
    try:
        parsed = [_parse_axis(s, world) for s in a.axis]
    except ValueError as exc:
        if rank == 0:
            print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    names = [n for n, _ in parsed]
    make, wrap, cfg = _models()[a.model]
    header = names + ["final_loss", "AG", "RS", "AR", "retries", "peak_param_bytes", "peak_total_bytes",
                      "ms_per_step", "tflops_per_gpu"]
    rows = []
    for combo in itertools.product(*(v for _, v in parsed)):
        pt = dict(zip(names, combo))
        F = pt.get("sharding_factor", world)
        strat = (ShardingStrategy.NO_SHARD if F == 1 else ShardingStrategy.FULL_SHARD if F == world
                 else ShardingStrategy.HYBRID_SHARD)
        if pt.get("raf") == "NRAF" and F > 1:
            strat = ShardingStrategy.SHARD_GRAD_OP if F == world else ShardingStrategy._HYBRID_SHARD_ZERO2
        pf = pt.get("prefetch", "on") == "on"
        torch.manual_seed(a.seed)
        with torch.device("meta"):
            m = make()
        fsdp = FullyShardedDataParallel(
            m, sharding_strategy=strat, auto_wrap_policy=ModuleWrapPolicy(wrap),
            backward_prefetch=BackwardPrefetch.BACKWARD_PRE if pf else None, forward_prefetch=pf,
            mixed_precision=MixedPrecision(param_dtype=torch.bfloat16), param_init_fn=param_init_fn,
            hybrid_shard_size=F if strat.name.startswith("_HYBRID") or strat.name == "HYBRID_SHARD" else None,
            rate_limit=pt.get("rate_limit", 2), lr=a.lr)
        opt = fsdp.optimizer()
        g = torch.Generator().manual_seed(a.seed + 1 + rank)
        if hasattr(cfg, "seq"):
            inputs = tuple(torch.randint(0, cfg.vocab, (a.micro, cfg.seq), generator=g).cuda() for _ in range(2))
            flops = cfg.flops_per_token() * a.micro * cfg.seq
        else:
            inputs = (torch.randint(0, cfg.vocab, (a.micro, cfg.enc_seq), generator=g).cuda(),
                      torch.randint(0, cfg.vocab, (a.micro, cfg.dec_seq), generator=g).cuda(),
                      torch.randint(0, cfg.vocab, (a.micro, cfg.dec_seq), generator=g).cuda())
            flops = cfg.flops_per_sample() * a.micro
        fsdp(*inputs).backward()          # warm-up step (not counted)
        opt.step()
        torch.cuda.synchronize()
        fsdp.rt.ledger.reset_peaks()
        torch.cuda.reset_peak_memory_stats()
        t0 = len(fsdp.rt.trace)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            loss = fsdp(*inputs)
            loss.backward()
            opt.step()
        e1.record()
        torch.cuda.synchronize()
        fsdp.check_errors()
        ms = e0.elapsed_time(e1) / a.steps
        cnt = {k: sum(1 for kind, _ in fsdp.rt.trace[t0:] if kind == k + "_issue") for k in ("AG", "RS", "AR")}
        led = fsdp.memory_ledger()
        row = [("on" if pf else "off") if n == "prefetch" else str(pt[n]) for n in names]
        row += [f"{loss.item():.12g}", str(cnt["AG"]), str(cnt["RS"]), str(cnt["AR"]),
                str(led["torch"]["num_alloc_retries"]), str(led["peak_param_bytes"]),
                str(led["peak_total_bytes"]), f"{ms:.3f}", f"{flops / (ms * 1e-3) / 1e12:.1f}"]
        rows.append(row)
        fsdp.close()
        del fsdp, opt
        torch.cuda.empty_cache()
    table = "\t".join(header) + "\n" + "\n".join("\t".join(r) for r in rows)
    if rank == 0:
        if a.out:
            with open(a.out, "w") as fh:
                fh.write(table + "\n")
        else:
            print(table, flush=True)
    return 0


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
    p.add_argument("--strategy", default="FULL_SHARD")
    p.add_argument("--hybrid-shard-size", type=int, default=None)
    p.add_argument("--inject-fault", choices=["misordered-reduction", "inf-grad"], default=None,
                   help="corrupt the sharded run to demonstrate sensitivity (cli.py:568-574)")
    p.add_argument("--serialized", action="store_true",
                   help="rate_limit 1, no prefetch, no keep-outermost: adds the peak-memory formula check")
    p = sub.add_parser("sweep")
    p.add_argument("--model", default="tiny")
    p.add_argument("--axis", action="append", required=True,
                   help="e.g. --axis F=1,2,4 --axis raf=RAF,NRAF --axis rate_limit=1,2,none "
                        "--axis prefetch=on,off (repeatable)")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--micro", type=int, default=2)
    p.add_argument("--lr", type=float, default=1e-4)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    return {"dump-plan": cmd_dump_plan, "run": cmd_run, "verify": cmd_verify,
            "sweep": cmd_sweep}[a.cmd](a)


if __name__ == "__main__":
    sys.exit(main())
