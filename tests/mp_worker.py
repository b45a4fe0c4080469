"""Multi-GPU parity worker (launched by tests/test_multigpu.py via torchrun,
one process per GPU, NCCL only for bootstrap/ground truth).

Shared mode: when the box has fewer GPUs than ranks (the 1-GPU CI box), the
ranks share devices round-robin and bootstrap over gloo.  The CUDA-IPC
communicator, the copy-engine collectives, the symmetric slots, limiter,
prefetch and every strategy run unchanged between processes on one device
(the contexts time-slice the GPU); only the NVLS and NCCL-backend scenarios
are skipped (multicast needs distinct devices; NCCL refuses duplicates).

1. raw IPC collectives (AG with fused cast, RS with fp32 accumulation and
   /W, AR, hybrid RS->AR, scalar AR) vs the oracle — bit-exact;
2. a full FSDP training step of the tiny GPT for every strategy available at
   this world size: the wrapped model's loss equals an unwrapped bf16 copy on
   the rank's slice bit-for-bit, the reduced gradient shard equals the
   oracle's reduction of every rank's write-back gradients bit-for-bit, the
   post-Adam shard equals the oracle's Adam bit-for-bit, and the second step
   (after re-gathering updated parameters) again matches an unwrapped model
   loaded from the gathered state;
3. the NCCL comparison backend agrees within bf16 tolerance.
Rank 0 prints one JSON line; any failure raises (non-zero exit).
"""
import json
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import shardsim_port as sp  # noqa: E402
from oracle.bf16 import round_to_bf16  # noqa: E402


SHARED = False       # ranks share a GPU (set in main)


def gather_np(x: np.ndarray) -> list[np.ndarray]:
    t = torch.from_numpy(np.ascontiguousarray(x))
    if not SHARED:
        t = t.cuda()
    out = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [o.cpu().numpy() for o in out]


def check(cond, msg):
    if not cond:
        raise AssertionError(msg)


def raw_collectives(rank, world, results):
    from paper_2304_11277_b200.comm import DeviceComm
    comm = DeviceComm.create(256 << 20, max_ctas=32)
    comm.set_timeout_ms(20000)
    a, b = comm.alloc(64 << 20), comm.alloc(64 << 20)
    for n in (8, 1000, 262144 + 8):
        rngs = [np.random.default_rng(1000 * r + n) for r in range(world)]
        shards = [g.standard_normal(n).astype(np.float32) for g in rngs]
        grads = [round_to_bf16(g.standard_normal(n * world).astype(np.float32)) for g in rngs]
        acc0 = [g.standard_normal(n).astype(np.float32) for g in rngs]
        # AG fused cast
        comm.all_gather((world, 1), [torch.from_numpy(shards[rank]).cuda()], a, torch.bfloat16)
        got = comm.view(a, n * world, torch.bfloat16).float().cpu().numpy()
        check(np.array_equal(got, sp.cast(sp.all_gather(shards), sp.BF16)), f"AG n={n}")
        # RS bf16 payload, fp32 accumulate, / W, += accum
        out = torch.from_numpy(acc0[rank]).cuda()
        comm.reduce_scatter((world, 1), [torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16)], a,
                            [out], postdiv=float(world), accumulate=True)
        exp = sp.reduce_unit(grads, sp.Plan(world, world), reduce_dtype=sp.BF16, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True, accum=acc0)
        check(out.cpu().numpy().tobytes() == exp[rank].tobytes(), f"RS n={n}")
        # AR (F = 1 / NO_SHARD path)
        out = torch.empty(n * world, device="cuda")
        comm.all_reduce((world, 1), [torch.from_numpy(grads[rank]).cuda()], a, b, [out], postdiv=float(world))
        exp = sp.reduce_unit(grads, sp.Plan(world, 1), reduce_dtype=np.float32, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True)
        check(out.cpu().numpy().tobytes() == exp[rank].tobytes(), f"AR n={n}")
        # copy-engine AR: same bits (fp32 and bf16 payloads, accumulate)
        out_ce = torch.empty(n * world, device="cuda")
        comm.all_reduce_ce((world, 1), torch.from_numpy(grads[rank]).cuda(), a, b, out_ce, postdiv=float(world))
        check(out_ce.cpu().numpy().tobytes() == exp[rank].tobytes(), f"AR-CE n={n}")
        # pool-resident output: written in place on every member, no epilogue
        ob = comm.alloc(n * world * 4 + 256)
        comm.all_reduce_ce_pool((world, 1), torch.from_numpy(grads[rank]).cuda(), a, ob, postdiv=float(world))
        check(comm.view(ob, n * world, torch.float32).cpu().numpy().tobytes() == exp[rank].tobytes(),
              f"AR-CE pool n={n}")
        acc_full = [g.standard_normal(n * world).astype(np.float32) for g in
                    [np.random.default_rng(7 * r + n) for r in range(world)]]
        out_ce = torch.from_numpy(acc_full[rank]).cuda()
        comm.all_reduce_ce((world, 1), torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16), a, b, out_ce,
                           postdiv=float(world), accumulate=True)
        exp = sp.reduce_unit(grads, sp.Plan(world, 1), reduce_dtype=sp.BF16, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True, accum=acc_full)
        check(out_ce.cpu().numpy().tobytes() == exp[rank].tobytes(), f"AR-CE bf16 accumulate n={n}")
        for f in [f for f in (2, 4) if f < world and world % f == 0]:
            part = torch.empty(n * world // f, device="cuda")
            comm.reduce_scatter((f, 1), [torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16)], a, [part])
            out = torch.from_numpy(acc0[rank]).cuda().repeat(world // f)[: n * world // f].contiguous()
            base = out.cpu().numpy().copy()
            comm.all_reduce((world // f, f), [part], a, b, [out], postdiv=float(world), accumulate=True)
            bases = gather_np(base)
            exp = sp.reduce_unit(grads, sp.Plan(world, f), reduce_dtype=sp.BF16, full_dtype=np.float32,
                                 acc_dtype=np.float32, mean=True, accum=bases)
            check(out.cpu().numpy().tobytes() == exp[rank].tobytes(), f"hybrid n={n}")
            out2 = torch.from_numpy(base).cuda()
            comm.all_reduce_ce((world // f, f), part, a, b, out2, postdiv=float(world), accumulate=True)
            check(out2.cpu().numpy().tobytes() == exp[rank].tobytes(), f"hybrid AR-CE n={n}")
        # copy-engine variants: same bits
        sh = torch.from_numpy(shards[rank]).cuda().to(torch.bfloat16)
        comm.all_gather_ce((world, 1), sh, a)
        got = comm.view(a, n * world, torch.bfloat16).float().cpu().numpy()
        check(np.array_equal(got, sp.cast(sp.all_gather(shards), sp.BF16)), f"AG-CE n={n}")
        comm.view(b, n * world, torch.bfloat16).copy_(torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16))
        out = torch.from_numpy(acc0[rank]).cuda()
        comm.reduce_scatter_ce((world, 1), b, torch.bfloat16, a, out, postdiv=float(world), accumulate=True)
        exp = sp.reduce_unit(grads, sp.Plan(world, world), reduce_dtype=sp.BF16, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True, accum=acc0)
        check(out.cpu().numpy().tobytes() == exp[rank].tobytes(), f"RS-CE n={n}")
    flag = torch.tensor([1.0 if rank == world - 1 else 0.0], device="cuda")
    tot = torch.zeros(1, device="cuda")
    comm.scalar_all_reduce([flag], [tot])
    check(tot.item() == 1.0, "scalar AR")
    torch.cuda.synchronize()
    check(comm.device_error() == 0, "device error word")
    comm.close()
    results["raw_collectives"] = "bit-exact"


def full_size_properties(rank, world, results):
    """Size-independent properties at the configs' real sizes (too large for
    the oracle): a GPT-1.3B block's psi = 50,358,272 for the copy-engine
    all-reduce (NO_SHARD / hybrid stage 2) and the split/CE reduce-scatter;
    the LL threshold (6 MB unsharded) for the LL pair.  Inputs are small
    integers, so every fp32 sum is exact and order-independent: the result
    must equal the closed form bit for bit on every rank."""
    from paper_2304_11277_b200.comm import DeviceComm
    psi = 50358272
    n = psi // world
    comm = DeviceComm.create(10 * psi + (256 << 20), max_ctas=32)   # stage + gather fp32, src bf16, LL
    comm.set_timeout_ms(20000)
    stage, gath, src = comm.alloc(psi * 4), comm.alloc(psi * 4), comm.alloc(psi * 2)
    idx = torch.arange(psi, device="cuda", dtype=torch.float32)
    x = ((idx % 7) + rank).to(torch.bfloat16)                 # small integers, exact in bf16
    tot = float(sum(range(world)))
    expect = ((idx % 7) * world + tot) / world                 # exact: integers / power of two
    out = torch.ones(psi, device="cuda")
    comm.all_reduce_ce((world, 1), x, stage, gath, out, postdiv=float(world), accumulate=True)
    check(torch.equal(out, expect + 1.0), "full-size AR-CE")
    comm.view(src, psi, torch.bfloat16).copy_(x)
    o = torch.zeros(n, device="cuda")
    comm.reduce_scatter_ce((world, 1), src, torch.bfloat16, stage, o, postdiv=float(world))
    check(torch.equal(o, expect[rank * n:(rank + 1) * n]), "full-size RS-CE")
    o.zero_()
    comm.reduce_scatter_pull((world, 1), src, torch.bfloat16, [o], postdiv=float(world), tma=True)
    check(torch.equal(o, expect[rank * n:(rank + 1) * n]), "full-size RS TMA pull")
    # LL at the threshold: 6 MB unsharded bf16
    m = (6 << 20) // 2 // world
    ll_a = comm.alloc(comm.ll_bytes(world, m, torch.bfloat16), 16)
    ll_r = comm.alloc(comm.ll_bytes(world, m, torch.bfloat16), 16)
    sh = ((torch.arange(m, device="cuda") % 5) + 10 * rank).to(torch.float32)
    comm.all_gather_ll((world, 1), [sh], gath, torch.bfloat16, ll_a)
    full = comm.view(gath, m * world, torch.bfloat16).float()
    want = torch.cat([(torch.arange(m, device="cuda") % 5 + 10 * r).float() for r in range(world)])
    check(torch.equal(full, want), "LL AG at the threshold")
    y = x[: m * world].contiguous()
    o = torch.zeros(m, device="cuda")
    comm.reduce_scatter_ll((world, 1), [y], ll_r, [o], postdiv=float(world))
    check(torch.equal(o, expect[rank * m:(rank + 1) * m]), "LL RS at the threshold")
    torch.cuda.synchronize()
    check(comm.device_error() == 0, "device error word (full size)")
    comm.close()
    results["full_size_properties"] = f"exact (psi={psi}, LL n={m})"


def ce_schedules(rank, world, results):
    """Every copy-engine schedule gives the same bits: serial-staggered or
    concurrent DMA, reduce-scatter by pull or by push (FSDP_CE_SERIAL,
    FSDP_CE_RS_PUSH, read when a communicator first uses the copy engines)."""
    from paper_2304_11277_b200.comm import DeviceComm
    done = []
    # 262152: one piece.  (1 << 23) + 24 pipelined (FSDP_CE_RS_PIPE_MIN =
    # 2*min_piece): pull with uniform pieces (FSDP_CE_RS_GEOM=0: 4 pieces,
    # short last one); push with geometric pieces (3 pieces at min_piece 2M,
    # 5 at 512K)
    # last case: hybrid -- copy engines for 75 % of every chunk, an SM TMA
    # pull reducing the last 25 % from the peers (FSDP_CE_RS_SM_FRAC)
    # last-but-one: piece-major all-gather DMA (FSDP_CE_AG_PIECE = 4 MB: 5 pieces
    # of the 16.8 MB bf16 shard, every peer per piece)
    for n, serial, push, minp, smf, agp in ((262144 + 8, 1, 0, 0, 0, 0), ((1 << 23) + 24, 1, 0, 1 << 21, 0, 0),
                                            ((1 << 23) + 24, 1, 1, 1 << 21, 0, 0),
                                            ((1 << 23) + 24, 1, 1, 1 << 19, 0, 0),
                                            (262144 + 8, 1, 1, 0, 0, 0),
                                            (262144 + 8, 0, 0, 0, 0, 0), (262144 + 8, 0, 1, 0, 0, 0),
                                            ((1 << 23) + 24, 1, 0, 0, 0, 4 << 20),
                                            ((1 << 23) + 24, 1, 1, 1 << 21, 0.25, 0)):
        rngs = [np.random.default_rng(555 + r) for r in range(world)]
        shards = [g.standard_normal(n).astype(np.float32) for g in rngs]
        grads = [round_to_bf16(g.standard_normal(n * world).astype(np.float32)) for g in rngs]
        acc0 = [g.standard_normal(n).astype(np.float32) for g in rngs]
        exp_ag = sp.cast(sp.all_gather(shards), sp.BF16)
        exp_rs = sp.reduce_unit(grads, sp.Plan(world, world), reduce_dtype=sp.BF16, full_dtype=np.float32,
                                acc_dtype=np.float32, mean=True, accum=acc0)
        exp_rs_b = sp.cast(sp.reduce_scatter(grads, np.float32)[rank], sp.BF16)
        os.environ["FSDP_CE_SERIAL"], os.environ["FSDP_CE_RS_PUSH"] = str(serial), str(push)
        os.environ["FSDP_CE_RS_MIN_PIECE"] = str(minp or (4 << 20))
        os.environ["FSDP_CE_RS_PIPE_MIN"] = str(2 * minp if minp else (64 << 20))
        os.environ["FSDP_CE_RS_GEOM"] = "0" if (minp and not push) else "1"
        os.environ["FSDP_CE_RS_SM_FRAC"] = str(smf)
        os.environ["FSDP_CE_AG_PIECE"] = str(agp)
        nb = n * world * 2 + (1 << 20)
        comm = DeviceComm.create(3 * nb + (4 << 20), max_ctas=32)
        try:
            comm.set_timeout_ms(20000)
            a, b, st = comm.alloc(nb), comm.alloc(nb), comm.alloc(nb)
            for _ in range(3):        # repeated: stale staging / flags would show up here
                comm.all_gather_ce((world, 1), torch.from_numpy(shards[rank]).cuda().to(torch.bfloat16), a)
                got = comm.view(a, n * world, torch.bfloat16).float().cpu().numpy()
                check(np.array_equal(got, exp_ag), f"AG-CE serial={serial}")
                comm.view(b, n * world, torch.bfloat16).copy_(torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16))
                out = torch.from_numpy(acc0[rank]).cuda()
                comm.reduce_scatter_ce((world, 1), b, torch.bfloat16, st, out, postdiv=float(world),
                                       accumulate=True)
                check(out.cpu().numpy().tobytes() == exp_rs[rank].tobytes(),
                      f"RS-CE serial={serial} push={push}")
                # bf16 result (hybrid stage-1 partial in the reduce dtype): the
                # ascending fp32 sum rounded once
                outb = torch.empty(n, dtype=torch.bfloat16, device="cuda")
                comm.reduce_scatter_ce((world, 1), b, torch.bfloat16, st, outb)
                check(np.array_equal(outb.float().cpu().numpy(), exp_rs_b), f"RS-CE bf16 out serial={serial} push={push}")
            torch.cuda.synchronize()
            check(comm.device_error() == 0, "device error word (CE)")
        finally:
            comm.close()
            for k in ("FSDP_CE_SERIAL", "FSDP_CE_RS_PUSH", "FSDP_CE_RS_MIN_PIECE", "FSDP_CE_RS_PIPE_MIN",
                      "FSDP_CE_RS_GEOM", "FSDP_CE_RS_SM_FRAC", "FSDP_CE_AG_PIECE"):
                del os.environ[k]
        done.append(f"n={n}/serial={serial}/push={push}/min_piece={minp}" + (f"/sm_frac={smf}" if smf else "")
                    + (f"/ag_piece={agp}" if agp else ""))
    results["ce_schedules"] = done


def ll_collectives(rank, world, results):
    """Low-latency one-kernel AG/RS (no barriers, epoch-parity double buffer):
    24 back-to-back calls per kind with changing data, one rank delayed on
    device every third call so ranks drift apart, plus hybrid sub-groups at
    W = 4 — every result bit-exact with the oracle."""
    from paper_2304_11277_b200.comm import DeviceComm
    comm = DeviceComm.create(256 << 20, max_ctas=32)
    comm.set_timeout_ms(20000)
    iters = 24
    done = []
    for n, gs in ((1000, world), (65536 + 3, world), (262144, world)) + (((4099, 2),) if world == 4 else ()):
        dst = [comm.alloc(n * gs * 2 + 256) for _ in range(iters)]
        ll_ag = comm.alloc(comm.ll_bytes(gs, n, torch.bfloat16), 16)
        ll_rs = comm.alloc(comm.ll_bytes(gs, n, torch.bfloat16), 16)
        rngs = [np.random.default_rng(77 * r + n) for r in range(world)]
        shards = [[g.standard_normal(n).astype(np.float32) for _ in range(iters)] for g in rngs]
        grads = [[round_to_bf16(g.standard_normal(n * gs).astype(np.float32)) for _ in range(iters)]
                 for g in rngs]
        outs = [torch.zeros(n, device="cuda") for _ in range(iters)]
        dev_sh = [torch.from_numpy(s).cuda() for s in shards[rank]]
        dev_gr = [torch.from_numpy(g).cuda().to(torch.bfloat16) for g in grads[rank]]
        torch.cuda.synchronize()
        dist.barrier()
        for it in range(iters):
            if it % 3 == 0 and rank == it % world:
                torch.cuda._sleep(2_000_000)          # ~1 ms: this rank falls behind
            comm.all_gather_ll((gs, 1), [dev_sh[it]], dst[it], torch.bfloat16, ll_ag)
            comm.reduce_scatter_ll((gs, 1), [dev_gr[it]], ll_rs, [outs[it]], postdiv=float(gs))
        torch.cuda.synchronize()
        start = (rank // gs) * gs
        members = list(range(start, start + gs))
        for it in range(iters):
            exp = sp.cast(sp.all_gather([shards[m][it] for m in members]), sp.BF16)
            got = comm.view(dst[it], n * gs, torch.bfloat16).float().cpu().numpy()
            check(np.array_equal(got, exp), f"AG-LL n={n} gs={gs} it={it}")
            exp = sp.reduce_unit([grads[m][it] for m in members], sp.Plan(gs, gs), reduce_dtype=sp.BF16,
                                 full_dtype=np.float32, acc_dtype=np.float32, mean=True)
            check(outs[it].cpu().numpy().tobytes() == exp[rank - start].tobytes(),
                  f"RS-LL n={n} gs={gs} it={it}")
        done.append(f"n={n}/gs={gs}")
    check(comm.device_error() == 0, "device error word (LL)")
    comm.close()
    results["ll_collectives"] = done


def nvls_collectives(rank, world, results):
    """NVLS multicast all-gather (multimem.st through the NVSwitch): bit-exact
    vs the oracle, fallback sizes, and a 20-iteration stress on changing data
    checked against NCCL's all-gather of the same bf16 shards."""
    from paper_2304_11277_b200 import _lib
    from paper_2304_11277_b200.comm import DeviceComm
    if SHARED:
        results["nvls"] = "skipped: ranks share one GPU (multicast needs distinct devices)"
        return
    if not _lib.lib.fsdp_nvls_supported(torch.cuda.current_device()):
        results["nvls"] = "unsupported on this device: " + _lib.last_error()
        return
    groups = [world] + ([2] if world == 4 else [])
    for F in groups:
        comm = DeviceComm.create(256 << 20, max_ctas=32, nvls_group=F)
        check(comm.nvls_group == F, f"NVLS setup failed (F={F}): {DeviceComm.last_nvls_error}")
        comm.set_timeout_ms(20000)
        a = comm.alloc(128 << 20)
        for n in (8, 1000, 262144 + 8, 4 << 20):
            rngs = [np.random.default_rng(7000 * r + n) for r in range(world)]
            shards = [g.standard_normal(n).astype(np.float32) for g in rngs]
            comm.all_gather_nvls((F, 1), torch.from_numpy(shards[rank]).cuda(), a, torch.bfloat16)
            got = comm.view(a, n * F, torch.bfloat16).float().cpu().numpy()
            g0 = rank // F * F
            check(np.array_equal(got, sp.cast(sp.all_gather(shards[g0:g0 + F]), sp.BF16)),
                  f"AG-NVLS F={F} n={n}")
        if F == world:
            n = 8 << 20
            ref = torch.empty(n * world, dtype=torch.bfloat16, device="cuda")
            for it in range(20):
                x = torch.randn(n, device="cuda", generator=torch.Generator("cuda").manual_seed(rank * 100 + it))
                comm.all_gather_nvls((world, 1), x, a, torch.bfloat16)
                dist.all_gather_into_tensor(ref, x.to(torch.bfloat16))
                torch.cuda.current_stream().synchronize()
                check(torch.equal(comm.view(a, n * world, torch.bfloat16), ref), f"AG-NVLS stress it={it}")
        torch.cuda.synchronize()
        check(comm.device_error() == 0, "device error word (NVLS)")
        comm.close()
    results["nvls"] = f"bit-exact (groups {groups})"


def fsdp_step_parity(rank, world, strategy, hybrid, results, backend="ipc", opt_in_bwd=False,
                     engine="ce", ll=False, fused=False, num_slots=None, split_geom=False,
                     stage2="fp32"):
    """ll=False pins every unit to `engine` (the tiny GPT's units are all
    small enough for the low-latency path, which ll=True exercises)."""
    from paper_2304_11277_b200 import kernels  # noqa: F401
    from paper_2304_11277_b200.fsdp import (FullyShardedDataParallel, MixedPrecision,
                                            ModuleWrapPolicy, ShardingStrategy)
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_, synthetic_batch
    cfg = CONFIGS["tiny"]
    fsdp = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0),
                                    sharding_strategy=ShardingStrategy[strategy],
                                    auto_wrap_policy=ModuleWrapPolicy({Block}),
                                    mixed_precision=MixedPrecision(param_dtype=torch.bfloat16),
                                    hybrid_shard_size=hybrid, comm_backend=backend, lr=1e-3,
                                    optimizer_in_backward=opt_in_bwd, ag_engine=engine,
                                    rs_engine="sm" if engine == "nvls" else engine,
                                    ll_max_bytes=(6 << 20) if ll else 0, fused_cast_ag=fused,
                                    num_slots=num_slots, opt_split_first=1 if split_geom else 2,
                                    opt_split_geom=split_geom, hybrid_stage2=stage2)
    plan = fsdp.plan
    ref = init_gpt_(GPT(cfg), seed=0).cuda().to(torch.bfloat16)
    x, y = synthetic_batch(cfg, 2, seed=100 + rank, device="cuda")
    loss = fsdp(x, y)
    loss.backward()
    lref = ref(x, y)
    lref.backward()
    key = (f"{strategy}{'' if hybrid is None else hybrid}/{backend}/{'ll' if ll else engine}"
           f"{'/opt-in-bwd' if opt_in_bwd else ''}{'/fused-cast-ag' if fused else ''}"
           f"{'' if num_slots is None else '/slots%d' % num_slots}{'/opt-split-geom' if split_geom else ''}"
           f"{'/stage2-reduce-dtype' if stage2 == 'reduce' else ''}")
    torch.cuda.synchronize()
    # initial shards from the oracle (flatten + shard of the same init)
    vals = {k: v.detach().float().cpu().numpy() for k, v in init_gpt_(GPT(cfg), seed=0).named_parameters()}
    k_idx = plan.shard_index(rank)
    before = [sp.shard(sp.flatten(vals, lay, np.float32), lay, k_idx) for lay in fsdp.layouts]
    if backend == "ipc":
        check(loss.item() == lref.item(), f"{key}: loss differs from the unwrapped model")
        g = {n: p.grad.float().cpu().numpy() for n, p in ref.named_parameters()}
        for lay, u in zip(fsdp.layouts, fsdp.rt.units):
            flat = sp.writeback_grad(lay, g, np.float32)[0]
            flats = gather_np(flat)
            exp = sp.reduce_unit(flats, sp.Plan(plan.world_size, plan.shard_factor), reduce_dtype=sp.BF16,
                                 full_dtype=np.float32, acc_dtype=np.float32, mean=True,
                                 stage2_dtype=sp.BF16 if stage2 == "reduce" else None)
            check(u.grad.cpu().numpy().tobytes() == exp[rank].tobytes(),
                  f"{key}: reduced grad of unit {lay.unit_id}")
    fsdp.optimizer().step()
    torch.cuda.synchronize()
    for b, u in zip(before, fsdp.rt.units):
        p = b.copy()
        sp.adam_step(p, u.grad.cpu().numpy(), sp.adam_init(p.size, np.float32), lr=1e-3)
        check(u.master.cpu().numpy().tobytes() == p.tobytes(), f"{key}: Adam shard")
    # step 2: re-gather the updated shards, compare against an unwrapped copy
    sd = fsdp.full_state_dict()
    ref2 = GPT(cfg).cuda()
    ref2.load_state_dict({k: v for k, v in sd.items()}, strict=False)
    ref2 = ref2.to(torch.bfloat16)
    x2, y2 = synthetic_batch(cfg, 2, seed=200 + rank, device="cuda")
    l2 = fsdp(x2, y2)
    l2.backward()
    fsdp.optimizer().step()
    l2r = ref2(x2, y2)
    torch.cuda.synchronize()
    if backend == "ipc":
        check(l2.item() == l2r.item(), f"{key}: step-2 loss after re-gather")
    else:
        check(abs(l2.item() - l2r.item()) < 1e-2, f"{key}: nccl step-2 loss")
    losses = gather_np(np.array([l2.item()], dtype=np.float64))
    results[key] = {"step2_loss_rank0": float(losses[0][0]), "checks": "bit-exact" if backend == "ipc" else "tol"}
    fsdp.close()


def deadlock_detection(rank, world, results):
    """A member that never enters the collective: the others time out on
    device into the error word and surface DeadlockError (the analogue of
    collectives.py:461-483) instead of hanging the GPU."""
    from paper_2304_11277_b200 import _lib
    from paper_2304_11277_b200.comm import DeviceComm
    from paper_2304_11277_b200.plan import DeadlockError
    comm = DeviceComm.create(8 << 20, max_ctas=8)
    comm.set_timeout_ms(1500)
    off = comm.alloc(1 << 16)
    dist.barrier()
    if rank == 0:
        comm.all_gather((world, 1), [torch.ones(64, device="cuda")], off, torch.float32)
        torch.cuda.synchronize()
        check(comm.device_error() == _lib.E_TIMEOUT, "timeout not recorded")
        try:
            comm.raise_device_error()
            check(False, "DeadlockError not raised")
        except DeadlockError:
            pass
    dist.barrier()
    comm.close()
    # the low-latency path polls data lines, not barrier flags: a missing
    # sender must time out the same way
    comm = DeviceComm.create(8 << 20, max_ctas=8)
    comm.set_timeout_ms(1500)
    off = comm.alloc(1 << 16)
    ll = comm.alloc(comm.ll_bytes(world, 64, torch.float32), 16)
    dist.barrier()
    if rank == 0:
        comm.all_gather_ll((world, 1), [torch.ones(64, device="cuda")], off, torch.float32, ll)
        torch.cuda.synchronize()
        check(comm.device_error() == _lib.E_TIMEOUT, "LL timeout not recorded")
        try:
            comm.raise_device_error()
            check(False, "DeadlockError not raised (LL)")
        except DeadlockError:
            pass
    dist.barrier()
    comm.close()
    results["deadlock_detection"] = "ok (split and LL)"


def wrapper_mesh(rank, world, results):
    """HYBRID_SHARD named three ways gives the same sharding and bit-identical
    training: hybrid_shard_size=F, a 2-D device_mesh (replicate, shard), and
    process_group=(shard_group, replicate_group) (collectives.py:63-72)."""
    import torch.distributed as dist
    from paper_2304_11277_b200.fsdp import (FullyShardedDataParallel, MixedPrecision, ModuleWrapPolicy,
                                            ShardingStrategy)
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_, synthetic_batch
    cfg = CONFIGS["tiny"]
    F = 2
    R = world // F
    shard_pgs = [dist.new_group(list(range(g * F, (g + 1) * F))) for g in range(R)]
    rep_pgs = [dist.new_group(list(range(k, world, F))) for k in range(F)]
    mesh_kind = "stub"
    try:
        from torch.distributed.device_mesh import DeviceMesh
        mesh = DeviceMesh("cuda", torch.arange(world).view(R, F), mesh_dim_names=("replicate", "shard"))
        mesh_kind = "torch DeviceMesh"
    except Exception:  # noqa: BLE001 — e.g. ranks sharing one GPU
        class _M:
            pass
        mesh = _M()
        mesh.mesh, mesh.mesh_dim_names = torch.arange(world).view(R, F), ("replicate", "shard")
    variants = {"hybrid_shard_size": dict(hybrid_shard_size=F), "device_mesh": dict(device_mesh=mesh),
                "group_tuple": dict(process_group=(shard_pgs[rank // F], rep_pgs[rank % F]))}
    got = {}
    for name, kw in variants.items():
        fsdp = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0), sharding_strategy=ShardingStrategy.HYBRID_SHARD,
                                        auto_wrap_policy=ModuleWrapPolicy({Block}),
                                        mixed_precision=MixedPrecision(param_dtype=torch.bfloat16), lr=1e-3, **kw)
        check(fsdp.plan.shard_factor == F, f"{name}: F = {fsdp.plan.shard_factor}")
        x, y = synthetic_batch(cfg, 2, seed=400 + rank, device="cuda")
        loss = fsdp(x, y)
        loss.backward()
        fsdp.optimizer().step()
        torch.cuda.synchronize()
        got[name] = (loss.item(), torch.cat([u.master for u in fsdp.rt.units]).cpu())
        fsdp.close()
    ref = got["hybrid_shard_size"]
    for name, (l, m) in got.items():
        check(l == ref[0] and torch.equal(m, ref[1]), f"{name}: differs from hybrid_shard_size")
    try:
        FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0), sharding_strategy=ShardingStrategy.HYBRID_SHARD,
                                 auto_wrap_policy=ModuleWrapPolicy({Block}))
        check(False, "HYBRID_SHARD without a shard-group size did not raise")
    except ValueError:
        pass
    results["wrapper_mesh"] = f"bit-identical ({mesh_kind}, group tuple, hybrid_shard_size; F={F})"


def abort_in_step(rank, world, results):
    """A member stalls past the timeout INSIDE a wrapped training step (its
    compute stream sleeps before the step's first all-gather): the waiting
    members' flag waits time out and abort the communicator on every rank;
    the data kernels stop touching peer memory, the optimizer launch of the
    step is skipped on device (the error word is folded into its predicate),
    and every rank raises DeadlockError (collectives.py:461-483) -- with its
    shards and optimizer state bit-identical to before the step."""
    from paper_2304_11277_b200.fsdp import FullyShardedDataParallel, MixedPrecision, ModuleWrapPolicy
    from paper_2304_11277_b200.plan import DeadlockError
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_, synthetic_batch
    cfg = CONFIGS["tiny"]
    fsdp = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0), auto_wrap_policy=ModuleWrapPolicy({Block}),
                                    mixed_precision=MixedPrecision(param_dtype=torch.bfloat16), lr=1e-3)
    opt = fsdp.optimizer()
    x, y = synthetic_batch(cfg, 2, seed=300 + rank, device="cuda")
    fsdp(x, y).backward()
    opt.step()
    fsdp.check_errors()                               # healthy step: no error
    torch.cuda.synchronize()
    rt = fsdp.rt
    before = [t.clone() for t in (rt.master, rt.exp_avg, rt.exp_avg_sq, rt.low)]
    fsdp.comm.set_timeout_ms(1500)
    dist.barrier()
    if rank == world - 1:
        torch.cuda._sleep(6_000_000_000)              # ~3 s on the compute stream: misses the timeout
    raised = False
    try:
        fsdp(x, y).backward()
        opt.step()
        fsdp.check_errors()
    except DeadlockError:
        raised = True
    torch.cuda.synchronize()
    check(raised, f"rank {rank}: DeadlockError not raised after a peer stalled past the timeout")
    after = [rt.master, rt.exp_avg, rt.exp_avg_sq, rt.low]
    for name, a, b in zip(("master", "exp_avg", "exp_avg_sq", "low"), before, after):
        check(torch.equal(a, b), f"rank {rank}: {name} changed by an aborted step")
    # the next step refuses to run on an aborted communicator
    again = False
    try:
        opt.step()
    except DeadlockError:
        again = True
    check(again, "optimizer step on an aborted communicator did not raise")
    dist.barrier()
    fsdp.close()
    results["abort_in_step"] = "DeadlockError on every rank; shards and Adam state unchanged"


def _sess(w, f, spec=None, seed=0, **kw):
    from paper_2304_11277_b200.data import ModelSpec
    from paper_2304_11277_b200.plan import build_plan
    from paper_2304_11277_b200.session import EngineConfig, Session
    spec = spec or ModelSpec(dims=(4, 8, 8, 2))
    return Session(spec, EngineConfig(plan=build_plan(w, f), **kw), seed=seed)


def _ag_split(trace):
    """(forward AG issues, backward AG issues) of the first step region."""
    fwd = bwd = 0
    phase = "fwd"
    for kind, _ in trace:
        if kind == "backward_begin":
            phase = "bwd"
        elif kind == "step":
            break
        elif kind == "AG_issue":
            if phase == "fwd":
                fwd += 1
            else:
                bwd += 1
    return fwd, bwd


def session_parity(rank, world, results):
    """The reference's test_engine.py scenarios on real ranks."""
    from paper_2304_11277_b200.data import ModelSpec
    from paper_2304_11277_b200.session import NRAF, PrecisionPolicy, StaticOrderError
    torch.backends.cuda.matmul.allow_tf32 = False
    spec3 = sp.MLPSpec(dims=(4, 8, 8, 2))
    uniform = ModelSpec(dims=(8, 8, 8, 8))
    out = {}
    # equivalence vs the oracle restatement of Session.run (fp32): bitwise for
    # the first step (integer data + dyadic init keep every op exact), then
    # within 1e-5 (later steps carry more mantissa bits, and cuBLAS and numpy
    # sum GEMM products in different orders)
    for f in [x for x in (1, 2, 4, 8) if world % x == 0 and x <= world]:
        for opt in ("sgd", "adam"):
            s = _sess(world, f, seed=3, optimizer=opt)
            s.run(steps=1, batch=8)
            exp, losses, _, _ = sp.sharded_train(spec3, sp.Plan(world, f), 3, 1, 8, optimizer=opt,
                                                 full=np.float32, acc_dtype=np.float32)
            got = s.gather_full_params()
            for k in exp:
                check(got[k].tobytes() == exp[k].astype(np.float32).tobytes(), f"session F={f} {opt} {k}")
            s.close()
            s = _sess(world, f, seed=3, optimizer=opt)      # run() restarts the data stream
            s.run(steps=3, batch=8)
            exp, *_ = sp.sharded_train(spec3, sp.Plan(world, f), 3, 3, 8, optimizer=opt)
            got = s.gather_full_params()
            d = max(float(np.abs(got[k] - exp[k]).max()) for k in exp)
            # Adam normalises by sqrt(v)+eps: a ~1e-8 grad difference on an
            # element whose v is ~0 moves it by up to lr; SGD stays tight
            check(d < (1e-5 if opt == "sgd" else 5e-3), f"session F={f} {opt} 3-step delta {d}")
            check(s.replica_divergence() == 0.0, f"replicas diverged F={f}")
            check(s.check_reduction_ordering() == [], "reduction ordering")
            s.close()
    out["bitwise_vs_oracle"] = "step 1 bit-exact, 3 steps < 1e-5 vs float64 reference"
    # AG counts: keep outermost (3, 2); without (3, 3); NRAF (3, 0)   (test_engine.py:190-206)
    for kw, exp in (({}, (3, 2)), ({"keep_outermost_unsharded": False}, (3, 3)),
                    ({"reshard_after_forward": NRAF}, (3, 0))):
        s = _sess(world, world, **kw)
        s.run(steps=1, batch=8)
        check(_ag_split(s.trace) == exp, f"AG split {kw}: {_ag_split(s.trace)}")
        s.close()
    # backward prefetch: AG(u-1) before RS(u)                         (test_engine.py:209-231)
    s = _sess(world, world, keep_outermost_unsharded=False, backward_prefetch=True)
    s.run(steps=1, batch=8)
    tail = [(k, u) for k, u in s.trace if k in ("AG_issue", "RS_issue")][3:]
    check(tail == [("AG_issue", 2), ("AG_issue", 1), ("RS_issue", 2), ("AG_issue", 0),
                   ("RS_issue", 1), ("RS_issue", 0)], f"bwd prefetch order {tail}")
    s.close()
    s = _sess(world, world, keep_outermost_unsharded=False, backward_prefetch=False)
    s.run(steps=1, batch=8)
    tail = [(k, u) for k, u in s.trace if k in ("AG_issue", "RS_issue")][3:]
    check(tail == [("AG_issue", 2), ("RS_issue", 2), ("AG_issue", 1), ("RS_issue", 1),
                   ("AG_issue", 0), ("RS_issue", 0)], f"no-prefetch order {tail}")
    s.close()
    # forward prefetch begins on the second iteration                 (test_engine.py:247-262)
    s = _sess(world, world, spec=uniform, forward_prefetch=True, keep_outermost_unsharded=False)
    s.run(steps=2, batch=8)
    second = s.trace[s.trace.index(("step", None)) + 1:]
    ag1 = second.index(("AG_issue", 1))
    c0 = second.index(("compute_begin", 0))
    check(ag1 < c0, "forward prefetch: AG(1) before compute(0)")
    s.close()
    s = _sess(world, world, spec=uniform, forward_prefetch=True)
    s.order_hook = lambda step: [0, 1, 2] if step == 0 else [0, 2, 1]
    try:
        s.run(steps=2, batch=8)
        check(False, "StaticOrderError not raised")
    except StaticOrderError:
        pass
    torch.cuda.synchronize()
    s.close()
    # scaler: inf on one rank skips everywhere                          (test_engine.py:351-361)
    s = _sess(world, max(1, world // 2), seed=1, use_scaler=True)
    s.inject_inf = {(world - 1, 1)}
    res = s.run(steps=3, batch=8)
    check([r.stepped for r in res] == [True, False, True], "scaler verdict")
    check(res[1].scale == 65536.0 * 0.5, "scaler backoff")
    exp, _, stepped, _ = sp.sharded_train(spec3, sp.Plan(world, max(1, world // 2)), 1, 3, 8,
                                          use_scaler=True, inject_inf={(world - 1, 1)})
    check(stepped == [r.stepped for r in res], "scaler verdicts vs reference")
    got = s.gather_full_params()
    d = max(float(np.abs(got[k] - exp[k]).max()) for k in exp)
    check(d < 1e-5, f"scaler params delta {d}")
    s.close()
    # accumulation: RS every micro vs once                              (test_engine.py:158-183)
    for mode, rs in (("with_comm", world * 3 * 2), ("no_comm", world * 3)):
        s = _sess(world, world, seed=8, accumulation=mode, accumulation_steps=2)
        r = s.run(steps=1, batch=8)
        check(r[0].event_counts.get("RS") == rs, f"{mode} RS count {r[0].event_counts}")
        exp, *_ = sp.sharded_train(spec3, sp.Plan(world, world), 8, 1, 8, accumulation=mode,
                                   accumulation_steps=2, full=np.float32, acc_dtype=np.float32)
        got = s.gather_full_params()
        check(all(got[k].tobytes() == exp[k].astype(np.float32).tobytes() for k in exp), f"{mode} params")
        s.close()
    # rate limiter: resident unsharded buffers (the ledger peak of test_engine.py:294-317:
    # one buffer without prefetch, two with backward prefetch)
    for limit, bwdp, expect in ((1, False, 1), (2, False, 1), (1, True, 2), (2, True, 2)):
        s = _sess(world, world, spec=uniform, rate_limit=limit, backward_prefetch=bwdp,
                  keep_outermost_unsharded=False)
        s.run(steps=2, batch=8)
        check(s.rt.max_live_slots == expect, f"limiter {limit}/{bwdp}: {s.rt.max_live_slots}")
        s.close()
    # mixed precision: masters fp32, close to full precision           (test_engine.py:331-348)
    s = _sess(world, world, seed=4, precision=PrecisionPolicy(mixed=True))
    s.run(steps=3, batch=8)
    ref, *_ = sp.sharded_train(spec3, sp.Plan(world, world), 4, 3, 8)
    g = s.gather_full_params()
    d = max(float(np.abs(g[k] - ref[k]).max()) for k in ref)
    check(0 < d < 1e-2, f"mixed delta {d}")
    check(all(u.master.dtype == torch.float32 for u in s.rt.units), "fp32 masters")
    # AG payload is low precision: issue bytes = psi x 2 (test_engine.py:331-341, low = bf16)
    ag_bytes = [b for (k, u), b in zip(s.trace, s.trace.nbytes) if k == "AG_issue"]
    check(ag_bytes[0] == s.layouts[0].psi * 2, f"mixed AG bytes {ag_bytes[0]}")
    s.close()
    results["session"] = out


class _Done(Exception):
    pass


def main():
    global SHARED
    from paper_2304_11277_b200.dist_util import init_from_env, shared_gpu
    world = int(os.environ["WORLD_SIZE"])
    SHARED = shared_gpu(world)
    rank, world, _ = init_from_env()
    results = {"world": world, "shared_gpu": SHARED, "backend": dist.get_backend()}
    ok = True
    only = os.environ.get("MP_ONLY")       # debugging: a comma list of scenario functions
    try:
        if only:
            for name in only.split(","):
                globals()[name](rank, world, results)
            raise _Done()
        hybrids = [f for f in (2, 4) if f < world and world % f == 0]
        steps = [("FULL_SHARD", None, {}), ("SHARD_GRAD_OP", None, {}), ("NO_SHARD", None, {})]
        steps += [("HYBRID_SHARD", f, {}) for f in hybrids]
        steps += [("FULL_SHARD", None, {"opt_in_bwd": True}), ("FULL_SHARD", None, {"ll": True}),
                  ("SHARD_GRAD_OP", None, {"ll": True})]
        steps += [("HYBRID_SHARD", f, {"ll": True}) for f in hybrids]
        steps += [("FULL_SHARD", None, {"engine": "sm"}), ("FULL_SHARD", None, {"fused": True}),
                  ("FULL_SHARD", None, {"fused": True, "ll": True})]
        steps += [("HYBRID_SHARD", f, {"fused": True}) for f in hybrids]
        # slot-starved: 2 slots for 3 units (root kept + one block at a time;
        # backward prefetch finds no free slot and is skipped).  The default 3
        # slots already re-gather each block into a different slot in backward
        # (saved tensors re-materialise against it, pack_hook)
        steps += [("FULL_SHARD", None, {"num_slots": 2}), ("FULL_SHARD", None, {"split_geom": True})]
        if not SHARED:
            steps += [("FULL_SHARD", None, {"engine": "nvls"})]
            steps += [("HYBRID_SHARD", f, {"engine": "nvls"}) for f in hybrids]
        steps += [("HYBRID_SHARD", f, {"engine": "sm"}) for f in hybrids]
        steps += [("HYBRID_SHARD", f, {"opt_in_bwd": True}) for f in hybrids]
        # stage-2 payload in the reduce dtype: copy-engine reduce-scatter
        # writing bf16, the SM tail and the LL path through fp32 + one rounding
        steps += [("HYBRID_SHARD", f, {"stage2": "reduce"}) for f in hybrids]
        steps += [("HYBRID_SHARD", f, {"stage2": "reduce", "ll": True}) for f in hybrids[:1]]
        if not SHARED:
            steps += [("FULL_SHARD", None, {"backend": "nccl"})]
        scen = [("raw_collectives", raw_collectives), ("full_size_properties", full_size_properties),
                ("ll_collectives", ll_collectives), ("nvls_collectives", nvls_collectives),
                ("ce_schedules", ce_schedules), ("session_parity", session_parity)]
        scen += [("fsdp_step", lambda r, w, res, s=s, h=h, kw=kw: fsdp_step_parity(r, w, s, h, res, **kw))
                 for s, h, kw in steps]
        if world >= 4:
            scen += [("wrapper_mesh", wrapper_mesh)]
        scen += [("deadlock_detection", deadlock_detection), ("abort_in_step", abort_in_step)]
        # MP_SCENARIOS: comma list of scenario names to run (default: all)
        pick = os.environ.get("MP_SCENARIOS")
        pick = set(pick.split(",")) if pick else None
        for name, fn in scen:
            if pick is None or name in pick:
                fn(rank, world, results)
    except _Done:
        pass
    except Exception:
        ok = False
        traceback.print_exc()
    flag = torch.tensor([0.0 if ok else 1.0], device="cpu" if SHARED else "cuda")
    dist.all_reduce(flag)
    if rank == 0:
        results["ok"] = flag.item() == 0.0
        print(json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0.0 else 1)


if __name__ == "__main__":
    main()
