"""Multi-GPU parity worker (launched by tests/test_multigpu.py via torchrun,
one process per GPU, NCCL only for bootstrap/ground truth).

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


def gather_np(x: np.ndarray) -> list[np.ndarray]:
    t = torch.from_numpy(np.ascontiguousarray(x)).cuda()
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
        if world == 4:
            f = 2
            part = torch.empty(n * world // f, device="cuda")
            comm.reduce_scatter((f, 1), [torch.from_numpy(grads[rank]).cuda().to(torch.bfloat16)], a, [part])
            out = torch.from_numpy(acc0[rank]).cuda().repeat(world // f)[: n * world // f].contiguous()
            base = out.cpu().numpy().copy()
            comm.all_reduce((world // f, f), [part], a, b, [out], postdiv=float(world), accumulate=True)
            bases = gather_np(base)
            exp = sp.reduce_unit(grads, sp.Plan(world, f), reduce_dtype=sp.BF16, full_dtype=np.float32,
                                 acc_dtype=np.float32, mean=True, accum=bases)
            check(out.cpu().numpy().tobytes() == exp[rank].tobytes(), f"hybrid n={n}")
    flag = torch.tensor([1.0 if rank == world - 1 else 0.0], device="cuda")
    tot = torch.zeros(1, device="cuda")
    comm.scalar_all_reduce([flag], [tot])
    check(tot.item() == 1.0, "scalar AR")
    torch.cuda.synchronize()
    check(comm.device_error() == 0, "device error word")
    comm.close()
    results["raw_collectives"] = "bit-exact"


def fsdp_step_parity(rank, world, strategy, hybrid, results, backend="ipc"):
    from paper_2304_11277_b200 import kernels  # noqa: F401
    from paper_2304_11277_b200.fsdp import (FullyShardedDataParallel, MixedPrecision,
                                            ModuleWrapPolicy, ShardingStrategy)
    from paper_2304_11277_b200.workloads import CONFIGS, GPT, Block, init_gpt_, synthetic_batch
    cfg = CONFIGS["tiny"]
    fsdp = FullyShardedDataParallel(init_gpt_(GPT(cfg), seed=0),
                                    sharding_strategy=ShardingStrategy[strategy],
                                    auto_wrap_policy=ModuleWrapPolicy({Block}),
                                    mixed_precision=MixedPrecision(param_dtype=torch.bfloat16),
                                    hybrid_shard_size=hybrid, comm_backend=backend, lr=1e-3)
    plan = fsdp.plan
    ref = init_gpt_(GPT(cfg), seed=0).cuda().to(torch.bfloat16)
    x, y = synthetic_batch(cfg, 2, seed=100 + rank, device="cuda")
    loss = fsdp(x, y)
    loss.backward()
    lref = ref(x, y)
    lref.backward()
    key = f"{strategy}{'' if hybrid is None else hybrid}/{backend}"
    before = [u.master.clone() for u in fsdp.rt.units]
    torch.cuda.synchronize()
    if backend == "ipc":
        check(loss.item() == lref.item(), f"{key}: loss differs from the unwrapped model")
        g = {n: p.grad.float().cpu().numpy() for n, p in ref.named_parameters()}
        for lay, u in zip(fsdp.layouts, fsdp.rt.units):
            flat = sp.writeback_grad(lay, g, np.float32)[0]
            flats = gather_np(flat)
            exp = sp.reduce_unit(flats, sp.Plan(plan.world_size, plan.shard_factor), reduce_dtype=sp.BF16,
                                 full_dtype=np.float32, acc_dtype=np.float32, mean=True)
            check(u.grad.cpu().numpy().tobytes() == exp[rank].tobytes(),
                  f"{key}: reduced grad of unit {lay.unit_id}")
    fsdp.optimizer().step()
    torch.cuda.synchronize()
    for b, u in zip(before, fsdp.rt.units):
        p = b.cpu().numpy().copy()
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


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    results = {"world": world}
    ok = True
    try:
        raw_collectives(rank, world, results)
        cases = [("FULL_SHARD", None), ("SHARD_GRAD_OP", None), ("NO_SHARD", None)]
        if world == 4:
            cases.append(("HYBRID_SHARD", 2))
        for strat, hyb in cases:
            fsdp_step_parity(rank, world, strat, hyb, results)
        fsdp_step_parity(rank, world, "FULL_SHARD", None, results, backend="nccl")
    except Exception:
        ok = False
        traceback.print_exc()
    flag = torch.tensor([0.0 if ok else 1.0], device="cuda")
    dist.all_reduce(flag)
    if rank == 0:
        results["ok"] = flag.item() == 0.0
        print(json.dumps(results), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if flag.item() == 0.0 else 1)


if __name__ == "__main__":
    main()
