"""torch.distributed plumbing: process-group setup and small host-side
collectives (losses, counters, test ground truth).  The data path never goes
through here — it is the C-ABI communicator (`comm.py`).

One process per GPU is the production layout (backend "nccl").  When a box has
fewer GPUs than ranks (a 1-GPU CI box running a W-rank test), ranks share
devices round-robin ("shared" mode): the CUDA-IPC communicator works unchanged
between processes on one device (the contexts time-slice the GPU), but NCCL
refuses duplicate devices, so the plumbing backend becomes gloo.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def env_ranks() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shared_gpu(world: int | None = None) -> bool:
    """True when ranks must share devices (fewer visible GPUs than local ranks)."""
    if world is None:
        world = int(os.environ.get("LOCAL_WORLD_SIZE", os.environ.get("WORLD_SIZE", "1")))
    n = torch.cuda.device_count()
    return world > 1 and 0 < n < world


def init_from_env() -> tuple[int, int, torch.device]:
    """Set the device of this rank and initialise the default process group
    (nccl, or gloo in shared mode / when FSDP_DIST_BACKEND says so)."""
    rank, world, local = env_ranks()
    n = max(1, torch.cuda.device_count())
    dev = torch.device("cuda", local % n)
    torch.cuda.set_device(dev)
    if world > 1 and not dist.is_initialized():
        backend = os.environ.get("FSDP_DIST_BACKEND") or ("gloo" if shared_gpu() else "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return rank, world, dev


def backend() -> str | None:
    return dist.get_backend() if dist.is_available() and dist.is_initialized() else None


def _host(t: torch.Tensor) -> bool:
    return t.is_cuda and backend() != "nccl"


def all_reduce_(t: torch.Tensor, op=None, group=None) -> torch.Tensor:
    """In-place all-reduce of a (small) tensor on either backend."""
    op = dist.ReduceOp.SUM if op is None else op
    if _host(t):
        c = t.cpu()
        dist.all_reduce(c, op=op, group=group)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def all_gather(t: torch.Tensor, group=None) -> list[torch.Tensor]:
    """List of every rank's tensor (same device as `t`), either backend."""
    w = dist.get_world_size(group)
    if _host(t):
        c = t.detach().cpu().contiguous()
        out = [torch.empty_like(c) for _ in range(w)]
        dist.all_gather(out, c, group=group)
        return [o.to(t.device) for o in out]
    out = [torch.empty_like(t) for _ in range(w)]
    dist.all_gather(out, t.contiguous(), group=group)
    return out


def barrier() -> None:
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def broadcast_(t: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """In-place broadcast from global rank `src`, either backend."""
    if _host(t):
        c = t.cpu()
        dist.broadcast(c, src=src, group=group)
        t.copy_(c)
    else:
        dist.broadcast(t, src=src, group=group)
    return t
