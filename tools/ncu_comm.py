"""Profiling harness for the collective DATA kernels with NVLink counters.

One process drives every visible GPU (one VMM communicator per device, peer
pools imported by file descriptor in-process, the NVLS multicast object bound
on every device).  Barrier kernels are switched off
(`fsdp_comm_set_barriers(0)`), and all devices are synchronised between
collectives, so no kernel ever waits on another GPU: safe under ncu's
kernel serialisation and replay.  Run as

    ncu --replay-mode application --clock-control none --metrics \
gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,\
dram__bytes_write.sum -k regex:"allgather|reduce_scatter" --csv \
        python tools/ncu_comm.py --mb 256 --iters 1

Without ncu it prints per-kernel CUDA-event times (all devices concurrently).
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2304_11277_b200 import _lib  # noqa: E402
from paper_2304_11277_b200._lib import check, lib  # noqa: E402
from paper_2304_11277_b200.comm import DeviceComm, _handle_bytes  # noqa: E402


def make_comms(W: int, pool_bytes: int, ctas: int):
    hs = []
    for r in range(W):
        with torch.cuda.device(r):
            h = C.c_void_p()
            check(lib.fsdp_comm_create_vmm(r, W, pool_bytes, ctas, _lib.HANDLE_POSIX_FD, C.byref(h)),
                  "create_vmm")
            hs.append(h)
    fds = []
    for r in range(W):
        buf = (C.c_char * 64)()
        check(lib.fsdp_comm_export_pool(hs[r], buf), "export")
        fds.append(int.from_bytes(bytes(buf)[:4], "little", signed=True))
    for r in range(W):
        with torch.cuda.device(r):
            for p in range(W):
                if p != r:
                    check(lib.fsdp_comm_import_pool(hs[r], p, _handle_bytes(fds[p])), "import")
    buf = (C.c_char * 64)()
    with torch.cuda.device(0):
        check(lib.fsdp_nvls_create(hs[0], W, buf), "nvls_create")
    mc_fd = int.from_bytes(bytes(buf)[:4], "little", signed=True)
    for r in range(1, W):
        with torch.cuda.device(r):
            check(lib.fsdp_nvls_import(hs[r], W, _handle_bytes(mc_fd)), "nvls_import")
    for r in range(W):
        with torch.cuda.device(r):
            check(lib.fsdp_nvls_add_device(hs[r]), "add_device")
    for r in range(W):
        with torch.cuda.device(r):
            check(lib.fsdp_nvls_bind(hs[r]), "bind")
            check(lib.fsdp_comm_set_barriers(hs[r], 0), "barriers")
    for fd in fds + [mc_fd]:
        os.close(fd)
    comms = []
    for r in range(W):
        with torch.cuda.device(r):
            comms.append(DeviceComm(hs[r].value, r, W, False, torch.device("cuda", r)))
    return comms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=256, help="unsharded bf16 bytes per collective (MiB)")
    ap.add_argument("--ctas", type=int, default=64)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--kinds", default="allgather_sm,allgather_nvls,reduce_scatter_pull",
                    help="reduce_scatter_tma waits on peers inside its kernel: not for ncu")
    args = ap.parse_args()
    W = torch.cuda.device_count()
    S = args.mb << 20
    n = S // 2 // W
    comms = make_comms(W, 2 * S + (64 << 20), args.ctas)
    dst = [c.alloc(S) for c in comms][0]
    src_off = [c.alloc(S) for c in comms][0]
    shards, outs = [], []
    for r in range(W):
        with torch.cuda.device(r):
            shards.append(torch.randn(n, device=f"cuda:{r}").to(torch.bfloat16))
            outs.append(torch.empty(n, device=f"cuda:{r}"))
            comms[r].view(src_off, n * W, torch.bfloat16).normal_()

    kinds = {
        "allgather_sm": lambda r: comms[r].all_gather((W, 1), [shards[r]], dst, torch.bfloat16),
        "allgather_nvls": lambda r: comms[r].all_gather_nvls((W, 1), shards[r], dst, torch.bfloat16),
        "reduce_scatter_pull": lambda r: comms[r].reduce_scatter_pull((W, 1), src_off, torch.bfloat16,
                                                                      [outs[r]], postdiv=float(W), tma=False),
        "reduce_scatter_tma": lambda r: comms[r].reduce_scatter_pull((W, 1), src_off, torch.bfloat16,
                                                                     [outs[r]], postdiv=float(W), tma=True),
    }
    res = {"W": W, "unsharded_bytes": S, "bus_bytes_per_rank": S * (W - 1) // W, "ctas": args.ctas}
    kinds = {k: v for k, v in kinds.items() if k in args.kinds.split(",")}
    for name, fn in kinds.items():
        times = []
        for _ in range(args.iters):
            evs = []
            for r in range(W):
                with torch.cuda.device(r):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record()
                    fn(r)
                    b.record()
                    evs.append((a, b))
            for r in range(W):
                torch.cuda.synchronize(r)
            times.append(max(a.elapsed_time(b) for a, b in evs))
        ms = min(times)
        res[name] = {"ms": round(ms, 4), "busbw_gbs": round(S * (W - 1) / W / (ms * 1e-3) / 1e9, 1)}
    for r, c in enumerate(comms):
        with torch.cuda.device(r):
            c.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
