"""Cost of back-to-back copy-engine (DMA) peer copies, one process driving
every visible GPU (raw cudaMemcpyAsync on peer pointers via cuda-python, no
torch cross-device synchronisation): GPU 0 pushes `total` bytes to each peer
in turn (the serial staggered schedule of fsdp_*_ce), cut into pieces, the
pieces dealt round-robin over `lanes` streams (lanes > 1: consecutive pieces
to the SAME destination overlap, so one copy's start/drain latency can hide
behind another's transfer).  Reports GB/s and the implied fixed cost per
copy (t = copies * c + bytes / bw).

    python tools/dma_probe.py
"""
import json
import sys

import torch
from cuda.bindings import runtime as rt


def ck(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != rt.cudaError_t.cudaSuccess:
        raise RuntimeError(str(err))
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


def main():
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"error": "needs >= 2 GPUs"}))
        return
    total = 256 << 20
    torch.cuda.set_device(0)
    for d in range(1, n):
        ck(rt.cudaSetDevice(0))
        r = rt.cudaDeviceEnablePeerAccess(d, 0)
        if r[0] not in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
            raise RuntimeError(str(r[0]))
    ck(rt.cudaSetDevice(0))
    src = torch.empty(total, dtype=torch.uint8, device=0).fill_(1)
    dst = [torch.empty(total, dtype=torch.uint8, device=d) for d in range(1, n)]
    main_s = torch.cuda.Stream(0)
    lanes_all = [torch.cuda.Stream(0) for _ in range(4)]
    kind = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice
    res = []
    for lanes in (1, 2, 4):
        for piece in (4 << 20, 16 << 20, 32 << 20, 64 << 20, 256 << 20):
            ls = lanes_all[:lanes]

            def run():
                fork = torch.cuda.Event()
                fork.record(main_s)
                for s in ls:
                    s.wait_event(fork)
                i = 0
                for d in dst:
                    for off in range(0, total, piece):
                        s = ls[i % lanes]
                        i += 1
                        ck(rt.cudaMemcpyAsync(d.data_ptr() + off, src.data_ptr() + off, piece, kind,
                                              s.cuda_stream))
                for s in ls:
                    e = torch.cuda.Event()
                    e.record(s)
                    main_s.wait_event(e)
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(main_s)
            for _ in range(5):
                run()
            b.record(main_s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            res.append({"lanes": lanes, "piece_mb": piece >> 20, "copies": len(dst) * (total // piece),
                        "ms": round(ms, 4), "gbs": round(len(dst) * total / (ms * 1e-3) / 1e9, 1)})
    fixed = {}
    for lanes in (1, 2, 4):
        rows = [r for r in res if r.get("lanes") == lanes]
        big, small = rows[-1], rows[0]
        fixed[lanes] = round((small["ms"] - big["ms"]) / (small["copies"] - big["copies"]) * 1e3, 2)
    print(json.dumps({"gpus": n, "destinations": len(dst), "bytes_per_destination": total, "cases": res,
                      "fixed_cost_per_copy_us_by_lanes": fixed}))


if __name__ == "__main__":
    sys.exit(main())
