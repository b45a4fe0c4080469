"""Per-copy cost of back-to-back copy-engine (DMA) peer copies, one process
driving every visible GPU: GPU 0 pushes `total` bytes to each peer in turn
(the serial staggered schedule of fsdp_*_ce), cut into pieces of `piece`
bytes, all on one stream.  Reports GB/s and the implied fixed cost per copy
(t = copies * c + bytes / bw).  python tools/dma_probe.py"""
import json
import sys

import torch


def main():
    n = torch.cuda.device_count()
    if n < 2:
        print(json.dumps({"error": "needs >= 2 GPUs"}))
        return
    total = 256 << 20
    src = torch.empty(total, dtype=torch.uint8, device=0).fill_(1)
    dst = [torch.empty(total, dtype=torch.uint8, device=d) for d in range(1, n)]
    s = torch.cuda.Stream(0)
    res = []
    for piece in (1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 64 << 20, 256 << 20):
        def run():
            with torch.cuda.stream(s):
                for d in dst:
                    for off in range(0, total, piece):
                        d[off:off + piece].copy_(src[off:off + piece], non_blocking=True)
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(5):
            run()
        b.record(s)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 5
        copies = len(dst) * (total // piece)
        res.append({"piece_mb": piece >> 20, "copies": copies, "ms": round(ms, 4),
                    "gbs": round(len(dst) * total / (ms * 1e-3) / 1e9, 1)})
    # fixed cost per copy from the two extremes: t = copies * c + bytes / bw
    big, small = res[-1], res[0]
    c_us = (small["ms"] - big["ms"]) / (small["copies"] - big["copies"]) * 1e3
    print(json.dumps({"gpus": n, "destinations": len(dst), "bytes_per_destination": total, "cases": res,
                      "fixed_cost_per_copy_us": round(c_us, 2)}))


if __name__ == "__main__":
    sys.exit(main())
