"""DRAM bytes of the copy-engine all-gather's DMA pattern, measured by ncu
range replay (ncu cannot attribute DMA to a kernel).  One process drives
every visible GPU; GPU 0 does what one rank of `fsdp_allgather_ce` does:
push the same bf16 shard to each peer in turn (serial staggered), plus its
own chunk as a local copy.  Whether the W-1 re-reads of the shard hit L2 or
DRAM shows in GPU 0's dram__bytes_read.

    ncu --replay-mode range \\
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \\
        python tools/ncu_dma_range.py [shard_mb] [piece_mb]

piece_mb > 0: the piece-major order of FSDP_CE_AG_PIECE (every peer gets
piece q before piece q+1 is sent to anyone).
"""
import sys

import torch
from cuda.bindings import runtime as rt


def main():
    n = torch.cuda.device_count()
    shard = int(float(sys.argv[1]) * (1 << 20)) if len(sys.argv) > 1 else 25 << 20   # GPT-1.3B block at F=4
    piece = int(float(sys.argv[2]) * (1 << 20)) if len(sys.argv) > 2 else 0
    piece = piece if 0 < piece < shard else shard
    torch.cuda.set_device(0)
    for d in range(1, n):
        r = rt.cudaDeviceEnablePeerAccess(d, 0)
        assert r[0] in (rt.cudaError_t.cudaSuccess, rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled), r
    src = torch.empty(shard, dtype=torch.uint8, device=0).fill_(3)
    own = torch.empty(shard, dtype=torch.uint8, device=0)
    dst = [torch.empty(shard, dtype=torch.uint8, device=d) for d in range(1, n)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=0)
    marker = torch.zeros(1, device=0)
    s = torch.cuda.Stream(0)
    kind = rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice
    for rep in range(2):
        flush.zero_()                                   # src out of L2 before the range
        torch.cuda.synchronize()
        if rep == 1:
            torch.cuda.profiler.start()               # cudaProfilerStart: opens ncu's range
            marker.add_(1)                            # a kernel in the range (ranges need one)
        for off in range(0, shard, piece):              # piece-major when piece < shard
            ln = min(piece, shard - off)
            for d in dst:                               # remote copies, one destination at a time
                assert rt.cudaMemcpyAsync(d.data_ptr() + off, src.data_ptr() + off, ln, kind,
                                          s.cuda_stream)[0] == rt.cudaError_t.cudaSuccess
        rt.cudaMemcpyAsync(own.data_ptr(), src.data_ptr(), shard, kind, s.cuda_stream)
        s.synchronize()
        if rep == 1:
            torch.cuda.profiler.stop()
    print(f"shard {shard} B (pieces of {piece} B), {len(dst)} peers + own copy: algorithmic DRAM read on GPU 0 = "
          f"{shard} B (once) vs {shard * (len(dst) + 1)} B (once per copy); write = {shard} B (own chunk)")


if __name__ == "__main__":
    main()
