"""Exercise every kernel of the library once at small sizes on cuda:0, for
compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck --kernel-name kns=fsdp python tools/sanitize_driver.py

Covers the layout kernels (aligned and ragged tensors, every dtype pair), the
optimizer kernels (TMA and register Adam with a scalar tail, SGD, unscale),
and the collectives on an emulated 4-rank communicator: split AG / RS (push,
register pull, TMA pull), the two-shot all-reduce, the LL kernels and the
scalar all-reduce.  Results are checked loosely (finite); the parity tests
are elsewhere -- this only drives the code under the sanitizer.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2304_11277_b200 import kernels  # noqa: E402
from paper_2304_11277_b200.comm import DeviceComm  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    # layout kernels: ragged tensors, every dtype pair, accumulate
    shapes = [(3, 5), (17,), (64, 33), (1,), (1000,)]
    for sd in (torch.float32, torch.bfloat16):
        for fd in (torch.float32, torch.bfloat16):
            ts = [torch.randn(s, device=dev).to(sd) for s in shapes]
            offs, o = [], 0
            for t in ts:
                offs.append(o)
                o += t.numel() + 3
            flat = torch.empty(o + 5, dtype=fd, device=dev)
            kernels.flatten(ts, offs, flat)
            kernels.flatten(ts, offs, flat, accumulate=True)
            outs = [torch.empty(s, dtype=sd, device=dev) for s in shapes]
            kernels.unflatten(flat, outs, offs)
            sh = torch.empty(flat.numel() // 4, dtype=fd, device=dev)
            kernels.shard_copy(flat, sh, 1)
            kernels.cast(flat, torch.empty(flat.numel(), dtype=sd, device=dev))
    # optimizer kernels
    for n in (1000 + 3, 6144 * 148 + 6144 * 3 + 7):
        p, g = torch.randn(n, device=dev), torch.randn(n, device=dev) * 1e-2
        m, v = torch.zeros_like(p), torch.zeros_like(p)
        low = torch.empty(n, dtype=torch.bfloat16, device=dev)
        kernels.adam_step(p, g, m, v, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=1, p_lowp=low)
        kernels.sgd_step(p, g, lr=1e-3, p_lowp=low)
        found = torch.zeros(1, device=dev)
        kernels.unscale_found_inf(g, 0.5, found)
    torch.cuda.synchronize()
    # collectives, emulated W = 4 (one cooperative launch per collective)
    W, n = 4, 4099 * 8
    c = DeviceComm.create_emulated(W, 64 << 20, max_ctas=4)
    c.set_timeout_ms(120000)
    a, b = c.alloc(8 << 20), c.alloc(8 << 20)
    ll_ag = c.alloc(c.ll_bytes(W, n, torch.float32), 16)
    ll_rs = c.alloc(c.ll_bytes(W, n, torch.bfloat16), 16)
    shards = [torch.randn(n, device=dev) for _ in range(W)]
    flats = [torch.randn(n * W, device=dev).to(torch.bfloat16) for _ in range(W)]
    outs = [torch.zeros(n, device=dev) for _ in range(W)]
    c.all_gather((W, 1), shards, a, torch.bfloat16)
    c.reduce_scatter((W, 1), flats, a, outs, postdiv=float(W), accumulate=True)
    for e in range(W):
        c.view(b, n * W, torch.bfloat16, e).copy_(flats[e])
    c.reduce_scatter_pull((W, 1), b, torch.bfloat16, outs, postdiv=float(W), tma=False)
    c.reduce_scatter_pull((W, 1), b, torch.bfloat16, outs, postdiv=float(W), tma=True)
    full = [torch.zeros(n * W, device=dev) for _ in range(W)]
    c.all_reduce((W, 1), [f.float() for f in flats], a, a + (2 << 20), full, postdiv=float(W))
    for _ in range(2):                                  # both LL parities
        c.all_gather_ll((W, 1), shards, a, torch.bfloat16, ll_ag)
        c.reduce_scatter_ll((W, 1), flats, ll_rs, outs, postdiv=float(W), accumulate=True)
    fl = [torch.ones(1, device=dev) for _ in range(W)]
    fo = [torch.zeros(1, device=dev) for _ in range(W)]
    c.scalar_all_reduce(fl, fo)
    torch.cuda.synchronize()
    assert c.device_error() == 0
    assert all(torch.isfinite(o).all().item() for o in outs)
    c.close()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
