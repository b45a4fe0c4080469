"""Locate mismatches of the bf16-gradient Adam against the fp32-gradient one."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2304_11277_b200 import kernels as K  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1048579
rng = np.random.default_rng(7 + n)
p0 = rng.standard_normal(n).astype(np.float32)
g16 = torch.from_numpy((rng.standard_normal(n) * 1e-2).astype(np.float32)).to(torch.bfloat16).cuda()
g32 = g16.float()
pa, pb = torch.from_numpy(p0).cuda(), torch.from_numpy(p0).cuda()
ma, va, mb, vb = (torch.zeros(n, device="cuda") for _ in range(4))
K.adam_step(pa, g16, ma, va, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=1)
K.adam_step(pb, g32, mb, vb, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=1)
torch.cuda.synchronize()
for name, a, b in (("p", pa, pb), ("m", ma, mb), ("v", va, vb)):
    bad = (a != b).nonzero().flatten().cpu().numpy()
    print(f"variant {os.environ.get('FSDP_ADAM_VARIANT', '0')} {name}: {len(bad)} mismatches of {n}",
          f"first {bad[:8].tolist()}" if len(bad) else "")
    if len(bad):
        i = int(bad[0])
        print("   a", a[i].item(), "b", b[i].item(), "g", g32[i].item(),
              "tile3072", i // 3072, "in-tile", i % 3072, "tile2048", i // 2048, "in2048", i % 2048)
        d = np.diff(bad)
        print("   mismatch spacing histogram:", np.unique(d[:2000], return_counts=True))
