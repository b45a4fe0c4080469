"""Bit-exactness of one Adam kernel variant (FSDP_ADAM_VARIANT, read once per
process) against the oracle, for fp32 and bf16 gradients, on a length that
takes the TMA path with an uneven tile split and a scalar tail.  Prints one
JSON line; exit 1 on any mismatch.  tests/test_gpu_kernels.py runs it for
every variant.

    FSDP_ADAM_VARIANT=k python tools/adam_check.py [n]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import shardsim_port as sp  # noqa: E402  (checker only)
from paper_2304_11277_b200 import kernels as K  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 6144 * 148 * 2 + 6144 * 5 + 11
    rng = np.random.default_rng(11)
    p0 = rng.standard_normal(n).astype(np.float32)
    g16 = torch.from_numpy((rng.standard_normal(n) * 1e-2).astype(np.float32)).to(torch.bfloat16)
    g32 = g16.float().numpy()
    exp, st = p0.copy(), sp.adam_init(n, np.float32)
    out = {"variant": int(os.environ.get("FSDP_ADAM_VARIANT", "0")), "n": n}
    ok = True
    p = {k: torch.from_numpy(p0).cuda() for k in ("f32", "bf16")}
    m = {k: torch.zeros(n, device="cuda") for k in p}
    v = {k: torch.zeros(n, device="cuda") for k in p}
    g = {"f32": torch.from_numpy(g32).cuda(), "bf16": g16.cuda()}
    for t in (1, 2):
        sp.adam_step(exp, g32, st, lr=1e-3)
        for k in p:
            K.adam_step(p[k], g[k], m[k], v[k], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=t)
    torch.cuda.synchronize()
    for k in p:
        bad = int((p[k].cpu() != torch.from_numpy(exp)).sum()) + int((m[k].cpu() != torch.from_numpy(st["m"])).sum())
        out[f"mismatches_{k}"] = bad
        ok = ok and bad == 0
    out["ok"] = ok
    print(json.dumps(out))
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
