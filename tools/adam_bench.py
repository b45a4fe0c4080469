"""HBM roofline of the sharded Adam launch on one GPU, per kernel variant.

    python tools/adam_bench.py [n_elems]          # spawns one process per variant

Each variant (FSDP_ADAM_TMA / FSDP_ADAM_VARIANT, read once per process) runs
fsdp_adam_step over fp32 p, g, m, v (+ the bf16 copy) of n elements — by
default the GPT-1.3B arena at N=1 (every array far larger than L2) — and is
timed with CUDA events on its stream (2 warm-up + 10 timed launches).
Algorithmic bytes = 30 B/elem (16 read + 14 written).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = [("register", {"FSDP_ADAM_TMA": "0"})] + \
    [(f"tma{v}", {"FSDP_ADAM_TMA": "1", "FSDP_ADAM_VARIANT": str(v)}) for v in range(6)]


def one(n: int) -> dict:
    sys.path.insert(0, ROOT)
    import torch
    from paper_2304_11277_b200 import kernels  # noqa: F401
    from paper_2304_11277_b200._lib import lib
    dev = torch.device("cuda", 0)
    torch.manual_seed(0)
    p, g, m, v = (torch.randn(n, device=dev) * 1e-2 for _ in range(4))
    v.abs_()
    low = torch.empty(n, dtype=torch.bfloat16, device=dev)
    st = torch.cuda.current_stream()

    def launch():
        rc = lib.fsdp_adam_step(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), n, 1e-4, 0.9, 0.1,
                                0.999, 0.001, 0.1, 0.001, 1e-8, None, low.data_ptr(), st.cuda_stream)
        assert rc == 0
    for _ in range(2):
        launch()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        launch()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ms = sorted(ts)[len(ts) // 2]
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6512.6
    gbs = 30 * n / (ms * 1e-3) / 1e9
    # exact integer checksum of the final state: every variant must agree bit for bit
    cks = [int(t.view(torch.int32).to(torch.int64).sum().item()) for t in (p, m, v)]
    cks.append(int(low.view(torch.int16).to(torch.int64).sum().item()))
    return {"checksum": cks, "n": n, "median_ms": round(ms, 4), "min_ms": round(min(ts), 4), "gbs": round(gbs, 1),
            "frac_of_hbm": round(gbs / peak, 4)}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "--one" else 1315819520
    if "--one" in sys.argv:
        print(json.dumps(one(int(sys.argv[sys.argv.index("--one") + 1]))))
        return
    out = {}
    for name, env in VARIANTS:
        r = subprocess.run([sys.executable, __file__, "--one", str(n)], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=600)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")]
        out[name] = json.loads(line[-1]) if line else {"error": r.stderr[-500:]}
        print(name, out[name], file=sys.stderr, flush=True)
    sums = {json.dumps(r.get("checksum")) for r in out.values()}
    out["bit_identical"] = len(sums) == 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
