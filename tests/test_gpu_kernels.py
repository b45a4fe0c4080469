"""Parity of the copy / cast / optimizer kernels (through the C ABI) with the
oracle and with the reference's own golden vectors.  Bit-exact."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import shardsim_port as sp
from oracle.bf16 import round_to_bf16

pytestmark = pytest.mark.gpu

DT = {"f32": torch.float32, "bf16": torch.bfloat16}


@pytest.fixture(scope="module")
def K():
    from paper_2304_11277_b200 import kernels
    return kernels


def to_np(t):
    return t.float().cpu().numpy()


@pytest.mark.parametrize("src,dst", [("f32", "f32"), ("f32", "bf16"), ("bf16", "bf16"), ("bf16", "f32")])
@pytest.mark.parametrize("shapes,F", [
    ([(2, 3), (2,), (3, 3)], 4),
    ([(768, 256), (768,), (256, 256), (256,)], 2),
    ([(7,), (13, 5), (1,), (33,)], 8),         # unaligned offsets -> scalar paths
    ([(4096,)], 1),
    ([(3,)], 7),
])
def test_flatten_matches_oracle(K, src, dst, shapes, F):
    rng = np.random.default_rng(0)
    names = [f"p{i}" for i in range(len(shapes))]
    lay = sp.build_unit_layouts(list(zip(names, shapes)), [names], F)[0]
    vals = {n: rng.standard_normal(s).astype(np.float32) for n, s in zip(names, shapes)}
    if src == "bf16":
        vals = {n: round_to_bf16(v) for n, v in vals.items()}
    ts = [torch.from_numpy(vals[n]).to("cuda", DT[src]) for n in names]
    flat = torch.full((lay.psi,), 7.0, dtype=DT[dst], device="cuda")
    K.flatten(ts, [o.offset for o in lay.originals], flat)
    exp = sp.flatten(vals, lay, sp.BF16 if dst == "bf16" else np.float32)
    assert to_np(flat).tobytes() == exp.astype(np.float32).tobytes()
    # accumulate: flat += values (fp32 add, rounded to dst)
    K.flatten(ts, [o.offset for o in lay.originals], flat, accumulate=True)
    exp2 = exp.astype(np.float32) + exp.astype(np.float32)
    exp2 = sp.cast(exp2, sp.BF16 if dst == "bf16" else np.float32)
    assert np.array_equal(to_np(flat), exp2)
    # unflatten round trip + shard copy
    outs = [torch.empty(s, dtype=DT[src], device="cuda") for s in shapes]
    K.flatten(ts, [o.offset for o in lay.originals], flat)
    K.unflatten(flat, outs, [o.offset for o in lay.originals])
    for o, n in zip(outs, names):
        exp_o = sp.cast(sp.cast(vals[n], sp.BF16 if dst == "bf16" else np.float32),
                        sp.BF16 if src == "bf16" else np.float32)
        assert np.array_equal(to_np(o), exp_o)
    for k in range(F):
        sh = torch.empty(lay.shard_numel, dtype=DT[dst], device="cuda")
        K.shard_copy(flat, sh, k)
        assert to_np(sh).tobytes() == sp.shard(exp.astype(np.float32), lay, k).tobytes()


def test_flatten_missing_grads_zero_filled(K):
    lay = sp.build_unit_layouts([("a", (5,)), ("b", (9,))], [["a", "b"]], 4)[0]
    flat = torch.full((lay.psi,), 3.0, device="cuda")
    K.flatten([None, torch.ones(9, device="cuda")], [0, 5], flat)
    exp, warns = sp.writeback_grad(lay, {"b": np.ones(9, np.float32)}, np.float32)
    assert np.array_equal(to_np(flat), exp) and len(warns) == 1


def test_flatten_large_vector_path(K):
    n = (1 << 22) + 24
    a = torch.randn(n, device="cuda")
    b = torch.randn(1000, device="cuda")
    flat = torch.empty(n + 1000 + 8, dtype=torch.bfloat16, device="cuda")
    K.flatten([a, b], [0, n], flat)
    exp = torch.cat([a, b, torch.zeros(8, device="cuda")]).to(torch.bfloat16)
    assert torch.equal(flat, exp)


def test_cast_bits_match_torch_rne(K):
    x = torch.randn(1 << 20, device="cuda") * 1e3
    x[:6] = torch.tensor([0.0, -0.0, float("inf"), -float("inf"), 1e-40, 3.3e38])
    y = torch.empty_like(x, dtype=torch.bfloat16)
    K.cast(x, y)
    assert torch.equal(y.view(torch.int16), x.to(torch.bfloat16).view(torch.int16))
    # odd length, unaligned start
    y2 = torch.empty(999, dtype=torch.bfloat16, device="cuda")
    K.cast(x[1:1000], y2)
    assert torch.equal(y2, x[1:1000].to(torch.bfloat16))


@pytest.mark.parametrize("lr", [1e-3, 0.01])
def test_adam_bit_exact_vs_reference_golden(K, golden, lr):
    arrays, _ = golden
    p = torch.from_numpy(arrays[f"adam/lr{lr}/p0"].copy()).cuda()
    m = torch.zeros_like(p)
    v = torch.zeros_like(p)
    for t in range(4):
        g = torch.from_numpy(arrays[f"adam/lr{lr}/g{t}"]).cuda()
        K.adam_step(p, g, m, v, lr=lr, betas=(0.9, 0.999), eps=1e-8, t=t + 1)
        assert p.cpu().numpy().tobytes() == arrays[f"adam/lr{lr}/p{t + 1}"].tobytes()
        assert m.cpu().numpy().tobytes() == arrays[f"adam/lr{lr}/m{t + 1}"].tobytes()
        assert v.cpu().numpy().tobytes() == arrays[f"adam/lr{lr}/v{t + 1}"].tobytes()


@pytest.mark.parametrize("n", [(1 << 20) + 3, 6144 * 148 * 2 + 6144 * 5 + 11])
def test_adam_large_with_lowp_and_skip(K, n):
    """Large n: the TMA-pipelined kernel (uneven contiguous tile ranges per
    CTA) plus its scalar tail."""
    rng = np.random.default_rng(1)
    p0 = rng.standard_normal(n).astype(np.float32)
    g0 = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    p = torch.from_numpy(p0).cuda()
    g = torch.from_numpy(g0).cuda()
    m, v = torch.zeros_like(p), torch.zeros_like(p)
    low = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    pe = p0.copy()
    st = sp.adam_init(n, np.float32)
    for t in (1, 2, 3):
        K.adam_step(p, g, m, v, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, t=t, p_lowp=low)
        sp.adam_step(pe, g0, st, lr=3e-4, betas=(0.9, 0.95), eps=1e-8)
        assert p.cpu().numpy().tobytes() == pe.tobytes()
        assert m.cpu().numpy().tobytes() == st["m"].tobytes()
        assert v.cpu().numpy().tobytes() == st["v"].tobytes()
        assert torch.equal(low, p.to(torch.bfloat16))
    skip = torch.ones(1, device="cuda")
    before = p.clone()
    K.adam_step(p, g, m, v, lr=3e-4, betas=(0.9, 0.95), eps=1e-8, t=2, skip_flag=skip)
    assert torch.equal(p, before)


@pytest.mark.parametrize("n", [1000, (1 << 20) + 3, 6144 * 148 * 2 + 6144 * 5 + 11])
def test_adam_bf16_grad_matches_fp32_grad(K, n):
    """The W = 1 bf16-gradient optimizer (fsdp_adam_step_bf16g /
    fsdp_sgd_step_bf16g) against the fp32-gradient kernels on the exact fp32
    copy of the same bf16 gradient, and against the oracle: bit-identical for
    the register kernel (small n) and the TMA kernel (+ scalar tail)."""
    rng = np.random.default_rng(7 + n)
    p0 = rng.standard_normal(n).astype(np.float32)
    g16 = torch.from_numpy((rng.standard_normal(n) * 1e-2).astype(np.float32)).to(torch.bfloat16).cuda()
    g32 = g16.float()
    pa, pb = torch.from_numpy(p0).cuda(), torch.from_numpy(p0).cuda()
    ma, va, mb, vb = (torch.zeros(n, device="cuda") for _ in range(4))
    la = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    lb = torch.empty_like(la)
    pe, st = p0.copy(), sp.adam_init(n, np.float32)
    for t in (1, 2):
        K.adam_step(pa, g16, ma, va, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=t, p_lowp=la)
        K.adam_step(pb, g32, mb, vb, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=t, p_lowp=lb)
        sp.adam_step(pe, g32.cpu().numpy(), st, lr=1e-3)
        assert torch.equal(pa, pb) and torch.equal(ma, mb) and torch.equal(va, vb) and torch.equal(la, lb)
        assert pa.cpu().numpy().tobytes() == pe.tobytes()
    K.sgd_step(pa, g16, lr=0.03125)
    K.sgd_step(pb, g32, lr=0.03125)
    assert torch.equal(pa, pb)


@pytest.mark.parametrize("variant", range(6))
def test_adam_every_ring_variant_bit_exact(variant):
    """Every TMA ring geometry of the Adam kernel (FSDP_ADAM_VARIANT, one per
    process), fp32 and bf16 gradients, against the oracle."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "tools/adam_check.py"], cwd=root, capture_output=True, text=True,
                       timeout=300, env=dict(os.environ, FSDP_ADAM_VARIANT=str(variant)))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_sgd_golden(K, golden):
    arrays, _ = golden
    p = torch.from_numpy(arrays["sgd/p0"].copy()).cuda()
    K.sgd_step(p, torch.from_numpy(arrays["sgd/g"]).cuda(), lr=0.03125)
    assert p.cpu().numpy().tobytes() == arrays["sgd/p1"].tobytes()


def test_unscale_found_inf(K):
    g = torch.randn(100003, device="cuda")
    ref = g.cpu().numpy().copy()
    flag = torch.zeros(1, device="cuda")
    K.unscale_found_inf(g, 1.0 / 65536.0, flag)
    assert flag.item() == 0.0
    assert not sp.unscale_and_check([ref], 65536.0)
    assert g.cpu().numpy().tobytes() == ref.tobytes()
    g[777] = float("nan")
    K.unscale_found_inf(g, 0.5, flag)
    assert flag.item() == 1.0


def test_launch_counter_advances(K):
    from paper_2304_11277_b200 import _lib
    n0 = _lib.launch_count()
    K.cast(torch.ones(10, device="cuda"), torch.empty(10, device="cuda"))
    assert _lib.launch_count() == n0 + 1


@pytest.mark.parametrize("seed", range(24))
def test_layout_kernels_randomized(K, seed):
    """Random layouts against a plain torch restatement: 1..130 tensors
    (beyond one launch's table), sizes 0..3000 incl. empty tensors, sources
    that are views at odd element offsets (scalar paths), odd padding,
    every dtype pair, plain and accumulate; unflatten into odd-offset views;
    cast of odd-start slices."""
    g = torch.Generator().manual_seed(seed)
    rnd = lambda a, b: int(torch.randint(a, b, (1,), generator=g))  # noqa: E731
    src_dt = [torch.float32, torch.bfloat16][seed % 2]
    dst_dt = [torch.float32, torch.bfloat16][(seed // 2) % 2]
    nt = rnd(1, 131)
    numels = [rnd(0, 3000) if rnd(0, 4) else rnd(0, 9) for _ in range(nt)]
    base = torch.randn(sum(numels) + 7 * nt + 8, generator=g).to("cuda", src_dt)
    ts, cur = [], rnd(0, 8)
    for n in numels:
        ts.append(base[cur: cur + n])
        cur += n + rnd(0, 8)
    offsets, o = [], 0
    for n in numels:
        offsets.append(o)
        o += n
    psi = o + rnd(0, 300)
    ref = torch.zeros(psi, dtype=torch.float32, device="cuda")
    for t, off in zip(ts, offsets):
        ref[off: off + t.numel()] = t.float()
    flat = torch.full((psi,), 5.0, dtype=dst_dt, device="cuda")
    K.flatten(ts, offsets, flat)
    assert torch.equal(flat, ref.to(dst_dt)), "flatten"
    prev = flat.clone()
    K.flatten(ts, offsets, flat, accumulate=True)
    assert torch.equal(flat, (prev.float() + ref).to(dst_dt)), "flatten accumulate"
    # unflatten into views at odd offsets of one buffer
    obuf = torch.full((sum(numels) + 5 * nt + 8,), -1.0, dtype=src_dt, device="cuda")
    outs, cur = [], rnd(0, 6)
    for n in numels:
        outs.append(obuf[cur: cur + n])
        cur += n + rnd(0, 6)
    K.flatten(ts, offsets, flat)
    K.unflatten(flat, outs, offsets)
    for t, out in zip(ts, outs):
        assert torch.equal(out, t.to(dst_dt).to(src_dt)), "unflatten"
    # cast of an odd-start slice
    s0 = rnd(0, 9)
    src = base[s0:]
    dst = torch.empty(src.numel() + 3, dtype=dst_dt, device="cuda")[3:]
    K.cast(src, dst)
    assert torch.equal(dst, src.to(dst_dt)), "cast"
