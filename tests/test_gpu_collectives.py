"""Cross-rank collectives on ONE GPU: an emulated communicator runs all W
ranks' pools on cuda:0 and launches each collective as one cooperative
kernel (blockIdx.y = rank) — the same flag protocol and address arithmetic
as the multi-GPU path.  Checked bit-exactly against the reference's golden
vectors (shardsim fabric, float32) and the oracle (bf16 payloads)."""
import numpy as np
import pytest
import torch

from oracle import shardsim_port as sp
from oracle.bf16 import round_to_bf16

pytestmark = pytest.mark.gpu


def make_comm(w, mb=64):
    from paper_2304_11277_b200.comm import DeviceComm
    c = DeviceComm.create_emulated(w, mb << 20, max_ctas=8)
    c.set_timeout_ms(5000)
    return c


def cu(a, dt=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)


@pytest.mark.parametrize("w", [1, 2, 3, 4, 8])
def test_ag_rs_ar_match_reference_golden(golden, w):
    arrays, _ = golden
    inputs = [arrays[f"coll/in/w{w}/r{r}"] for r in range(w)]
    n = inputs[0].size
    c = make_comm(w)
    try:
        off = c.alloc(1 << 20)
        c.all_gather((w, 1), [cu(x[: n // w]) for x in inputs], off, torch.float32)
        for r in range(w):
            got = c.view(off, n, torch.float32, r).cpu().numpy()
            assert got.tobytes() == arrays[f"coll/ag/w{w}/out{r}"].tobytes()
        outs = [torch.empty(n // w, device="cuda") for _ in range(w)]
        c.reduce_scatter((w, 1), [cu(x) for x in inputs], off, outs)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == arrays[f"coll/rs/w{w}/out{r}"].tobytes()
        off_b = c.alloc(1 << 20)
        outs = [torch.empty(n, device="cuda") for _ in range(w)]
        c.all_reduce((w, 1), [cu(x) for x in inputs], off, off_b, outs)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == arrays[f"coll/ar/w{w}/out{r}"].tobytes()
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


@pytest.mark.parametrize("w,f", [(w, f) for w in range(2, 9) for f in range(1, w + 1) if w % f == 0])
def test_hybrid_rs_then_ar_matches_golden(golden, w, f):
    """Eq. (1): RS in the sharded group then AR in the replicated group."""
    arrays, _ = golden
    grads = [arrays[f"hyb/w{w}f{f}/in{r}"] for r in range(w)]
    psi = grads[0].size
    n = psi // f
    c = make_comm(w)
    try:
        a, b = c.alloc(1 << 20), c.alloc(1 << 20)
        if f == 1:
            outs = [torch.empty(psi, device="cuda") for _ in range(w)]
            c.all_reduce((w, 1), [cu(g) for g in grads], a, b, outs)
        else:
            part = [torch.empty(n, device="cuda") for _ in range(w)]
            c.reduce_scatter((f, 1), [cu(g) for g in grads], a, part)
            outs = part
            if f < w:
                outs = [torch.empty(n, device="cuda") for _ in range(w)]
                c.all_reduce((w // f, f), part, a, b, outs)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == arrays[f"hyb/w{w}f{f}/out{r}"].tobytes(), (w, f, r)
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


@pytest.mark.parametrize("w", [2, 4, 8])
@pytest.mark.parametrize("n", [8, 1000, 65536 + 24, 300007])
def test_allgather_cast_bf16_bit_exact(w, n):
    rng = np.random.default_rng(n + w)
    shards = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
    c = make_comm(w)
    try:
        off = c.alloc(n * w * 2 + 256)
        c.all_gather((w, 1), [cu(s) for s in shards], off, torch.bfloat16)
        exp = sp.cast(sp.all_gather(shards), sp.BF16)    # gather-then-cast == cast-then-gather
        for r in range(w):
            assert np.array_equal(c.view(off, n * w, torch.bfloat16, r).float().cpu().numpy(), exp)
        # bf16 -> bf16 (the runtime's path: shards pre-cast by the optimizer)
        c.all_gather((w, 1), [cu(s, torch.bfloat16) for s in shards], off, torch.bfloat16)
        for r in range(w):
            assert np.array_equal(c.view(off, n * w, torch.bfloat16, r).float().cpu().numpy(), exp)
    finally:
        c.close()


@pytest.mark.parametrize("w", [2, 4, 8])
@pytest.mark.parametrize("n", [16, 4104, 262144])
def test_reduce_scatter_bf16_fp32_accumulate_divide(w, n):
    """bf16 payloads, fp32 ascending accumulation from +0, / W, += accum
    (engine.py:789-820 with the build's fp32 accumulation)."""
    rng = np.random.default_rng(w * 7 + n)
    grads = [round_to_bf16(rng.standard_normal(n * w).astype(np.float32)) for _ in range(w)]
    acc0 = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
    c = make_comm(w)
    try:
        off = c.alloc(n * w * 2 + 256)
        outs = [cu(a) for a in acc0]
        c.reduce_scatter((w, 1), [cu(g, torch.bfloat16) for g in grads], off, outs,
                         postdiv=float(w), accumulate=True)
        exp = sp.reduce_unit(grads, sp.Plan(w, w), reduce_dtype=sp.BF16, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True, accum=acc0)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == exp[r].tobytes()
    finally:
        c.close()


@pytest.mark.parametrize("tma", [False, True])
@pytest.mark.parametrize("w", [1, 2, 3, 4, 8])
def test_reduce_scatter_pull_matches_golden(golden, w, tma):
    arrays, _ = golden
    inputs = [arrays[f"coll/in/w{w}/r{r}"] for r in range(w)]
    n = inputs[0].size
    c = make_comm(w)
    try:
        off = c.alloc(1 << 20)
        for r in range(w):
            c.view(off, n, torch.float32, r).copy_(cu(inputs[r]))
        outs = [torch.empty(n // w, device="cuda") for _ in range(w)]
        c.reduce_scatter_pull((w, 1), off, torch.float32, outs, tma=tma)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == arrays[f"coll/rs/w{w}/out{r}"].tobytes()
    finally:
        c.close()


@pytest.mark.parametrize("w,f", [(2, 2), (4, 4), (8, 8), (8, 4), (6, 3), (4, 2)])
@pytest.mark.parametrize("n", [16, 1000, 65536 + 8, 1 << 20])
@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("tma", [False, True])
def test_reduce_scatter_pull_bf16_divide_accumulate(w, f, n, dt, tma):
    rng = np.random.default_rng(w * 100 + f * 10 + n)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    grads = [rng.standard_normal(n * f).astype(np.float32) for _ in range(w)]
    if dt == "bf16":
        grads = [round_to_bf16(g) for g in grads]
    acc0 = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
    c = make_comm(w)
    try:
        off = c.alloc(n * f * 4 + 256)
        for r in range(w):
            c.view(off, n * f, tdt, r).copy_(cu(grads[r], tdt))
        outs = [cu(a) for a in acc0]
        c.reduce_scatter_pull((f, 1), off, tdt, outs, postdiv=float(w), accumulate=True, tma=tma)
        for g0 in range(0, w, f):
            grp = list(range(g0, g0 + f))
            res = sp.reduce_scatter([grads[r] for r in grp], acc_dtype=np.float32)
            for pos, r in enumerate(grp):
                exp = acc0[r] + res[pos] / np.float32(w)
                assert outs[r].cpu().numpy().tobytes() == exp.tobytes(), (r, pos)
    finally:
        c.close()


@pytest.mark.parametrize("w,f", [(8, 4), (8, 2), (4, 2)])
def test_hybrid_bf16_reduce_unit(w, f):
    """Full hybrid reduction of bf16 grads incl. / W and accumulation."""
    rng = np.random.default_rng(w * 10 + f)
    psi = 8 * 1024 * f
    grads = [round_to_bf16(rng.standard_normal(psi).astype(np.float32)) for _ in range(w)]
    n = psi // f
    acc0 = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
    c = make_comm(w)
    try:
        a, b = c.alloc(psi * 4 + 4096), c.alloc(psi * 4 + 4096)
        part = [torch.empty(n, device="cuda") for _ in range(w)]
        c.reduce_scatter((f, 1), [cu(g, torch.bfloat16) for g in grads], a, part)
        outs = [cu(x) for x in acc0]
        c.all_reduce((w // f, f), part, a, b, outs, postdiv=float(w), accumulate=True)
        exp = sp.reduce_unit(grads, sp.Plan(w, f), reduce_dtype=sp.BF16, full_dtype=np.float32,
                             acc_dtype=np.float32, mean=True, accum=acc0)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == exp[r].tobytes()
    finally:
        c.close()


def test_kth_call_pairs_and_scalar_allreduce():
    w = 4
    c = make_comm(w)
    try:
        off = c.alloc(4096)
        for k in range(5):    # repeated calls on one channel: epochs pair k-th with k-th
            c.all_gather((w, 1), [torch.full((4,), float(10 * k + r), device="cuda") for r in range(w)],
                         off, torch.float32)
            exp = np.repeat([10.0 * k + r for r in range(w)], 4)
            for r in range(w):
                assert np.array_equal(c.view(off, 16, torch.float32, r).cpu().numpy(), exp)
        ins = [torch.tensor([float(r == 2)], device="cuda") for r in range(w)]
        outs = [torch.zeros(1, device="cuda") for _ in range(w)]
        c.scalar_all_reduce(ins, outs)
        assert all(o.item() == 1.0 for o in outs)
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


def test_fabric_entry_contract():
    from paper_2304_11277_b200.comm import DeviceFabric
    from paper_2304_11277_b200.plan import CollectiveError
    c = make_comm(2)
    try:
        fab = DeviceFabric(c, 1 << 16)
        with pytest.raises(CollectiveError):
            fab.all_gather(3, (0, 1), [torch.zeros(2, device="cuda")] * 2)     # not a member
        with pytest.raises(CollectiveError):
            fab.all_gather(0, (0, 1), [torch.zeros(2, 2, device="cuda")] * 2)  # not flat
        with pytest.raises(CollectiveError):
            fab.reduce_scatter(0, (0, 1), [torch.zeros(3, device="cuda")] * 2)  # 3 % 2
        with pytest.raises(CollectiveError):
            fab.all_gather(0, (0, 1), [torch.zeros(2, device="cuda"), torch.zeros(3, device="cuda")])
        out = fab.reduce_scatter(0, (0, 1), [cu([1., 2, 3, 4]), cu([10., 20, 30, 40])])
        assert out[0].tolist() == [11, 22] and out[1].tolist() == [33, 44]
    finally:
        c.close()


def test_full_size_unit_properties():
    """BASELINE config size (one GPT-1.3B block unit, psi = 50,358,272 at
    F = W = 8), checked through size-independent properties on an emulated
    8-rank communicator:
      * gather(shard_k(flatten(x)) for k) == flatten(x), bit for bit, with
        the fp32 -> bf16 cast fused (== cast(flatten(x)));
      * reduce-scatter of W identical bf16 payloads of small integers, / W,
        returns the payload chunk exactly (every partial sum is exact in
        fp32), for every rank's chunk."""
    from paper_2304_11277_b200 import kernels
    from paper_2304_11277_b200.workloads import CONFIGS
    cfg = CONFIGS["gpt1.3b"]
    W = 8
    d = cfg.d
    shapes = [(d,), (d,), (3 * d, d), (3 * d,), (d, d), (d,), (d,), (d,), (4 * d, d), (4 * d,),
              (d, 4 * d), (d,)]
    numels = [int(np.prod(s)) for s in shapes]
    raw = sum(numels)
    psi = -(-raw // W) * W
    assert raw == cfg.block_params and psi == 50_358_272
    n = psi // W
    offsets = list(np.cumsum([0] + numels[:-1]))
    g = torch.Generator(device="cuda").manual_seed(0)
    ts = [torch.randn(s, device="cuda", generator=g) for s in shapes]
    flat = torch.empty(psi, device="cuda")
    kernels.flatten(ts, offsets, flat)
    shards = []
    for k in range(W):
        sh = torch.empty(n, device="cuda")
        kernels.shard_copy(flat, sh, k)
        shards.append(sh)
    c = make_comm(W, mb=psi * 2 // (1 << 20) + 8)
    try:
        c.set_timeout_ms(20000)
        off = c.alloc(psi * 2)
        c.all_gather((W, 1), shards, off, torch.bfloat16)
        exp = flat.to(torch.bfloat16)
        for r in range(W):
            assert torch.equal(c.view(off, psi, torch.bfloat16, r), exp), f"AG rank {r}"
        payload = torch.randint(-64, 64, (psi,), device="cuda", generator=g).to(torch.bfloat16)
        outs = [torch.empty(n, device="cuda") for _ in range(W)]
        c.reduce_scatter((W, 1), [payload] * W, off, outs, postdiv=float(W))
        for r in range(W):
            assert torch.equal(outs[r], payload[r * n:(r + 1) * n].float()), f"RS rank {r}"
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


# ------------------------------------------------- low-latency one-shot path
@pytest.mark.parametrize("w", [1, 2, 3, 4, 8])
def test_ll_ag_rs_match_reference_golden(golden, w):
    """The LL one-kernel variants against the shardsim fabric's golden AG/RS."""
    arrays, _ = golden
    inputs = [arrays[f"coll/in/w{w}/r{r}"] for r in range(w)]
    n = inputs[0].size
    c = make_comm(w)
    try:
        off = c.alloc(1 << 20)
        ll = c.alloc(c.ll_bytes(w, n, torch.float32), 16)
        c.all_gather_ll((w, 1), [cu(x[: n // w]) for x in inputs], off, torch.float32, ll)
        for r in range(w):
            got = c.view(off, n, torch.float32, r).cpu().numpy()
            assert got.tobytes() == arrays[f"coll/ag/w{w}/out{r}"].tobytes()
        outs = [torch.empty(n // w, device="cuda") for _ in range(w)]
        ll_rs = c.alloc(c.ll_bytes(w, n // w, torch.float32), 16)   # one region per channel
        c.reduce_scatter_ll((w, 1), [cu(x) for x in inputs], ll_rs, outs)
        for r in range(w):
            assert outs[r].cpu().numpy().tobytes() == arrays[f"coll/rs/w{w}/out{r}"].tobytes()
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


@pytest.mark.parametrize("w", [2, 4, 8])
@pytest.mark.parametrize("n", [1, 7, 1000, 65536 + 24, 300007])
def test_ll_allgather_cast_bit_exact_repeated(w, n):
    """fp32 -> bf16 fused cast and bf16 -> bf16, odd lengths (partial last
    line), 5 back-to-back calls on changing data through the same LL region
    (both epoch parities, stale lines from earlier epochs present)."""
    rng = np.random.default_rng(n + 31 * w)
    c = make_comm(w)
    try:
        off = c.alloc(n * w * 4 + 256)
        ll = c.alloc(c.ll_bytes(w, n, torch.float32), 16)
        for it in range(5):
            shards = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
            exp = sp.cast(sp.all_gather(shards), sp.BF16)
            src_dt = torch.float32 if it % 2 == 0 else torch.bfloat16
            c.all_gather_ll((w, 1), [cu(s, src_dt) for s in shards], off, torch.bfloat16, ll)
            for r in range(w):
                got = c.view(off, n * w, torch.bfloat16, r).float().cpu().numpy()
                assert np.array_equal(got, exp), (it, r)
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


@pytest.mark.parametrize("w", [2, 4, 8])
@pytest.mark.parametrize("n", [1, 5, 4104, 262147])
def test_ll_reduce_scatter_bf16_accumulate_divide(w, n):
    """bf16 payload, fp32 ascending sum from +0, prediv/postdiv, += accum;
    4 back-to-back calls (both parities) — bit-exact with the oracle."""
    rng = np.random.default_rng(w * 13 + n)
    c = make_comm(w)
    try:
        ll = c.alloc(c.ll_bytes(w, n, torch.bfloat16), 16)
        acc0 = [rng.standard_normal(n).astype(np.float32) for _ in range(w)]
        outs = [cu(a) for a in acc0]
        exp = acc0
        for it in range(4):
            grads = [round_to_bf16(rng.standard_normal(n * w).astype(np.float32)) for _ in range(w)]
            c.reduce_scatter_ll((w, 1), [cu(g, torch.bfloat16) for g in grads], ll, outs,
                                postdiv=float(w), accumulate=True)
            exp = sp.reduce_unit(grads, sp.Plan(w, w), reduce_dtype=sp.BF16, full_dtype=np.float32,
                                 acc_dtype=np.float32, mean=True, accum=exp)
            for r in range(w):
                assert outs[r].cpu().numpy().tobytes() == exp[r].tobytes(), (it, r)
        torch.cuda.synchronize()
        assert c.device_error() == 0
    finally:
        c.close()


@pytest.mark.parametrize("w,f", [(4, 2), (8, 2), (8, 4)])
def test_ll_reduce_scatter_subgroups(golden, w, f):
    """LL RS inside sharded sub-groups (hybrid stage 1) == the split RS."""
    arrays, _ = golden
    grads = [arrays[f"hyb/w{w}f{f}/in{r}"] for r in range(w)]
    n = grads[0].size // f
    c = make_comm(w)
    try:
        a = c.alloc(1 << 20)
        ll = c.alloc(c.ll_bytes(f, n, torch.float32), 16)
        ref = [torch.empty(n, device="cuda") for _ in range(w)]
        got = [torch.empty(n, device="cuda") for _ in range(w)]
        c.reduce_scatter((f, 1), [cu(g) for g in grads], a, ref)
        c.reduce_scatter_ll((f, 1), [cu(g) for g in grads], ll, got)
        for r in range(w):
            assert got[r].cpu().numpy().tobytes() == ref[r].cpu().numpy().tobytes()
    finally:
        c.close()
