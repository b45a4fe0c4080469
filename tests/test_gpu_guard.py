"""Out-of-bounds write checks (guard bands), in place of compute-sanitizer,
which this GPU pool does not offer: every destination is a window inside a
larger buffer filled with a canary byte pattern, and after the kernel the
bytes on both sides of the window must still be canary.  Covers ragged and
unaligned lengths (the scalar tails) of the layout, optimizer and collective
kernels, including the symmetric-pool regions the collectives write."""
import pytest
import torch

pytestmark = pytest.mark.gpu

CANARY = 0xA5
GUARD = 4096   # bytes on each side


def guarded(numel: int, dtype: torch.dtype, lead_elems: int = 0):
    """(window, check) -- window has `numel` elements, starting `lead_elems`
    elements after a GUARD-byte band (so its alignment can be varied)."""
    es = torch.tensor([], dtype=dtype).element_size()
    lead = GUARD + lead_elems * es
    raw = torch.full((lead + numel * es + GUARD,), CANARY, dtype=torch.uint8, device="cuda")
    win = raw[lead: lead + numel * es].view(dtype)

    def check():
        torch.cuda.synchronize()
        assert bool((raw[:lead] == CANARY).all()), "write before the window"
        assert bool((raw[lead + numel * es:] == CANARY).all()), "write after the window"
    return win, check


@pytest.mark.parametrize("lead", [0, 1, 3])
@pytest.mark.parametrize("sd,fd", [(torch.float32, torch.float32), (torch.bfloat16, torch.bfloat16),
                                   (torch.bfloat16, torch.float32), (torch.float32, torch.bfloat16)])
def test_layout_kernels_stay_in_bounds(lead, sd, fd):
    from paper_2304_11277_b200 import kernels
    shapes = [(3, 5), (17,), (64, 33), (1,), (1001,)]
    ts = [torch.randn(s, device="cuda").to(sd) for s in shapes]
    offs, o = [], 0
    for t in ts:
        offs.append(o)
        o += t.numel() + 3
    psi = o + 5
    flat, chk = guarded(psi, fd, lead)
    kernels.flatten(ts, offs, flat)
    kernels.flatten(ts, offs, flat, accumulate=True)
    chk()
    outs, chks = zip(*[guarded(t.numel(), sd, lead) for t in ts])
    kernels.unflatten(flat, [w.view(t.shape) for w, t in zip(outs, ts)], offs)
    for c in chks:
        c()
    sh, chk = guarded(psi // 4, fd, lead)
    kernels.shard_copy(flat, sh, 2)
    chk()
    dst, chk = guarded(psi, sd, lead)
    kernels.cast(flat, dst)
    chk()


@pytest.mark.parametrize("n", [1003, 6144 * 148 + 6144 * 3 + 7])
@pytest.mark.parametrize("lead", [0, 16])
def test_optimizer_kernels_stay_in_bounds(n, lead):
    from paper_2304_11277_b200 import kernels
    bufs = [guarded(n, torch.float32, lead) for _ in range(4)]
    (p, cp), (g, cg), (m, cm), (v, cv) = bufs
    p.copy_(torch.randn(n)); g.copy_(torch.randn(n) * 1e-2); m.zero_(); v.zero_()
    low, cl = guarded(n, torch.bfloat16, lead)
    kernels.adam_step(p, g, m, v, lr=1e-3, betas=(0.9, 0.999), eps=1e-8, t=1, p_lowp=low)
    kernels.sgd_step(p, g, lr=1e-3, p_lowp=low)
    found = torch.zeros(1, device="cuda")
    kernels.unscale_found_inf(g, 0.5, found)
    for c in (cp, cg, cm, cv, cl):
        c()


@pytest.mark.parametrize("w", [2, 4])
@pytest.mark.parametrize("n", [4099, 65536 + 24])
@pytest.mark.parametrize("lead", [0, 1])
def test_collectives_stay_in_their_pool_regions(w, n, lead):
    """Every collective writes only [region, region + size) of each pool
    (and its output tensors): the pools are canary-filled, the regions
    separated by canary bands that must survive."""
    from paper_2304_11277_b200.comm import DeviceComm
    c = DeviceComm.create_emulated(w, 64 << 20, max_ctas=8)
    c.set_timeout_ms(10000)
    try:
        for e in range(w):
            c._pools[e][c.reserved:].fill_(CANARY)
        regions = {}

        def region(name, nbytes):
            c.alloc(GUARD)                                   # leading band
            off = c.alloc(nbytes, 16)
            regions[name] = (off, nbytes)
            return off
        ag = region("ag", n * w * 2)
        ag_ll = region("ag_ll", n * w * 2)
        st = region("rs_stage", n * w * 2)
        pull = region("pull_src", n * w * 2)
        ar_st = region("ar_stage", c.ar_staging_elems(n * w, w) * 4)
        ar_g = region("ar_gather", c.ar_staging_elems(n * w, w) * 4)
        ll_ag = region("ll_ag", c.ll_bytes(w, n, torch.bfloat16))
        ll_rs = region("ll_rs", c.ll_bytes(w, n, torch.bfloat16))
        c.alloc(GUARD)
        shards = [torch.randn(n, device="cuda") for _ in range(w)]
        flats = [torch.randn(n * w, device="cuda").to(torch.bfloat16) for _ in range(w)]
        for e in range(w):
            c.view(pull, n * w, torch.bfloat16, e).copy_(flats[e])
        outs, chks = zip(*[guarded(n, torch.float32, lead) for _ in range(w)])
        for o in outs:
            o.zero_()
        full, fchks = zip(*[guarded(n * w, torch.float32, 3 * lead) for _ in range(w)])
        c.all_gather((w, 1), shards, ag, torch.bfloat16)
        c.all_gather_ll((w, 1), shards, ag_ll, torch.bfloat16, ll_ag)
        c.all_gather_ll((w, 1), shards, ag_ll, torch.bfloat16, ll_ag)
        c.reduce_scatter((w, 1), flats, st, list(outs), postdiv=float(w), accumulate=True)
        c.reduce_scatter_pull((w, 1), pull, torch.bfloat16, list(outs), tma=False)
        c.reduce_scatter_pull((w, 1), pull, torch.bfloat16, list(outs), tma=True)
        c.reduce_scatter_ll((w, 1), flats, ll_rs, list(outs), accumulate=True)
        c.reduce_scatter_ll((w, 1), flats, ll_rs, list(outs), accumulate=True)
        c.all_reduce((w, 1), [f.float() for f in flats], ar_st, ar_g, list(full))
        torch.cuda.synchronize()
        assert c.device_error() == 0
        for ck in chks + fchks:
            ck()
        # every pool byte outside the named regions is still canary
        for e in range(w):
            pool = c._pools[e]
            mask = torch.ones(c._cursor, dtype=torch.bool, device="cuda")
            mask[:c.reserved] = False
            for off, nb in regions.values():
                mask[off: off + nb] = False
            assert bool((pool[:c._cursor][mask] == CANARY).all()), f"pool {e}: write outside the regions"
    finally:
        c.close()
