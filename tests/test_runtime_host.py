"""Host-side sizing of the symmetric pool (no GPU): the low-latency regions
that `FSDPRuntime._alloc_pool_regions` carves must be covered by
`FSDPRuntime.pool_bytes_for`, and the Python formula must agree with the
C ABI's `fsdp_ll_bytes`."""
import pytest

from paper_2304_11277_b200._lib import BF16, F32, lib
from paper_2304_11277_b200.layout import build_unit_layouts
from paper_2304_11277_b200.plan import build_plan
from paper_2304_11277_b200.runtime import FSDPRuntime, RuntimeConfig


@pytest.mark.parametrize("gsize", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 3, 4, 7, 1000, 262147])
def test_ll_bytes_formula(gsize, n):
    for dt, es in ((F32, 4), (BF16, 2)):
        lines = -(-(n * es) // 8)                 # 8 payload bytes per 16-byte line
        blocks = -(-lines // 32)                  # whole 32-line blocks
        assert lib.fsdp_ll_bytes(gsize, n, dt) == 2 * gsize * blocks * 32 * 16
    assert lib.fsdp_ll_bytes(0, 8, F32) == -1
    assert lib.fsdp_ll_bytes(2, 8, 7) == -1


def _layouts(F):
    # root (0.59 MB bf16) + two 1.6 MB blocks + one 40 MB block at F
    shapes = [("root.w", (295424,)), ("b0.w", (789760,)), ("b1.w", (789760,)), ("big.w", (5000, 4096))]
    names = [["root.w"], ["b0.w"], ["b1.w"], ["big.w"]]
    return build_unit_layouts(shapes, names, F)


@pytest.mark.parametrize("W,F", [(2, 2), (4, 4), (4, 2), (8, 8)])
def test_pool_bytes_cover_ll_regions(W, F):
    lays = _layouts(F)
    plan = build_plan(W, F)
    on = RuntimeConfig(ll_max_bytes=6 << 20)
    off = RuntimeConfig(ll_max_bytes=0)
    extra = FSDPRuntime.pool_bytes_for(lays, plan, on) - FSDPRuntime.pool_bytes_for(lays, plan, off)
    small = [l for l in lays if l.psi * 2 <= on.ll_max_bytes]
    assert len(small) == 3                          # the 40 MB unit stays on the split path
    n = max(l.shard_numel for l in small)
    need = 2 * lib.fsdp_ll_bytes(F, n, BF16)        # one region per channel (AG, RS)
    assert need <= extra <= need + 2 * 512          # + allocator alignment padding


def test_ll_threshold_is_the_unsharded_payload():
    lays = _layouts(4)
    plan = build_plan(4, 4)
    cfg = RuntimeConfig(ll_max_bytes=(789760 * 2) - 1)   # the blocks just miss the threshold
    base = FSDPRuntime.pool_bytes_for(lays, plan, RuntimeConfig(ll_max_bytes=0))
    extra = FSDPRuntime.pool_bytes_for(lays, plan, cfg) - base
    n_root = next(l for l in lays if l.unit_id == 0).shard_numel
    assert extra >= 2 * lib.fsdp_ll_bytes(4, n_root, BF16)
    assert extra < 2 * lib.fsdp_ll_bytes(4, lays[1].shard_numel, BF16)
