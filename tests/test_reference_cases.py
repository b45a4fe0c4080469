"""Known-answer cases of the reference's own tests and SPEC examples, ported
(no GPU): the oracle and this package's host logic must give the reference's
answers.

Sources (relative to /root/reference): pkg/tests/test_flatparam.py:74-170,
pkg/tests/test_collectives.py:125-160.
"""
import numpy as np
import pytest
import torch

from oracle import shardsim_port as sp
from paper_2304_11277_b200 import layout as L
from paper_2304_11277_b200.comm import DeviceFabric
from paper_2304_11277_b200.plan import CollectiveError

TWO_UNIT = [("a.weight", (2, 3)), ("a.bias", (2,)), ("b.weight", (3, 3))]
TWO_UNIT_NAMES = [["a.weight", "a.bias"], ["b.weight"]]


def test_shard_gather_views_write_through_roundtrip():
    """test_flatparam.py:74-99: unit b (psi 12, shard 3) at W = F = 4."""
    lay = sp.build_unit_layouts(TWO_UNIT, TWO_UNIT_NAMES, 4)[1]
    assert (lay.psi, lay.shard_numel) == (12, 3)
    full = np.arange(12.0)
    shards = [sp.shard(full, lay, r) for r in range(4)]
    gathered = sp.all_gather(shards)
    assert np.array_equal(gathered, full)
    views = sp.unflatten(gathered, lay)
    assert np.array_equal(views["b.weight"], full[:9].reshape(3, 3))
    gathered[0] = 99.0                        # write-through of the b.weight[0, 0] view
    assert sp.shard(gathered, lay, 0)[0] == 99.0      # rank 0 owns offset 0
    assert sp.shard(gathered, lay, 1)[0] == full[3]


def test_trivial_f1_unit_is_the_whole_buffer():
    """test_flatparam.py:116-126: F = 1, the shard is the unsharded buffer."""
    for build in (sp.build_unit_layouts, L.build_unit_layouts):
        lay = build([("w", (3,))], [["w"]], 1)[0]
        assert (lay.psi, lay.padding, lay.shard_numel) == (3, 0, 3)
    flat = np.array([5.0, 2.0, 3.0])
    assert np.array_equal(sp.shard(flat, sp.build_unit_layouts([("w", (3,))], [["w"]], 1)[0], 0), flat)


def test_writeback_offsets_padding_missing_and_shape():
    """test_flatparam.py:141-170."""
    la, lb = sp.build_unit_layouts(TWO_UNIT, TWO_UNIT_NAMES, 4)
    flat, warns = sp.writeback_grad(lb, {"b.weight": np.ones((3, 3))}, np.float64)
    assert warns == [] and np.array_equal(flat[:9], np.ones(9)) and np.array_equal(flat[9:], np.zeros(3))
    flat, warns = sp.writeback_grad(la, {"a.weight": np.zeros((2, 3))}, np.float64)
    assert len(warns) == 1 and "a.bias" in warns[0] and np.array_equal(flat, np.zeros(8))
    with pytest.raises(sp.FlatParamError):
        sp.writeback_grad(la, {"a.weight": np.zeros((3, 2)), "a.bias": np.zeros(2)}, np.float64)
    out = np.full(8, 7.0)
    flat, _ = sp.writeback_grad(la, {"a.weight": np.ones((2, 3)), "a.bias": np.ones(2)}, np.float64, out=out)
    assert flat is out and np.array_equal(out, np.ones(8))


def test_spec_layout_examples():
    """4x3 weight at F = 16 -> psi 16, shard 1 (the last
    ranks hold padding); {2x2, 3} at F = 4 -> psi 8, padding 1, shard 2."""
    for build in (sp.build_unit_layouts, L.build_unit_layouts):
        lay = build([("w", (4, 3))], [["w"]], 16)[0]
        assert (lay.psi, lay.padding, lay.shard_numel) == (16, 4, 1)
        lay = build([("x", (2, 2)), ("y", (3,))], [["x", "y"]], 4)[0]
        assert (lay.psi, lay.padding, lay.shard_numel) == (8, 1, 2)
        lay = build([("x", (2, 2)), ("y", (3,))], [["x", "y"]], 1)[0]
        assert (lay.psi, lay.padding) == (7, 0)


def test_spec_collective_examples():
    """SPEC.md:136-157."""
    out = sp.reduce_scatter([np.array([1.0, 2, 3, 4]), np.array([10.0, 20, 30, 40])])
    assert np.array_equal(out[0], [11, 22]) and np.array_equal(out[1], [33, 44])
    assert np.array_equal(sp.all_reduce([np.array([1.0]), np.array([2.0]), np.array([3.0])]), [6.0])
    grads = [np.full(2, float(r + 1)) for r in range(4)]
    res = sp.hybrid_reduce(grads, sp.Plan(4, 2))
    assert all(np.array_equal(r, [10.0]) for r in res)
    # RS then AG == AR on 4 ranks
    rng = np.random.default_rng(0)
    xs = [rng.integers(-8, 8, 16).astype(np.float64) for _ in range(4)]
    assert np.array_equal(sp.all_gather(sp.reduce_scatter(xs)), sp.all_reduce(xs))


@pytest.mark.parametrize("W,F", [(4, 2), (8, 4), (8, 2)])
def test_hybrid_stage2_in_reduce_dtype(W, F):
    """engine.py:789-810: the reduce-scatter output is the all-reduce payload.
    stage2_dtype rounds the fp32 partial once to bf16; the all-reduce sums the
    rounded partials in fp32; F = W and F = 1 have no stage 2 to round."""
    rng = np.random.default_rng(3 + W + F)
    c = 8
    grads = [sp.cast(rng.standard_normal(c * F).astype(np.float32), sp.BF16) for _ in range(W)]
    plan = sp.Plan(W, F)
    hi = sp.hybrid_reduce(grads, plan, np.float32)
    lo = sp.hybrid_reduce(grads, plan, np.float32, stage2_dtype=sp.BF16)
    for r in range(W):
        g = [q for q in plan.sharded_groups if r in q][0]
        pos = list(g).index(r)
        parts = []
        for rr in [q for q in plan.replicated_groups if r in q][0]:       # ascending replica order
            gg = [q for q in plan.sharded_groups if rr in q][0]
            acc = np.zeros(c, np.float32)
            for m in gg:
                acc = acc + grads[m][pos * c:(pos + 1) * c].astype(np.float32)
            parts.append(sp.cast(acc, sp.BF16))
        exp = np.zeros(c, np.float32)
        for p_ in parts:
            exp = exp + p_
        assert lo[r].tobytes() == exp.tobytes()
    assert any(not np.array_equal(a, b) for a, b in zip(hi, lo))      # the rounding is visible
    for f in (1, W):                                                   # no stage 2 to round
        a = sp.hybrid_reduce(grads, sp.Plan(W, f), np.float32)
        b = sp.hybrid_reduce(grads, sp.Plan(W, f), np.float32, stage2_dtype=sp.BF16)
        assert all(x.tobytes() == y.tobytes() for x, y in zip(a, b))


def test_kth_call_pairs_with_kth_call():
    """test_collectives.py:125-138, as the sequence of two gathers."""
    first = sp.all_gather([np.array([0.0]), np.array([1.0])])
    second = sp.all_gather([np.array([10.0]), np.array([11.0])])
    assert np.array_equal(first, [0, 1]) and np.array_equal(second, [10, 11])


class _StubComm:
    """Enough of DeviceComm for DeviceFabric's host-side entry checks."""
    world, emulated, nranks_local = 2, False, 1

    def alloc(self, nbytes, align=256):
        return 65536


def test_fabric_entry_validation_matches_reference():
    """test_collectives.py:141-160: non-member, non-flat, indivisible RS and
    uneven lengths raise CollectiveError synchronously, before any device
    work (the stub communicator has none)."""
    fab = DeviceFabric(_StubComm(), 1 << 20)
    with pytest.raises(CollectiveError):
        fab.all_gather(3, (0, 1), torch.zeros(2))
    with pytest.raises(CollectiveError):
        fab.all_gather(0, (0, 1), torch.zeros(2, 2))
    with pytest.raises(CollectiveError):
        fab.reduce_scatter(0, (0, 1), torch.zeros(3))
    with pytest.raises(CollectiveError):
        fab.all_gather(0, (0, 1), [torch.zeros(2), torch.zeros(3)])
    with pytest.raises(CollectiveError):
        fab.all_gather(0, (0, 2, 3), torch.zeros(2))       # not a device-addressable group
