"""Host logic added for the drop-in wrapper and the CLI, no GPU needed:
shard-group size from torch-FSDP's ways of naming it (hybrid_shard_size,
DeviceMesh, group tuple; collectives.py:63-72, :89-96), the memory ledger
and its closed-form peak (memsim.py:113-185, flatparam.py:198-235), the
sweep axis parser (cli.py:626-654) and the fault-hook validation."""
from fractions import Fraction

import pytest
import torch

from paper_2304_11277_b200.__main__ import _parse_axis
from paper_2304_11277_b200.fsdp import _shard_factor_from
from paper_2304_11277_b200.ledger import CATEGORIES, MemoryLedger, peak_param_bytes


class _Mesh:
    def __init__(self, mesh, names=None):
        self.mesh = torch.as_tensor(mesh)
        self.mesh_dim_names = names


def test_hybrid_size_from_mesh_and_kwarg():
    assert _shard_factor_from(None, None, 4, True, False) == 4
    assert _shard_factor_from(None, _Mesh([[0, 1, 2, 3], [4, 5, 6, 7]], ("replicate", "shard")),
                              None, True, False) == 4
    assert _shard_factor_from(None, _Mesh([[0, 1], [2, 3], [4, 5], [6, 7]]), None, True, False) == 2
    # (shard, replicate) order is transposed to the convention
    assert _shard_factor_from(None, _Mesh([[0, 4], [1, 5], [2, 6], [3, 7]], ("shard", "replicate")),
                              None, True, False) == 4
    assert _shard_factor_from(None, _Mesh([0, 1, 2, 3]), None, False, False) == 4
    # nothing names F: the wrapper raises for HYBRID (returns None here)
    assert _shard_factor_from(None, None, None, True, False) is None
    # hybrid_shard_size is ignored by FULL/NO_SHARD
    assert _shard_factor_from(None, None, 2, False, False) is None


def test_mesh_convention_enforced():
    with pytest.raises(ValueError, match="convention"):
        _shard_factor_from(None, _Mesh([[0, 2], [1, 3]]), None, True, False)
    with pytest.raises(ValueError, match="inconsistent"):
        _shard_factor_from(None, _Mesh([[0, 1], [2, 3]]), 4, True, False)
    with pytest.raises(ValueError, match="1-D"):
        _shard_factor_from(None, _Mesh(torch.zeros(2, 2, 2, dtype=torch.int64)), None, True, False)


def test_ledger_peaks_and_reset():
    L = MemoryLedger()
    L.alloc("sharded_params", 600, 100)
    L.alloc("unsharded_params", 400, 200)
    L.free("unsharded_params", 400, 200)
    L.alloc("unsharded_params", 300, 150)
    assert L.peak_param_bytes == 1000 and L.peak_param_elements == 300
    L.set_level("activations", 50)
    assert L.peak_total_bytes == 1000
    old = L.reset_peaks()
    assert old["peak_param_bytes"] == 1000
    assert L.peak_param_bytes == 900 and L.peak_total_bytes == 950
    with pytest.raises(AssertionError):
        L.free("grads", 1, 1)
    assert set(L.snapshot()["peak_bytes"]) == set(CATEGORIES)


def test_peak_formula_matches_reference_shape():
    psis, F = [40, 72, 24], 4                       # dump-plan golden units (test_cli.py:221-233)
    shards = [p // F for p in psis]
    # reference flatparam.py:198-235 with k_full=8, fp64 shards, no low copy
    ref_bytes = Fraction(sum(psis), F) * 8 + max(psis) * 8
    assert peak_param_bytes(psis, shards, F, k_full=8, k_low=None, low_copy=False) == ref_bytes
    # mixed precision: fp32 master + bf16 copy resident, bf16 gathered
    assert peak_param_bytes(psis, shards, F) == sum(shards) * 6 + 72 * 2
    assert peak_param_bytes(psis, shards, F, variant="two_inflight") == sum(shards) * 6 + (72 + 40) * 2
    assert peak_param_bytes(psis, psis, 1) == sum(psis) * 6                 # F = 1 gathers nothing
    # wrapper nesting: the root (unit 0) stays gathered under every child
    assert peak_param_bytes(psis, shards, F, nested_root=True) == sum(shards) * 6 + (40 + 72) * 2
    # the tiny GPT fp32 verify case measured on the GPU: 8,090,624 bytes at F = 2
    tiny = [295424, 789760, 789760]
    assert peak_param_bytes(tiny, [p // 2 for p in tiny], 2, k_low=None, low_copy=False,
                            nested_root=True) == 8090624


def test_sweep_axis_parser():
    assert _parse_axis("F=1,2,4", 4) == ("sharding_factor", [1, 2, 4])
    assert _parse_axis("rate_limit=1,none", 4) == ("rate_limit", [1, None])
    assert _parse_axis("raf=RAF,NRAF", 2) == ("raf", ["RAF", "NRAF"])
    assert _parse_axis("prefetch=on,off", 2) == ("prefetch", ["on", "off"])
    for bad in ("F=3", "W=2", "raf=X", "prefetch=maybe", "nope=1", "F"):
        with pytest.raises(ValueError):
            _parse_axis(bad, 4)
