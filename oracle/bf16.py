"""ORACLE (test infrastructure only) — bfloat16 <-> float32 in integer numpy.

numpy has no bfloat16, so the low-precision dtype of the B200 build is
represented here as its uint16 bit pattern.  The conversion is IEEE
round-to-nearest-even on the upper 16 bits of the float32 pattern, NaN kept
quiet — the same rounding `torch.Tensor.to(torch.bfloat16)` and the CUDA
`__float2bfloat16_rn` intrinsic perform (pinned in tests against torch).

Reference context: shardsim casts full -> low before the all-gather
(`engine.py:661-662`) with low = float32; the B200 build's low is bf16.
"""
from __future__ import annotations

import numpy as np


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 array -> uint16 bf16 bit patterns (RNE, quiet NaN)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    rounded = (u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    out = rounded.astype(np.uint16)
    nan = np.isnan(x)
    if nan.any():
        out[nan] = ((u[nan] >> np.uint64(16)) | np.uint64(0x40)).astype(np.uint16)
    return out


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    """uint16 bf16 bit patterns -> float32 (exact)."""
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


def round_to_bf16(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest bf16 value, returned as float32."""
    return bf16_bits_to_f32(f32_to_bf16_bits(x))
