"""Thin typed wrappers over the copy / optimizer entry points of the C ABI.

All functions enqueue on `stream` (default: torch's current stream) and never
synchronise.  Inputs must be contiguous CUDA tensors; dtypes fp32 or bf16.
"""
from __future__ import annotations

from typing import Sequence

import torch

from . import _lib
from ._lib import check, lib
from .comm import dtype_code, stream_ptr


def _cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous CUDA tensor")


def flatten(tensors: Sequence[torch.Tensor | None], offsets: Sequence[int], flat: torch.Tensor,
            accumulate: bool = False, stream=None) -> None:
    """flat[off_i : off_i + numel_i] = cast(t_i); every other element 0 (or
    unchanged with accumulate=True, then flat += values).  None = zero-fill
    (a parameter without gradient, flatparam.py:181-185)."""
    _cuda(flat, "flatten")
    real = [t for t in tensors if t is not None]
    src_dt = real[0].dtype if real else flat.dtype
    for t in real:
        if t.dtype != src_dt:
            raise ValueError("flatten: all sources must share one dtype")
        _cuda(t, "flatten source")
    numels = [(t.numel() if t is not None else 0) for t in tensors]
    # a None keeps its slot in the table with numel 0 (zero-filled region)
    ptrs = [(t.data_ptr() if t is not None else 0) for t in tensors]
    for start in range(0, max(1, len(tensors)), _lib.MAX_TENSORS):
        chunk = slice(start, start + _lib.MAX_TENSORS)
        n = len(ptrs[chunk])
        first = start == 0
        check(lib.fsdp_flatten(_lib.ptr_array(ptrs[chunk]), _lib.i64_array(numels[chunk]),
                               _lib.i64_array(offsets[chunk]), n, dtype_code(src_dt),
                               flat.data_ptr(), flat.numel(), dtype_code(flat.dtype),
                               int(accumulate or not first), stream_ptr(stream)), "flatten")


def unflatten(flat: torch.Tensor, outs: Sequence[torch.Tensor], offsets: Sequence[int],
              stream=None) -> None:
    """outs[i] = flat[off_i : off_i + numel_i] (cast to outs[i].dtype)."""
    if not outs:
        return
    dt = outs[0].dtype
    for o in outs:
        _cuda(o, "unflatten dst")
        if o.dtype != dt:
            raise ValueError("unflatten: outputs must share one dtype")
    for start in range(0, len(outs), _lib.MAX_TENSORS):
        chunk = outs[start:start + _lib.MAX_TENSORS]
        check(lib.fsdp_unflatten(flat.data_ptr(), dtype_code(flat.dtype),
                                 _lib.ptr_array([o.data_ptr() for o in chunk]),
                                 _lib.i64_array([o.numel() for o in chunk]),
                                 _lib.i64_array(offsets[start:start + _lib.MAX_TENSORS]),
                                 len(chunk), dtype_code(dt), stream_ptr(stream)), "unflatten")


def shard_copy(flat: torch.Tensor, shard: torch.Tensor, shard_index: int, stream=None) -> None:
    """shard = flat[k*n:(k+1)*n] (FlatParameter.shard, flatparam.py:139-147)."""
    _cuda(flat, "shard_copy")
    _cuda(shard, "shard_copy")
    if flat.dtype != shard.dtype:
        raise ValueError("shard_copy: dtype mismatch")
    n = shard.numel()
    if (shard_index + 1) * n > flat.numel():
        raise ValueError("shard_copy: shard range outside the flat buffer")
    check(lib.fsdp_shard_copy(flat.data_ptr(), shard.data_ptr(), n, int(shard_index),
                              dtype_code(flat.dtype), stream_ptr(stream)), "shard_copy")


def cast(src: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    _cuda(src, "cast")
    _cuda(dst, "cast")
    if src.numel() != dst.numel():
        raise ValueError("cast: size mismatch")
    check(lib.fsdp_cast(src.data_ptr(), dtype_code(src.dtype), dst.data_ptr(),
                        dtype_code(dst.dtype), src.numel(), stream_ptr(stream)), "cast")


def _f32(x: float) -> float:
    import numpy as np
    return float(np.float32(x))


def adam_scalars(lr: float, betas: tuple[float, float], eps: float, t: int) -> tuple:
    """float32 roundings of the python-double expressions numerics.py:278-285
    evaluates (NEP 50 weak scalars)."""
    b1, b2 = betas
    return (_f32(lr), _f32(b1), _f32(1.0 - b1), _f32(b2), _f32(1.0 - b2),
            _f32(1.0 - b1 ** t), _f32(1.0 - b2 ** t), _f32(eps))


def adam_step(p: torch.Tensor, g: torch.Tensor, m: torch.Tensor, v: torch.Tensor, *, lr: float,
              betas: tuple[float, float], eps: float, t: int, skip_flag: torch.Tensor | None = None,
              p_lowp: torch.Tensor | None = None, stream=None) -> None:
    for x in (p, g, m, v):
        _cuda(x, "adam_step")
        if x.numel() != p.numel() or x.dtype != (torch.float32 if (x is not g or g.dtype != torch.bfloat16)
                                                 else torch.bfloat16):
            raise ValueError("adam_step: param/state fp32 and grad fp32 or bf16, of equal length")
    s = adam_scalars(lr, betas, eps, t)
    fn = lib.fsdp_adam_step_bf16g if g.dtype == torch.bfloat16 else lib.fsdp_adam_step
    check(fn(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(),
                             *s, skip_flag.data_ptr() if skip_flag is not None else None,
                             p_lowp.data_ptr() if p_lowp is not None else None,
                             stream_ptr(stream)), "adam_step")


def sgd_step(p: torch.Tensor, g: torch.Tensor, *, lr: float, skip_flag=None, p_lowp=None,
             stream=None) -> None:
    _cuda(p, "sgd_step")
    _cuda(g, "sgd_step")
    if g.dtype not in (torch.float32, torch.bfloat16) or g.numel() != p.numel():
        raise ValueError("sgd_step: grad must be fp32 or bf16 of the param's length")
    fn = lib.fsdp_sgd_step_bf16g if g.dtype == torch.bfloat16 else lib.fsdp_sgd_step
    check(fn(p.data_ptr(), g.data_ptr(), p.numel(), _f32(lr),
                            skip_flag.data_ptr() if skip_flag is not None else None,
                            p_lowp.data_ptr() if p_lowp is not None else None,
                            stream_ptr(stream)), "sgd_step")


def unscale_found_inf(g: torch.Tensor, inv_scale: float, found_inf: torch.Tensor,
                      stream=None) -> None:
    _cuda(g, "unscale_found_inf")
    check(lib.fsdp_unscale_found_inf(g.data_ptr(), g.numel(), _f32(inv_scale),
                                     found_inf.data_ptr(), stream_ptr(stream)), "unscale_found_inf")
