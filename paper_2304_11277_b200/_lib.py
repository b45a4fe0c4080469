"""ctypes binding of the C ABI declared in include/fsdp_b200.h.

This is the whole Python <-> CUDA boundary: plain pointers, sizes and stream
handles.  The shared library is built in-tree (`build.py`); if it is missing
the import fails loudly — there is no CPU or eager fallback.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_fsdp_b200.so")

F32, BF16 = 0, 1
E_INVALID, E_TIMEOUT, E_IPC, E_UNSUPPORTED = 10001, 10002, 10003, 10004
CH_AG, CH_RS, CH_AR, CH_SCALAR = 0, 1, 2, 3
MAX_RANKS, MAX_CTAS, MAX_TENSORS, IPC_HANDLE_BYTES = 8, 160, 96, 64
HANDLE_FABRIC, HANDLE_POSIX_FD, SHAREABLE_BYTES = 1, 2, 64


class FsdpCudaError(RuntimeError):
    """A C-ABI call returned non-zero (cudaError_t or FSDP_E_*)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[fsdp_b200 rc={code}] {msg}")
        self.code = code


class FsdpTimeoutError(FsdpCudaError):
    """A cross-GPU flag wait timed out on device (shardsim DeadlockError analogue)."""


if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        f"(python -m paper_2304_11277_b200.build, or __graft_entry__.build()). "
        f"There is no CPU fallback.")

lib = C.CDLL(LIB_PATH)

_vp, _i64, _i32, _f32 = C.c_void_p, C.c_int64, C.c_int, C.c_float
_vpp = C.POINTER(C.c_void_p)
_i64p = C.POINTER(C.c_int64)
_fpp = C.POINTER(C.c_void_p)

_SIGS = {
    "fsdp_last_error": (C.c_char_p, []),
    "fsdp_abi_version": (_i32, []),
    "fsdp_launch_count": (C.c_uint64, []),
    "fsdp_num_sms": (_i32, [_i32]),
    "fsdp_flatten": (_i32, [_vpp, _i64p, _i64p, _i32, _i32, _vp, _i64, _i32, _i32, _vp]),
    "fsdp_unflatten": (_i32, [_vp, _i32, _vpp, _i64p, _i64p, _i32, _i32, _vp]),
    "fsdp_shard_copy": (_i32, [_vp, _vp, _i64, _i32, _i32, _vp]),
    "fsdp_cast": (_i32, [_vp, _i32, _vp, _i32, _i64, _vp]),
    "fsdp_unscale_found_inf": (_i32, [_vp, _i64, _f32, _vp, _vp]),
    "fsdp_adam_step": (_i32, [_vp, _vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _f32, _f32,
                              _f32, _f32, _vp, _vp, _vp]),
    "fsdp_sgd_step": (_i32, [_vp, _vp, _i64, _f32, _vp, _vp, _vp]),
    "fsdp_adam_step_bf16g": (_i32, [_vp, _vp, _vp, _vp, _i64, _f32, _f32, _f32, _f32, _f32, _f32,
                                    _f32, _f32, _vp, _vp, _vp]),
    "fsdp_sgd_step_bf16g": (_i32, [_vp, _vp, _i64, _f32, _vp, _vp, _vp]),
    "fsdp_comm_create": (_i32, [_i32, _i32, _i64, _i32, C.POINTER(_vp)]),
    "fsdp_comm_create_emulated": (_i32, [_i32, _i64, _i32, C.POINTER(_vp)]),
    "fsdp_comm_ipc_handle": (_i32, [_vp, _vp]),
    "fsdp_comm_open_peers": (_i32, [_vp, _vp]),
    "fsdp_comm_pool_ptr": (_vp, [_vp, _i32]),
    "fsdp_comm_pool_bytes": (_i64, [_vp]),
    "fsdp_comm_reserved_bytes": (_i64, []),
    "fsdp_comm_device_error": (_i32, [_vp]),
    "fsdp_comm_set_timeout_ms": (_i32, [_vp, _i64]),
    "fsdp_comm_fold_error": (_i32, [_vp, _vp, _i32, _vp, _vp]),
    "fsdp_comm_clear_error": (_i32, [_vp]),
    "fsdp_comm_timeout_info": (_i32, [_vp, C.POINTER(C.c_uint32)]),
    "fsdp_comm_set_fault": (_i32, [_vp, _i32]),
    "fsdp_comm_set_mode": (_i32, [_vp, _i32, _i32]),
    "fsdp_comm_set_barriers": (_i32, [_vp, _i32]),
    "fsdp_comm_set_ctas": (_i32, [_vp, _i32, _i32]),
    "fsdp_comm_timing_drain": (_i32, [_vp, _i32, C.POINTER(C.c_float), _i32, C.POINTER(_i32)]),
    "fsdp_comm_destroy": (_i32, [_vp]),
    "fsdp_allgather": (_i32, [_vp, _i32, _i32, _i32, _vpp, _i32, _i64, _i64, _i32, _vp]),
    "fsdp_reduce_scatter": (_i32, [_vp, _i32, _i32, _i32, _vpp, _i32, _i64, _i64, _vpp, _f32,
                                   _f32, _i32, _vp]),
    "fsdp_reduce_scatter_pull": (_i32, [_vp, _i32, _i32, _i32, _i64, _i32, _i64, _vpp, _f32, _f32,
                                        _i32, _vp]),
    "fsdp_reduce_scatter_tma": (_i32, [_vp, _i32, _i32, _i32, _i64, _i32, _i64, _vpp, _f32, _f32,
                                       _i32, _vp]),
    "fsdp_allgather_ce": (_i32, [_vp, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _vp]),
    "fsdp_reduce_scatter_ce": (_i32, [_vp, _i32, _i32, _i32, _i64, _i32, _i64, _i64, _vp, _f32,
                                      _f32, _i32, _vp]),
    "fsdp_reduce_scatter_ce_out": (_i32, [_vp, _i32, _i32, _i32, _i64, _i32, _i64, _i64, _vp, _i32,
                                          _f32, _f32, _i32, _vp]),
    "fsdp_allreduce": (_i32, [_vp, _i32, _i32, _i32, _vpp, _i32, _i64, _i64, _i64, _vpp, _f32,
                              _i32, _vp]),
    "fsdp_allreduce_ce": (_i32, [_vp, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _i64, _vp, _f32, _i32, _vp]),
    "fsdp_allreduce_ce_pool": (_i32, [_vp, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _i64, _f32, _vp]),
    "fsdp_allreduce_scalar": (_i32, [_vp, _vpp, _vpp, _vp]),
    "fsdp_ll_bytes": (_i64, [_i32, _i64, _i32]),
    "fsdp_allgather_ll": (_i32, [_vp, _i32, _i32, _i32, _vpp, _i32, _i64, _i64, _i32, _i64, _vp]),
    "fsdp_reduce_scatter_ll": (_i32, [_vp, _i32, _i32, _i32, _vpp, _i32, _i64, _i64, _vpp, _f32,
                                      _f32, _i32, _vp]),
    "fsdp_nvls_supported": (_i32, [_i32]),
    "fsdp_comm_create_vmm": (_i32, [_i32, _i32, _i64, _i32, _i32, C.POINTER(_vp)]),
    "fsdp_comm_export_pool": (_i32, [_vp, _vp]),
    "fsdp_comm_import_pool": (_i32, [_vp, _i32, _vp]),
    "fsdp_nvls_create": (_i32, [_vp, _i32, _vp]),
    "fsdp_nvls_import": (_i32, [_vp, _i32, _vp]),
    "fsdp_nvls_add_device": (_i32, [_vp]),
    "fsdp_nvls_bind": (_i32, [_vp]),
    "fsdp_nvls_group_size": (_i32, [_vp]),
    "fsdp_allgather_nvls": (_i32, [_vp, _i32, _i32, _i32, _vp, _i32, _i64, _i64, _i32, _vp]),
}

EXPORTS = tuple(_SIGS)

for _name, (_res, _args) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return lib.fsdp_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        cls = FsdpTimeoutError if rc == E_TIMEOUT else FsdpCudaError
        raise cls(rc, f"{what}: {last_error()}" if what else last_error())


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr


def i64_array(vals) -> "C.Array":
    arr = (C.c_int64 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def launch_count() -> int:
    return int(lib.fsdp_launch_count())
