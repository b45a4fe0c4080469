"""The C ABI boundary without a GPU: the shared library loads, exports every
function include/fsdp_b200.h declares, the ctypes binding covers exactly that
set, and argument validation fails loudly (no device work is needed for any
call made here)."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fsdp_b200.h")


def declared() -> set[str]:
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(fsdp_\w+)\s*\(", src, flags=re.M))


@pytest.fixture(scope="module")
def lib():
    from paper_2304_11277_b200 import build
    build.build()
    from paper_2304_11277_b200 import _lib
    return _lib


def test_header_parses():
    names = declared()
    assert len(names) > 30
    for must in ("fsdp_flatten", "fsdp_allgather", "fsdp_reduce_scatter", "fsdp_adam_step",
                 "fsdp_allgather_nvls", "fsdp_comm_create_vmm"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(declared()) if not hasattr(lib.lib, n)]
    assert not missing, f"declared in fsdp_b200.h but not exported: {missing}"


def test_ctypes_binding_matches_header(lib):
    assert set(lib.EXPORTS) == declared()


def test_calls_without_a_device(lib):
    L = lib.lib
    assert L.fsdp_abi_version() >= 1
    assert L.fsdp_comm_reserved_bytes() == 65536
    # argument validation returns FSDP_E_INVALID before touching a device
    assert L.fsdp_cast(None, lib.F32, None, lib.BF16, -1, None) == lib.E_INVALID
    assert b"negative" in L.fsdp_last_error()
    assert L.fsdp_cast(None, 7, None, lib.BF16, 4, None) == lib.E_INVALID
    assert L.fsdp_shard_copy(None, None, 4, -1, lib.F32, None) == lib.E_INVALID
    h = C.c_void_p()
    assert L.fsdp_comm_create(0, 9, 1 << 20, 32, C.byref(h)) == lib.E_INVALID
    assert L.fsdp_comm_create(0, 2, 1 << 20, 500, C.byref(h)) == lib.E_INVALID
    assert L.fsdp_comm_create_vmm(0, 2, 1 << 20, 32, 3, C.byref(h)) == lib.E_INVALID
    assert L.fsdp_comm_set_ctas(None, 0, 8) == lib.E_INVALID
    assert L.fsdp_nvls_add_device(None) == lib.E_INVALID
    assert L.fsdp_comm_pool_bytes(None) == -1
    # the Python wrapper raises with the library's message
    with pytest.raises(lib.FsdpCudaError, match="negative"):
        lib.check(L.fsdp_cast(None, lib.F32, None, lib.BF16, -1, None), "cast")
