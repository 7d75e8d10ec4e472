"""CPU checks of the C-ABI library: it loads (no GPU needed) and exports every
function include/kvtc.h declares; the binding declares exactly those."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_01815_b200", "libkvtc.so")


def _declared():
    src = open(os.path.join(ROOT, "include", "kvtc.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kvtc_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def built():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return LIB


def test_header_declares_the_paper_entry_points():
    names = _declared()
    for n in ("kvtc_calibrate", "kvtc_allocate_bits", "kvtc_compress", "kvtc_decompress"):
        assert n in names


def test_library_exports_every_declared_symbol(built):
    out = subprocess.check_output(["nm", "-D", "--defined-only", built]).decode()
    exported = set(re.findall(r" T (kvtc_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_matches_header(built):
    from paper_2511_01815_b200 import _lib
    L = _lib.lib()
    assert L.kvtc_abi_version() == 2
    assert sorted(_lib.exported_symbols()) == _declared()


def test_library_is_sm100a_only(built):
    out = subprocess.check_output(["cuobjdump", "--list-elf", built]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", built]).decode()
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "tcgen05.mma missing from the SASS"
    assert "UTMALDG" in sass, "TMA loads missing from the SASS"


@pytest.mark.parametrize("size,typ", [(17, 2), (18, 1), (300, 1), (257, 3), (0, 1)])
def test_plan_create_rejects_sizes_the_kernels_cannot_pack(built, size, typ):
    """sub-byte tokens wider than one 32-bit word (17 x int4 = 68 bits)
    or wide groups that are not whole 256-column pieces are refused before any
    device work (so this runs without a GPU)."""
    import ctypes as C
    import numpy as np
    from paper_2511_01815_b200 import _lib
    L = _lib.lib()
    st, sz, tp = (np.array([v], dtype=np.int32) for v in (0, size, typ))
    out = C.c_void_p()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))
    rc = L.kvtc_plan_create(2048, 1, p(st), p(sz), p(tp), C.byref(out))
    assert rc == -1
    assert b"group" in L.kvtc_last_error()
