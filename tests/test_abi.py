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
    assert L.kvtc_abi_version() == 1
    assert sorted(_lib.exported_symbols()) == _declared()


def test_library_is_sm100a_only(built):
    out = subprocess.check_output(["cuobjdump", "--list-elf", built]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", built]).decode()
    assert "UTCHMMA" in sass or "UTCMMA" in sass, "tcgen05.mma missing from the SASS"
    assert "UTMALDG" in sass, "TMA loads missing from the SASS"
