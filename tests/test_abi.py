"""libsplatct.so builds for sm_100a, loads, and exports every C-ABI symbol
declared in include/splatct.h (no GPU calls)."""
import ctypes
import os
import re
import subprocess

from paper_2411_04844_b200 import _lib, build

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                      "include", "splatct.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(splatct_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_all_header_symbols():
    path = build.build()
    assert os.path.exists(path)
    L = ctypes.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), f"{s} declared in splatct.h but not exported"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes signature table out of sync with header"


def test_abi_version_and_error_plumbing():
    L = _lib.load()
    assert L.splatct_abi_version() == 1
    assert isinstance(L.splatct_last_error(), bytes)
    n = ctypes.c_size_t(0)
    assert L.splatct_fvr_workspace_bytes(1000, 64, 64, 64, 8, 8, 8, ctypes.byref(n)) == 0
    assert n.value > 0


def test_sass_is_sm100a():
    """The fatbin carries sm_100a SASS (cuobjdump), not just PTX."""
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", build.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
