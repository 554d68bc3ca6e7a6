"""The C-ABI library loads (no GPU needed) and exports every entry point that
include/pkv200.h declares; the ctypes binding covers all of them."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2506_07311_b200 import _lib

HEADER = os.path.join(ROOT, "include", "pkv200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"\b(pkv_[a-z0-9_]+)\s*\(", text)
    return sorted(set(names))


def test_header_declares_the_hot_path():
    names = declared_functions()
    for must in ("pkv_pool_reserve", "pkv_pool_grow", "pkv_pool_free", "pkv_pool_fork",
                 "pkv_kv_append", "pkv_page_zero", "pkv_page_copy", "pkv_paged_attention",
                 "pkv_paged_prefill", "pkv_mirror_apply"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes binding"


def test_exports_are_c_linkage():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\s(pkv_[a-z0-9_]+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_library_is_built_for_sm100a():
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_codes_map_to_reference_errors():
    from paper_2506_07311_b200 import errors

    assert _lib._STATUS[1] is errors.CapacityExhausted
    assert _lib._STATUS[3] is errors.UnknownSequence
    assert _lib._STATUS[7] is errors.NoAllowedKeys
    lib = _lib.load()
    assert lib.pkv_abi_version() == 1
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _lib.check(lib.pkv_pool_create(0, 16, ctypes.byref(h)))
    assert b"capacity_pages" in lib.pkv_last_error()


def test_pure_c_client_compiles_and_links(tmp_path):
    """tests/abi_decode.cpp — a client of the C ABI only (no Python, no
    torch) — compiles against include/pkv200.h and links against
    libpkv200.so on a CPU host (it runs in the GPU suite)."""
    import os
    import shutil
    import subprocess

    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib_dir = os.path.join(root, "paper_2506_07311_b200")
    exe = str(tmp_path / "abi_decode")
    r = subprocess.run([gxx, "-O1", "-std=c++17", "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                        os.path.join(root, "tests", "abi_decode.cpp"), "-L", lib_dir, "-lpkv200",
                        "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}", "-o", exe],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
