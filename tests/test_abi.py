"""The C-ABI library builds for sm_100a, loads and exports every declared symbol (CPU only)."""

import ctypes
import os
import re
import subprocess

from conftest import ROOT
from paper_2404_12703_b200 import _lib

HEADER = os.path.join(ROOT, "include", "hexdg_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hdg_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_binding_covers_header():
    assert set(declared_functions()) == set(_lib.EXPORTED)


def test_descriptor_layout_matches():
    lib = _lib.load()
    assert lib.hdg_sizeof_domain() == ctypes.sizeof(_lib.HdgDomain)
    assert lib.hdg_sizeof_params() == ctypes.sizeof(_lib.HdgParams)
    assert lib.hdg_abi_version() == _lib.ABI_VERSION == 2


def test_argument_errors_without_gpu():
    lib = _lib.load()
    d = _lib.HdgDomain()
    p = _lib.HdgParams()
    d.N = 9
    assert lib.hdg_check_domain(ctypes.byref(d), ctypes.byref(p)) != 0
    assert b"unsupported" in lib.hdg_last_error()
    d.N = 3
    assert lib.hdg_check_domain(ctypes.byref(d), ctypes.byref(p)) != 0
    assert b"NULL" in lib.hdg_last_error()


def test_sass_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
