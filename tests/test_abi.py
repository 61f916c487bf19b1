"""CPU checks of the boundary: libvsag.so loads and exports every symbol include/vsag.h declares;
the binding refuses to run without the library (no CPU fallback); the oracle and the CUDA
path share no source."""
import ctypes
import os
import re
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2503_17911_b200")


def _declared():
    src = open(os.path.join(ROOT, "include", "vsag.h")).read()
    return sorted(set(re.findall(r"VSAG_API\s+[\w\s\*]+?\b(vsag_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for need in ("vsag_encode_sq", "vsag_index_load", "vsag_search_batch", "vsag_index_free", "vsag_last_error"):
        assert need in names


def test_library_exports_every_declared_symbol():
    from paper_2503_17911_b200 import build as b
    lib_path = b.build()
    lib = ctypes.CDLL(lib_path)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vsag_\w+)", out))
    assert exported == set(_declared())
    lib.vsag_code_bytes.restype = ctypes.c_int64
    assert lib.vsag_code_bytes(960, 4) == 480 and lib.vsag_code_bytes(128, 8) == 128
    lib.vsag_last_error.restype = ctypes.c_char_p
    assert lib.vsag_last_error() == b""


def test_binding_fails_loudly_without_library(tmp_path):
    pkg = tmp_path / "paper_2503_17911_b200"
    pkg.mkdir()
    shutil.copy(os.path.join(PKG, "__init__.py"), pkg / "__init__.py")
    r = subprocess.run([sys.executable, "-c", "import paper_2503_17911_b200"], cwd=tmp_path, capture_output=True,
                       text=True)
    assert r.returncode != 0 and "libvsag.so not built" in r.stderr


def test_oracle_and_cuda_path_are_independent():
    # the product package never references the oracle, and the oracle never includes libvsag sources
    for root, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(root, f)).read()
                assert "oracle" not in txt.lower(), f
    osrc = open(os.path.join(ROOT, "oracle", "oracle.cpp")).read()
    assert "vsag.h" not in osrc and "csrc" not in osrc
