"""CPU checks of the boundary: libgb.so builds, loads, exports every symbol
include/gb.h declares, and fails loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

import __graft_entry__
import paper_1303_7032_b200 as gb
from tests.helpers import ROOT


@pytest.fixture(scope="module")
def built():
    __graft_entry__.build()
    return gb.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "gb.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(gb_[a-z_]+)\s*\(", txt)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(gb.EXPORTS)


def test_library_exports_every_header_symbol(built):
    out = subprocess.check_output(["nm", "-D", "--defined-only", gb.LIB_PATH], text=True)
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for s in header_symbols():
        assert s in syms, s
        assert getattr(built, s) is not None


def test_sm100a_code_only(built):
    """The fat binary carries sm_100a SASS only (no PTX JIT path for other archs)."""
    out = subprocess.check_output(["cuobjdump", "--list-elf", gb.LIB_PATH], text=True)
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_version_and_no_gpu_failure(built):
    assert b"sm_100a" in built.gb_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: the no-device path is not reachable")
    h = ctypes.c_void_p()
    rc = built.gb_create(8, 128, 0, ctypes.byref(h))
    assert rc in (gb.GB_ECUDA, gb.GB_EINVAL, gb.GB_EUNSUPPORTED)
    assert h.value is None
    assert built.gb_last_error()
    with pytest.raises(gb.GBError):
        gb.Net(8, 128)


def test_argument_validation_without_gpu(built):
    """Pure host-side validation paths return the documented codes."""
    h = ctypes.c_void_p()
    assert built.gb_create(1, 16, 0, ctypes.byref(h)) == gb.GB_EINVAL
    assert built.gb_create(4, 0, 0, ctypes.byref(h)) == gb.GB_EINVAL
    assert built.gb_create(65, 16, 0, ctypes.byref(h)) == gb.GB_EUNSUPPORTED
    assert built.gb_create(16, 1024, 0, ctypes.byref(h)) == gb.GB_EUNSUPPORTED
    assert built.gb_decode(None, None, 0, 0, 0, 1, None, None, None, None) == gb.GB_EINVAL
    assert built.gb_destroy(None) == gb.GB_OK


def test_product_path_never_touches_oracle():
    """The product package shares nothing with oracle/: no import, include,
    dlopen or path reference in either direction."""
    pat = re.compile(r"(^\s*(import|from)\s+oracle\b)|(#include\s*[<\"].*oracle)|gb_oracle|"
                     r"libgb_oracle|['\"]oracle['\"/]", re.M)
    pkg = os.path.join(ROOT, "paper_1303_7032_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cuh", ".cpp")):
                assert not pat.search(open(os.path.join(dirpath, f)).read()), f
    assert not pat.search(open(os.path.join(ROOT, "include", "gb.h")).read())
    src = open(os.path.join(ROOT, "oracle", "gb_oracle.c")).read()
    assert not re.search(r"#include\s*[<\"][^>\"]*(gb\.h|gb_internal)", src)
    assert not re.search(r"^\s*(import|from)\s+paper_1303_7032_b200", 
                         open(os.path.join(ROOT, "oracle", "__init__.py")).read(), re.M)
