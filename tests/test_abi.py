"""CPU: the C-ABI library loads and exports every entry point that
include/cgmimo_b200.h declares (no compute call without a GPU)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_1404_0424_b200 as pkg
from paper_1404_0424_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cgmimo_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cgm_\w+)\s*\(", text)))


def test_library_is_built_and_loads():
    assert os.path.exists(_lib.LIB_PATH), "run __graft_entry__.build()"
    lib = _lib.load()
    assert lib.cgm_version().decode().startswith("cgmimo_b200")


def test_every_header_symbol_is_exported_and_bound():
    declared = header_functions()
    assert len(declared) >= 14
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in cgmimo_b200.h but not exported"
    assert sorted(_lib.SIGNATURES) == declared, "ctypes signatures out of sync with the header"


def test_exports_are_c_linkage_and_sm100a_only():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in header_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name
    sass = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "sm_100a" in sass and "sm_90" not in sass


def test_cxx_dropin_symbols_exported():
    out = subprocess.run(["nm", "-DC", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for sym in ("cgmimo::detect::detect_cg(", "cgmimo::precode::precode_cg(",
                "cgmimo::detect::compute_llrs(", "cgmimo::phy::make_constellation(",
                "cgmimo::detect::detect_cholesky(", "cgmimo::detect::detect_cgls(",
                "cgmimo::detect::detect_neumann(", "cgmimo::precode::precode_explicit(",
                "cgmimo::precode::precode_cgls(", "cgmimo::precode::precode_neumann("):
        assert sym in out, sym


def test_context_creation_fails_cleanly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _lib.load()
    h = C.c_void_p()
    rc = lib.cgm_ctx_create(0, C.byref(h))
    assert rc == _lib.CGM_ECUDA and not h.value
    with pytest.raises(pkg.CudaError):
        pkg.Context(0)
    # NULL context is rejected, never dereferenced
    assert lib.cgm_detect_cg(None, 8, 4, 1, 1, None, None, 1.0, 1.0, 1.0, 4, 2, 0, None, None,
                             None, None, None, 0) == _lib.CGM_EINVAL
    assert lib.cgm_last_error(None).decode() == "null context"
