"""CPU checks of the boundary: libfmm.so builds for sm_100a, loads, and exports every entry point
include/fmm.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fmm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1108_5815_b200 import build as fb

    return fb.build()


def test_library_exports_every_declared_symbol(libpath):
    syms = header_symbols()
    assert len(syms) >= 16
    L = ctypes.CDLL(libpath)
    for s in syms:
        assert hasattr(L, s), s
    from paper_1108_5815_b200 import fmm

    assert sorted(fmm.SYMBOLS) == syms


def test_binary_is_sm100a_cuda_core_code(libpath):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath],
                          capture_output=True, text=True).stdout
    funcs = {}
    for chunk in sass.split("Function : ")[1:]:
        funcs[chunk.split()[0]] = chunk
    m2l = [v for k, v in funcs.items() if "k_m2l_gemm" in k]
    assert m2l and "FFMA2" in m2l[0]  # packed FP32 FMA on the M2L hot loop
    p2p = [v for k, v in funcs.items() if "k_p2p_tma" in k]
    assert p2p and "MUFU.RSQ" in p2p[0] and "FFMA2" in p2p[0]
    assert "UBLKCP" in p2p[0]  # the producer warp's TMA bulk copies of the source ranges


def test_strerror_without_gpu(libpath):
    L = ctypes.CDLL(libpath)
    L.fmm_strerror.restype = ctypes.c_char_p
    assert L.fmm_strerror(0) == b"ok"
    assert b"non-finite" in L.fmm_strerror(-3)
    h = ctypes.c_void_p()
    L.fmm_create.argtypes = [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_double, ctypes.c_int]
    assert L.fmm_create(ctypes.byref(h), 0, 0.5, 8) == -1  # invalid p, rejected before any CUDA call
    assert L.fmm_create(ctypes.byref(h), 4, 1.5, 8) == -1
    assert L.fmm_create(ctypes.byref(h), 4, 0.5, 0) == -1
    assert L.fmm_destroy(None) == 0


def test_product_package_has_no_oracle_import():
    pkg = os.path.join(ROOT, "paper_1108_5815_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt, f
