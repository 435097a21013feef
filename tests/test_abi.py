"""CPU-side checks of the C ABI boundary: libapmm_b200.so loads, exports exactly what
include/apmm_cuda.h declares, and the host-side validation reproduces the reference's
error classes before any device work (no compute calls here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "apmm_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"APMM_API\s+[\w\s\*]+?\b(apmm_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2409_17870_b200 import _lib
    return _lib.load()


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "apmm_cu_matmul_ap" in syms and "apmm_matmul_ap" in syms and len(syms) >= 20


def test_library_exports_every_declared_symbol(lib):
    so = os.path.join(ROOT, "paper_2409_17870_b200", "libapmm_b200.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    extra = [s for s in exported if s.startswith("apmm_") and s not in declared_symbols()]
    assert not extra, extra
    from paper_2409_17870_b200 import _lib
    assert set(_lib.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a_only(lib):
    so = os.path.join(ROOT, "paper_2409_17870_b200", "libapmm_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    assert "UTCIMMA" in sass and "UTMALDG" in sass and "LDTM" in sass  # tcgen05 + TMA + TMEM


def test_status_names_match_reference_error_classes(lib):
    names = [lib.apmm_status_name(i).decode() for i in range(1, 9)]
    assert names == ["EvenValue", "OutOfRange", "NonFinite", "LengthMismatch",
                     "DimensionMismatch", "IndexOutOfBounds", "Overflow", "OverflowBound"]


def test_overflow_bound_without_device(lib):
    out = C.c_int64()
    assert lib.apmm_overflow_bound(8, 8, 33025, C.byref(out)) == 0 and out.value == 33025 * 255 * 255
    assert lib.apmm_overflow_bound(3, 4, 10752, C.byref(out)) == 0 and out.value == 1128960
    assert lib.apmm_overflow_bound(0, 4, 1, C.byref(out)) == 2  # OutOfRange (bipolar.hpp:17-19)
    assert lib.apmm_packed_words(3, 5, 45) == 3 * 5 * 2


def test_context_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2409_17870_b200 as ap
    with pytest.raises(ap.NoDevice):
        ap.Context(0)


def test_python_mirror_validation():
    import paper_2409_17870_b200 as ap
    with pytest.raises(ap.OutOfRange):
        ap.BitWidth(0)
    with pytest.raises(ap.OutOfRange):
        ap.BitWidth(9)
    with pytest.raises(ap.OutOfRange):
        ap.TileConfig(0, 1, 32)
    with pytest.raises(ap.OutOfRange):
        ap.TileConfig(1, 1, 48)
    ap.TileConfig(1, 1, 32)
    with pytest.raises(ap.LengthMismatch):  # test_bitplane.cpp:138-143
        ap.PackedBitPlanes(1, 33, ap.BitWidth(1), np.array([0xFFFFFFFF], np.uint32))
    with pytest.raises(ap.OutOfRange):
        ap.PackedBitPlanes(1, 1, ap.BitWidth(1), np.array([0x2], np.uint32))
    p = ap.PackedBitPlanes(2, 2, ap.BitWidth(2), np.array([1, 1, 3, 0], np.uint32))
    assert p.plane_row(1, 0).tolist() == [3]
    with pytest.raises(ap.IndexOutOfBounds):
        p.plane_row(2, 0)
    with pytest.raises(ap.DimensionMismatch):
        ap.PackedBitPlanes(0, 1, ap.BitWidth(1), np.zeros(0, np.uint32))
    assert ap.overflow_bound(ap.BitWidth(8), ap.BitWidth(8), 33026) > 2**31 - 1


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2409_17870_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "apmm_oracle" not in src and "liboracle" not in src, f


def test_release_library_reads_no_environment():
    """Dev instrumentation (route overrides, ablations that change results, timelines that
    synchronise inside a launch) is compiled only with -DAPMM_DEVTOOLS: the release .so holds
    none of those environment names (build.py, csrc/internal.h APMM_DEV_ENV)."""
    so = os.path.join(ROOT, "paper_2409_17870_b200", "libapmm_b200.so")
    data = open(so, "rb").read()
    for name in (b"APMM_PEAK_PROBE", b"APMM_FUSED_ABLATE", b"APMM_PAIR_TS", b"APMM_SKINNY_TS",
                 b"APMM_DEBUG_WAITS", b"APMM_MID", b"APMM_PSPLIT", b"APMM_FUSED",
                 b"APMM_FORCE_TC", b"APMM_FORCE_1SM", b"APMM_SK_STAGES", b"APMM_DEBUG_PLAN"):
        assert name not in data, name


def test_option_validation_without_device(lib):
    assert lib.apmm_ctx_set_option(None, 1, 0) == 9
    v = C.c_int()
    assert lib.apmm_ctx_get_option(None, 1, C.byref(v)) == 9
    assert lib.apmm_ctx_reserve(None, 1, 1, 1, 1) == 9
