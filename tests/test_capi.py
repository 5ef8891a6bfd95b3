"""CPU-side checks of the C-ABI library (no compute without a GPU).

* libshflbw_b200.so loads and exports every symbol include/shflbw_cu.h
  declares, with the argument lists the ctypes mirror binds;
* host-only entry points (conv_output_size, options) follow the reference's
  semantics (src/spmm.cpp:177-191);
* compute entry points fail loudly (status SHFLBW_CUDA_ERROR / BadParams)
  when no GPU is present -- there is no CPU fallback.
"""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2203_05016_b200 import _lib as L
    from paper_2203_05016_b200 import build
    build.build(verbose=False)
    return L.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "shflbw_cu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(shflbw_cu_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    from paper_2203_05016_b200 import _lib as L
    syms = header_symbols()
    assert len(syms) >= 16
    for s in syms:
        assert hasattr(lib, s), s
        assert s in L.SIGNATURES, f"ctypes mirror does not bind {s}"


def test_cpp_api_exported(lib):
    # the reference-compatible C++ API (include/shflbw/*.hpp) lives in the same .so
    out = os.popen(f"nm -DC {lib._name} | grep ' T shflbw::'").read()
    for fn in ["shflbw::compress_shflbw(", "shflbw::spmm_execute(", "shflbw::conv2d(",
               "shflbw::conv_output_size(", "shflbw::decompress(", "shflbw::validate_pattern(",
               "shflbw::TileConfig::validate() const"]:
        assert fn in out, fn


def test_conv_output_size_host(lib):
    P, Q = C.c_int32(0), C.c_int32(0)
    assert lib.shflbw_cu_conv_output_size(6, 6, 3, 3, 1, 0, C.byref(P), C.byref(Q)) == 0
    assert (P.value, Q.value) == (4, 4)
    assert lib.shflbw_cu_conv_output_size(6, 6, 3, 3, 1, 1, C.byref(P), C.byref(Q)) == 0
    assert (P.value, Q.value) == (6, 6)
    assert lib.shflbw_cu_conv_output_size(6, 6, 3, 3, 2, 0, C.byref(P), C.byref(Q)) == 4
    assert lib.shflbw_cu_conv_output_size(2, 2, 5, 5, 1, 0, C.byref(P), C.byref(Q)) == 4
    assert lib.shflbw_cu_conv_output_size(6, 6, 0, 3, 1, 0, C.byref(P), C.byref(Q)) == 4


def test_options(lib):
    assert lib.shflbw_cu_set_option(b"split", 2) == 0
    assert lib.shflbw_cu_set_option(b"split", 0) == 0
    assert lib.shflbw_cu_set_option(b"nonsense", 1) == 3
    assert b"unknown option" in lib.shflbw_cu_last_error()


def test_compute_fails_loudly_without_gpu(lib):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2203_05016_b200 import _lib as L
    m = L.CuMatrix()
    fr = C.c_uint32(0)
    st = lib.shflbw_cu_compress(None, 0, None, 4, 4, 2, 1, C.byref(m), C.byref(fr), None)
    assert st == L.CUDA_ERROR
    assert lib.shflbw_cu_last_error()
    # argument checks come first and keep the reference's error classes
    assert lib.shflbw_cu_compress(None, 0, None, 4, 4, 3, 1, C.byref(m), C.byref(fr), None) == L.BAD_PARAMS
    assert lib.shflbw_cu_spmm(None, None, 0, 0, 0, None, 0, 0, None) == L.BAD_PARAMS


def test_smx1_decode_rejects_like_the_reference_without_gpu(lib):
    """Every corrupted SMX1 container of tests/golden/smx1_cases.json gets the
    reference's status from the library's host-side validation (before any
    device work); a valid file then needs the GPU."""
    import json
    from paper_2203_05016_b200 import _lib as L
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "smx1_cases.json")))["cases"]
    for c in cases:
        data = bytes.fromhex(c["hex"])
        buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data or b"\0")
        m = L.CuMatrix()
        st = lib.shflbw_cu_smx1_decode(buf, len(data), L.BF16, C.byref(m), None)
        if c["status"] == 0:
            assert st in (L.OK, L.CUDA_ERROR), c["name"]
        else:
            assert st == c["status"], (c["name"], st, c["status"])


def test_conv_fdiv_reciprocal_exact():
    """The conv producers divide column ids by R*S and S with a float
    reciprocal (tc_kernels.cuh fdiv): trunc((c + 0.5f) * (1.0f / d)) == c / d
    for every c < 2^22 (the host-checked range) and every filter size used."""
    import numpy as np
    c = np.arange(0, 1 << 22, dtype=np.int64)
    cf = c.astype(np.float32) + np.float32(0.5)
    for d in list(range(1, 50)) + [64, 81, 121, 256]:
        q = np.trunc(cf * (np.float32(1.0) / np.float32(d))).astype(np.int64)
        assert np.array_equal(q, c // d), d
