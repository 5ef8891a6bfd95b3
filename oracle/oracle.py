"""ctypes bindings for the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Two backends expose the same methods:

* ``Oracle``    -- our C restatement, ``oracle/liboracle.so`` (shflbw_oracle.c)
* ``Reference`` -- the UNMODIFIED reference library compiled from
  /root/reference/proj/src by ``oracle/Makefile`` into
  ``oracle/_ref/libshflbw_ref.so`` (``ref_shim.cpp`` is its extern "C" face).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product library never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libshflbw_ref.so")

STATUS_NAMES = {0: "ok", 1: "ShapeMismatch", 2: "NonConformantMask", 3: "BadParams",
                4: "BadGeometry", 7: "BadMagic", 8: "UnsupportedVersion", 9: "CorruptPayload", 99: "Error"}

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(np.uint16, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


class OracleError(Exception):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {what}")
        self.code = code


@dataclass
class Packed:
    """The reference ShflBWMatrix, flattened (oracle/shflbw_oracle.h)."""
    M: int
    K: int
    V: int
    row_indices: np.ndarray  # u32 [M]
    group_ncols: np.ndarray  # u32 [G]
    cols: np.ndarray         # u32 [sum n_g]
    values: np.ndarray       # f32 [V * sum n_g]

    @property
    def G(self) -> int:
        return self.M // self.V if self.V else 0

    def group_cols(self, g: int) -> np.ndarray:
        off = int(self.group_ncols[:g].sum())
        return self.cols[off: off + int(self.group_ncols[g])]

    def group_values(self, g: int) -> np.ndarray:
        off = int(self.group_ncols[:g].sum())
        return self.values[off * self.V: (off + int(self.group_ncols[g])) * self.V]


REF_TESTS = os.path.join(HERE, "_ref", "reference_unit_tests_b200")


def build(force: bool = False, with_ref_tests: bool = False) -> None:
    """Compile liboracle.so (and _ref when /root/reference is present; with
    with_ref_tests also the reference's own unit tests linked against
    libshflbw_b200.so)."""
    targets = ["all"] + (["ref_tests"] if with_ref_tests else [])
    if force or with_ref_tests or not os.path.exists(ORACLE_SO) or (
            os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


class _Rng:
    def __init__(self, lib, new, nxt, free, seed):
        self._lib, self._free = lib, free
        self.h = new(C.c_uint64(seed))
        self._next = nxt

    def __call__(self) -> int:
        return int(self._next(self.h))

    def __del__(self):
        try:
            self._free(self.h)
        except Exception:
            pass


class _Backend:
    name = "?"

    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self._last_error())

    def _last_error(self) -> str:
        return ""

    # ---- generators -----------------------------------------------------
    def rng(self, seed: int) -> _Rng:
        return _Rng(self.lib, self._rng_new, self._rng_next, self._rng_free, seed)

    def random_dense(self, rows: int, cols: int, seed: int) -> np.ndarray:
        out = np.empty(rows * cols, np.float32)
        self._random_dense(rows, cols, C.c_uint64(seed), out)
        return out.reshape(rows, cols)

    def fill_uniform(self, rng: _Rng, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.empty(n, np.float32)
        self._fill_uniform(rng.h, C.c_size_t(n), C.c_float(lo), C.c_float(hi), out)
        return out

    def random_shflbw_mask(self, m: int, k: int, v: int, cols_per_group: int, rng: _Rng) -> np.ndarray:
        out = np.empty(max(m * k, 1), np.uint8)
        self._random_shflbw_mask(m, k, v, cols_per_group, rng.h, out)
        return out[: m * k].reshape(m, k)


class Oracle(_Backend):
    """The C restatement (oracle/shflbw_oracle.c)."""
    name = "oracle"

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        lib = self.lib = C.CDLL(path)
        vp = C.c_void_p
        lib.orc_rng_new.restype = vp
        lib.orc_rng_new.argtypes = [C.c_uint64]
        lib.orc_rng_next.restype = C.c_uint64
        lib.orc_rng_next.argtypes = [vp]
        lib.orc_rng_free.argtypes = [vp]
        self._rng_new, self._rng_next, self._rng_free = lib.orc_rng_new, lib.orc_rng_next, lib.orc_rng_free
        lib.orc_random_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _f32p]
        self._random_dense = lib.orc_random_dense
        lib.orc_fill_uniform.argtypes = [vp, C.c_size_t, C.c_float, C.c_float, _f32p]
        self._fill_uniform = lib.orc_fill_uniform
        lib.orc_random_shflbw_mask.argtypes = [C.c_uint32] * 4 + [vp, _u8p]
        self._random_shflbw_mask = lib.orc_random_shflbw_mask
        lib.orc_validate_shflbw.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
        lib.orc_compress.argtypes = [_f32p, _u8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                     _u32p, _u32p, _u32p, _f32p, C.POINTER(C.c_uint32)]
        lib.orc_decompress.argtypes = [C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p]
        lib.orc_spmm.argtypes = [C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p,
                                                    C.c_uint32, C.c_uint32, _f32p]
        lib.orc_spmm_groups.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _u32p, _f32p,
                                        _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _f32p]
        lib.orc_spmm_dense.argtypes = [_f32p, C.c_uint32, C.c_uint32, _f32p, C.c_uint32, _f32p]
        lib.orc_rel_frobenius.restype = C.c_double
        lib.orc_rel_frobenius.argtypes = [_f32p, _f32p, C.c_size_t]
        lib.orc_conv_output_size.argtypes = [C.c_uint32] * 6 + [C.POINTER(C.c_uint32)] * 2
        lib.orc_conv2d.argtypes = ([C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p]
                                   + [C.c_uint32] * 8 + [_f32p])
        lib.orc_conv_direct.argtypes = ([_f32p, C.c_uint32, _f32p] + [C.c_uint32] * 8 + [_f32p])
        lib.orc_stitch_to_blockwise.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _f32p,
                                                C.c_uint32, _u32p, _f32p, _u32p]
        lib.orc_round16.argtypes = [_f32p, C.c_size_t, C.c_int]
        lib.orc_pack_device.restype = C.c_int64
        lib.orc_pack_device.argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, _f32p, C.c_uint32,
                                        C.c_int, _i32p, _i32p, _u16p]

    # ---- hot path ------------------------------------------------------
    def validate(self, mask: np.ndarray, V: int):
        mask = np.ascontiguousarray(mask, np.uint8)
        M, K = mask.shape
        p, fr = C.c_int(0), C.c_uint32(0)
        self._check(self.lib.orc_validate_shflbw(mask.reshape(-1) if mask.size else np.zeros(1, np.uint8),
                                                 M, K, V, C.byref(p), C.byref(fr)))
        return bool(p.value), int(fr.value)

    def compress(self, dense: np.ndarray, mask: np.ndarray, V: int) -> Packed:
        dense = np.ascontiguousarray(dense, np.float32)
        mask = np.ascontiguousarray(mask, np.uint8)
        if dense.shape != mask.shape:
            raise OracleError(1, "compress_shflbw: dense and mask shapes differ")
        M, K = mask.shape
        cap = max(M * K, 1)
        ri = np.zeros(max(M, 1), np.uint32)
        gn = np.zeros(max(M, 1), np.uint32)
        cols = np.zeros(cap, np.uint32)
        vals = np.zeros(cap, np.float32)
        fr = C.c_uint32(0)
        st = self.lib.orc_compress(dense.reshape(-1) if dense.size else np.zeros(1, np.float32),
                                   mask.reshape(-1) if mask.size else np.zeros(1, np.uint8),
                                   M, K, V, ri, gn, cols, vals, C.byref(fr))
        if st == 2:
            raise OracleError(2, f"(row {fr.value})")
        self._check(st)
        G = M // V
        nnzc = int(gn[:G].sum())
        return Packed(M, K, V, ri[:M].copy(), gn[:G].copy(), cols[:nnzc].copy(), vals[: nnzc * V].copy())

    def decompress(self, a: Packed) -> np.ndarray:
        out = np.zeros(max(a.M * a.K, 1), np.float32)
        self.lib.orc_decompress(a.M, a.K, a.V, _nz(a.row_indices), _nz(a.group_ncols), _nz(a.cols),
                                _nz(a.values), out)
        return out[: a.M * a.K].reshape(a.M, a.K)

    def spmm(self, a: Packed, B: np.ndarray) -> np.ndarray:
        B = np.ascontiguousarray(B, np.float32)
        Kb, N = B.shape
        out = np.zeros(max(a.M * N, 1), np.float32)
        self._check(self.lib.orc_spmm(a.M, a.K, a.V, _nz(a.row_indices), _nz(a.group_ncols),
                                      _nz(a.cols), _nz(a.values), _nz(B.reshape(-1)), Kb, N, out))
        return out[: a.M * N].reshape(a.M, N)

    def spmm_groups(self, a: Packed, B: np.ndarray, g_begin: int, g_end: int,
                    C_out: np.ndarray) -> None:
        B = np.ascontiguousarray(B, np.float32)
        self.lib.orc_spmm_groups(a.M, a.V, _nz(a.row_indices), _nz(a.group_ncols), _nz(a.cols),
                                 _nz(a.values), _nz(B.reshape(-1)), B.shape[1], g_begin, g_end,
                                 C_out.reshape(-1))

    def spmm_dense(self, A: np.ndarray, B: np.ndarray) -> np.ndarray:
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        if A.shape[1] != B.shape[0]:
            raise OracleError(1, "oracle: A columns != B rows")
        out = np.zeros(max(A.shape[0] * B.shape[1], 1), np.float32)
        self.lib.orc_spmm_dense(_nz(A.reshape(-1)), A.shape[0], A.shape[1], _nz(B.reshape(-1)),
                                B.shape[1], out)
        return out[: A.shape[0] * B.shape[1]].reshape(A.shape[0], B.shape[1])

    def rel_frobenius(self, x: np.ndarray, y: np.ndarray) -> float:
        x = np.ascontiguousarray(x, np.float32).reshape(-1)
        y = np.ascontiguousarray(y, np.float32).reshape(-1)
        if x.shape != y.shape:
            raise OracleError(1, "relative_frobenius_error: shapes differ")
        return float(self.lib.orc_rel_frobenius(_nz(x), _nz(y), x.size))

    def conv_output_size(self, H, W, R, S, stride, pad):
        P, Q = C.c_uint32(0), C.c_uint32(0)
        self._check(self.lib.orc_conv_output_size(H, W, R, S, stride, pad, C.byref(P), C.byref(Q)))
        return int(P.value), int(Q.value)

    def conv2d(self, w: Packed, inp: np.ndarray, R, S, stride, pad) -> np.ndarray:
        inp = np.ascontiguousarray(inp, np.float32)
        Cc, H, W, Nb = inp.shape
        P, Q = self.conv_output_size(H, W, R, S, stride, pad)
        out = np.zeros(max(w.M * P * Q * Nb, 1), np.float32)
        self._check(self.lib.orc_conv2d(w.M, w.K, w.V, _nz(w.row_indices), _nz(w.group_ncols),
                                        _nz(w.cols), _nz(w.values), _nz(inp.reshape(-1)), Cc, H, W,
                                        Nb, R, S, stride, pad, out))
        return out[: w.M * P * Q * Nb].reshape(w.M, P, Q, Nb)

    def conv_direct(self, w_dense: np.ndarray, inp: np.ndarray, R, S, stride, pad) -> np.ndarray:
        inp = np.ascontiguousarray(inp, np.float32)
        w_dense = np.ascontiguousarray(w_dense, np.float32)
        Cc, H, W, Nb = inp.shape
        P, Q = self.conv_output_size(H, W, R, S, stride, pad)
        out = np.zeros(max(w_dense.shape[0] * P * Q * Nb, 1), np.float32)
        self._check(self.lib.orc_conv_direct(_nz(w_dense.reshape(-1)), w_dense.shape[0],
                                             _nz(inp.reshape(-1)), Cc, H, W, Nb, R, S, stride,
                                             pad, out))
        return out[: w_dense.shape[0] * P * Q * Nb].reshape(w_dense.shape[0], P, Q, Nb)

    def stitch_to_blockwise(self, a: Packed, tile_width: int):
        total = sum((int(n) + tile_width - 1) // tile_width for n in a.group_ncols) if tile_width else 0
        tc = np.zeros(max(total * tile_width, 1), np.uint32)
        tv = np.zeros(max(total * tile_width * a.V, 1), np.float32)
        tg = np.zeros(max(total, 1), np.uint32)
        n = self.lib.orc_stitch_to_blockwise(a.V, a.G, _nz(a.group_ncols), _nz(a.cols),
                                             _nz(a.values), tile_width, tc, tv, tg)
        if n < 0:
            raise OracleError(-n, "tile_width must be positive")
        return tg[:n], tc[: n * tile_width].reshape(n, tile_width), tv[: n * tile_width * a.V].reshape(
            n, tile_width * a.V)

    def round16(self, x: np.ndarray, dtype: str = "bf16") -> np.ndarray:
        y = np.ascontiguousarray(x, np.float32).copy()
        self.lib.orc_round16(_nz(y.reshape(-1)), y.size, 2 if dtype == "f16" else 1)
        return y

    def pack_device(self, a: Packed, k_tile: int, dtype: str = "bf16"):
        total_cap = sum((int(n) + k_tile - 1) // k_tile * k_tile for n in a.group_ncols)
        gp = np.zeros(a.G + 1, np.int32)
        ci = np.zeros(max(total_cap, 1), np.int32)
        vv = np.zeros(max(total_cap * a.V, 1), np.uint16)
        total = self.lib.orc_pack_device(a.M, a.V, _nz(a.group_ncols), _nz(a.cols), _nz(a.values),
                                         k_tile, 2 if dtype == "f16" else 1, gp, ci, vv)
        return gp, ci[:total], vv[: total * a.V]


class Reference(_Backend):
    """The compiled reference (oracle/_ref/libshflbw_ref.so)."""
    name = "reference"

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        lib = self.lib = C.CDLL(path)
        vp = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_rng_new.restype = vp
        lib.ref_rng_new.argtypes = [C.c_uint64]
        lib.ref_rng_next.restype = C.c_uint64
        lib.ref_rng_next.argtypes = [vp]
        lib.ref_rng_free.argtypes = [vp]
        self._rng_new, self._rng_next, self._rng_free = lib.ref_rng_new, lib.ref_rng_next, lib.ref_rng_free
        lib.ref_random_dense.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, _f32p]
        self._random_dense = lib.ref_random_dense
        lib.ref_fill_uniform.argtypes = [vp, C.c_size_t, C.c_float, C.c_float, _f32p]
        self._fill_uniform = lib.ref_fill_uniform
        lib.ref_random_shflbw_mask.argtypes = [C.c_uint32] * 4 + [vp, _u8p]
        self._random_shflbw_mask = lib.ref_random_shflbw_mask
        lib.ref_validate_shflbw.argtypes = [_u8p, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.POINTER(C.c_int), C.POINTER(C.c_uint32)]
        lib.ref_compress.argtypes = [_f32p, C.c_uint32, C.c_uint32, _u8p, C.c_uint32, C.c_uint32,
                                     C.c_uint32, _u32p, _u32p, _u32p, _f32p]
        lib.ref_spmm.argtypes = [C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p,
                                                    C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                                    C.c_uint, _f32p]
        lib.ref_matrix_new.restype = vp
        lib.ref_matrix_new.argtypes = [C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p]
        lib.ref_matrix_free.argtypes = [vp]
        lib.ref_dense_new.restype = vp
        lib.ref_dense_new.argtypes = [C.c_uint32, C.c_uint32, _f32p]
        lib.ref_dense_free.argtypes = [vp]
        lib.ref_spmm_prebuilt.argtypes = [vp, vp, C.c_uint, vp]
        lib.ref_spmm_dense.argtypes = [_f32p, C.c_uint32, C.c_uint32, _f32p, C.c_uint32, _f32p]
        lib.ref_decompress.argtypes = [C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p]
        lib.ref_conv_output_size.argtypes = [C.c_uint32] * 6 + [C.POINTER(C.c_uint32)] * 2
        lib.ref_conv2d.argtypes = ([C.c_uint32] * 3 + [_u32p, _u32p, _u32p, _f32p, _f32p]
                                   + [C.c_uint32] * 8 + [C.c_uint, _f32p])
        lib.ref_stitch_to_blockwise.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p,
                                                _f32p, C.c_uint32, _u32p, _f32p, _u32p,
                                                C.POINTER(C.c_int)]

    def _last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def validate(self, mask: np.ndarray, V: int):
        mask = np.ascontiguousarray(mask, np.uint8)
        M, K = mask.shape
        p, fr = C.c_int(0), C.c_uint32(0)
        self._check(self.lib.ref_validate_shflbw(_nz(mask.reshape(-1)), M, K, V, C.byref(p), C.byref(fr)))
        return bool(p.value), int(fr.value)

    def compress(self, dense: np.ndarray, mask: np.ndarray, V: int) -> Packed:
        dense = np.ascontiguousarray(dense, np.float32)
        mask = np.ascontiguousarray(mask, np.uint8)
        M, K = mask.shape
        cap = max(M * K, 1)
        ri = np.zeros(max(M, 1), np.uint32)
        gn = np.zeros(max(M, 1), np.uint32)
        cols = np.zeros(cap, np.uint32)
        vals = np.zeros(cap, np.float32)
        self._check(self.lib.ref_compress(_nz(dense.reshape(-1)), dense.shape[0], dense.shape[1],
                                          _nz(mask.reshape(-1)), M, K, V, ri, gn, cols, vals))
        G = M // V
        nnzc = int(gn[:G].sum())
        return Packed(M, K, V, ri[:M].copy(), gn[:G].copy(), cols[:nnzc].copy(), vals[: nnzc * V].copy())

    def decompress(self, a: Packed) -> np.ndarray:
        out = np.zeros(max(a.M * a.K, 1), np.float32)
        self._check(self.lib.ref_decompress(a.M, a.K, a.V, _nz(a.row_indices), _nz(a.group_ncols),
                                            _nz(a.cols), _nz(a.values), out))
        return out[: a.M * a.K].reshape(a.M, a.K)

    def spmm(self, a: Packed, B: np.ndarray, t_n: int = 0, t_k: int = 0, threads: int = 1) -> np.ndarray:
        B = np.ascontiguousarray(B, np.float32)
        Kb, N = B.shape
        out = np.zeros(max(a.M * N, 1), np.float32)
        self._check(self.lib.ref_spmm(a.M, a.K, a.V, _nz(a.row_indices), _nz(a.group_ncols),
                                      _nz(a.cols), _nz(a.values), _nz(B.reshape(-1)), Kb, N, t_n,
                                      t_k, threads, out))
        return out[: a.M * N].reshape(a.M, N)

    def spmm_dense(self, A: np.ndarray, B: np.ndarray) -> np.ndarray:
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        out = np.zeros(max(A.shape[0] * B.shape[1], 1), np.float32)
        self._check(self.lib.ref_spmm_dense(_nz(A.reshape(-1)), A.shape[0], A.shape[1],
                                            _nz(B.reshape(-1)), B.shape[1], out))
        return out[: A.shape[0] * B.shape[1]].reshape(A.shape[0], B.shape[1])

    def conv_output_size(self, H, W, R, S, stride, pad):
        P, Q = C.c_uint32(0), C.c_uint32(0)
        self._check(self.lib.ref_conv_output_size(H, W, R, S, stride, pad, C.byref(P), C.byref(Q)))
        return int(P.value), int(Q.value)

    def conv2d(self, w: Packed, inp: np.ndarray, R, S, stride, pad, threads: int = 1) -> np.ndarray:
        inp = np.ascontiguousarray(inp, np.float32)
        Cc, H, W, Nb = inp.shape
        P, Q = self.conv_output_size(H, W, R, S, stride, pad)
        out = np.zeros(max(w.M * P * Q * Nb, 1), np.float32)
        self._check(self.lib.ref_conv2d(w.M, w.K, w.V, _nz(w.row_indices), _nz(w.group_ncols),
                                        _nz(w.cols), _nz(w.values), _nz(inp.reshape(-1)), Cc, H, W,
                                        Nb, R, S, stride, pad, threads, out))
        return out[: w.M * P * Q * Nb].reshape(w.M, P, Q, Nb)

    def stitch_to_blockwise(self, a: Packed, tile_width: int):
        total = sum((int(n) + tile_width - 1) // tile_width for n in a.group_ncols) if tile_width else 0
        tc = np.zeros(max(total * tile_width, 1), np.uint32)
        tv = np.zeros(max(total * tile_width * a.V, 1), np.float32)
        tg = np.zeros(max(total, 1), np.uint32)
        n = C.c_int(0)
        self._check(self.lib.ref_stitch_to_blockwise(a.K, a.V, a.G, _nz(a.group_ncols), _nz(a.cols),
                                                     _nz(a.values), tile_width, tc, tv, tg, C.byref(n)))
        n = n.value
        return tg[:n], tc[: n * tile_width].reshape(n, tile_width), tv[: n * tile_width * a.V].reshape(
            n, tile_width * a.V)

    # prebuilt-object timing path used by bench.py --impl reference
    def prebuilt(self, a: Packed, B: np.ndarray):
        B = np.ascontiguousarray(B, np.float32)
        ha = self.lib.ref_matrix_new(a.M, a.K, a.V, _nz(a.row_indices), _nz(a.group_ncols),
                                     _nz(a.cols), _nz(a.values))
        hb = self.lib.ref_dense_new(B.shape[0], B.shape[1], _nz(B.reshape(-1)))
        return ha, hb

    def spmm_prebuilt(self, ha, hb, threads: int, out: np.ndarray | None = None) -> None:
        self._check(self.lib.ref_spmm_prebuilt(ha, hb, threads,
                                               out.ctypes.data if out is not None else None))

    def free_prebuilt(self, ha, hb) -> None:
        self.lib.ref_matrix_free(ha)
        self.lib.ref_dense_free(hb)

    # pruning (src/pruning.cpp)
    def kept_score(self, scores: np.ndarray, mask: np.ndarray) -> float:
        s = np.ascontiguousarray(scores, np.float32)
        m = np.ascontiguousarray(mask, np.uint8)
        out = C.c_double(0.0)
        f = self.lib.ref_kept_score
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_double)]
        self._check(f(_nz(s).ctypes.data, _nz(m).ctypes.data, s.shape[0], s.shape[1], C.byref(out)))
        return out.value

    def prune_unstructured(self, scores: np.ndarray, ratio: float) -> np.ndarray:
        s = np.ascontiguousarray(scores, np.float32)
        out = np.zeros(max(s.size, 1), np.uint8)
        f = self.lib.ref_prune_unstructured
        f.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_void_p]
        self._check(f(_nz(s).ctypes.data, s.shape[0], s.shape[1], ratio, out.ctypes.data))
        return out[: s.size].reshape(s.shape)

    def prune_vectorwise(self, scores: np.ndarray, v: int, alpha: float) -> np.ndarray:
        s = np.ascontiguousarray(scores, np.float32)
        out = np.zeros(max(s.size, 1), np.uint8)
        f = self.lib.ref_prune_vectorwise
        f.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_void_p]
        self._check(f(_nz(s).ctypes.data, s.shape[0], s.shape[1], v, alpha, out.ctypes.data))
        return out[: s.size].reshape(s.shape)

    def kmeans_row_grouping(self, mask: np.ndarray, scores: np.ndarray, cfg: dict) -> np.ndarray:
        s = np.ascontiguousarray(scores, np.float32)
        m = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros(max(s.shape[0], 1), np.uint32)
        f = self.lib.ref_kmeans_row_grouping
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint32,
                      C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p]
        self._check(f(_nz(m).ctypes.data, _nz(s).ctypes.data, s.shape[0], s.shape[1], cfg["alpha"],
                      cfg["beta_factor"], cfg["v"], cfg["kmeans_max_iters"], cfg["seed"], cfg["restarts"],
                      out.ctypes.data))
        return out[: s.shape[0]]

    def prune_shflbw(self, scores: np.ndarray, cfg: dict):
        """-> (mask u8 [M, K], permutation u32 [M], kept_score)"""
        s = np.ascontiguousarray(scores, np.float32)
        mask = np.zeros(max(s.size, 1), np.uint8)
        perm = np.zeros(max(s.shape[0], 1), np.uint32)
        kept = C.c_double(0.0)
        f = self.lib.ref_prune_shflbw
        f.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint32, C.c_uint32,
                      C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.POINTER(C.c_double)]
        self._check(f(_nz(s).ctypes.data, s.shape[0], s.shape[1], cfg["alpha"], cfg["beta_factor"], cfg["v"],
                      cfg["kmeans_max_iters"], cfg["seed"], cfg["restarts"], mask.ctypes.data, perm.ctypes.data,
                      C.byref(kept)))
        return mask[: s.size].reshape(s.shape), perm[: s.shape[0]], kept.value

    # SMX1 container (src/container.cpp)
    def smx1_encode(self, a: Packed) -> bytes:
        size = C.c_size_t(0)
        f = self.lib.ref_smx1_encode_shflbw
        args = [a.M, a.K, a.V, _nz(a.row_indices).ctypes.data, _nz(a.group_ncols).ctypes.data,
                _nz(a.cols).ctypes.data, _nz(a.values).ctypes.data]
        f.argtypes = [C.c_uint32] * 3 + [C.c_void_p] * 5 + [C.c_size_t, C.POINTER(C.c_size_t)]
        self._check(f(*args, None, 0, C.byref(size)))
        out = np.zeros(size.value, np.uint8)
        self._check(f(*args, out.ctypes.data, size.value, C.byref(size)))
        return out.tobytes()

    def smx1_encode_dense(self, d: np.ndarray) -> bytes:
        d = np.ascontiguousarray(d, np.float32)
        size = C.c_size_t(0)
        f = self.lib.ref_smx1_encode_dense
        f.argtypes = [C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        self._check(f(d.shape[0], d.shape[1], _nz(d).ctypes.data, None, 0, C.byref(size)))
        out = np.zeros(size.value, np.uint8)
        self._check(f(d.shape[0], d.shape[1], _nz(d).ctypes.data, out.ctypes.data, size.value, C.byref(size)))
        return out.tobytes()

    def smx1_decode(self, b: bytes) -> tuple[int, "Packed | None"]:
        f = self.lib.ref_smx1_decode_shflbw
        f.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p] + [C.c_void_p] * 4
        buf = np.frombuffer(b, np.uint8).copy() if len(b) else np.zeros(1, np.uint8)
        hdr = np.zeros(5, np.uint32)
        st = f(buf.ctypes.data, len(b), hdr.ctypes.data, None, None, None, None)
        if st:
            return st, None
        M, K, V, G, T = (int(x) for x in hdr)
        ri, gn = np.zeros(max(M, 1), np.uint32), np.zeros(max(G, 1), np.uint32)
        cols, vals = np.zeros(max(T, 1), np.uint32), np.zeros(max(T * V, 1), np.float32)
        st = f(buf.ctypes.data, len(b), hdr.ctypes.data, ri.ctypes.data, gn.ctypes.data, cols.ctypes.data,
               vals.ctypes.data)
        return st, Packed(M, K, V, ri[:M], gn[:G], cols[:T], vals[:T * V])


# --------------------------------------------------------------------------
# SMX1 container, kind 3 (Shfl-BW) -- restatement of the reference's byte
# format (include/shflbw/container.hpp:14-22, src/container.cpp): header
# "SMX1", u32 version = 1, kind, M, K, V, G (src/container.cpp:71-80); kind 3
# payload = M u32 row_indices, then per group u32 n_g, n_g u32 columns,
# V*n_g f32 values (src/container.cpp:82-88, :141-145); all little-endian.

SMX1_MAGIC = b"SMX1"


def smx1_encode(p: Packed) -> bytes:
    """encode_container(ShflBWMatrix) (src/container.cpp:141-145)."""
    G = p.G
    parts = [SMX1_MAGIC, np.array([1, 3, p.M, p.K, p.V, G], "<u4").tobytes(),
             np.asarray(p.row_indices, "<u4").tobytes()]
    off = 0
    for g in range(G):
        n = int(p.group_ncols[g])
        parts.append(np.array([n], "<u4").tobytes())
        parts.append(np.asarray(p.cols[off:off + n], "<u4").tobytes())
        parts.append(np.asarray(p.values[off * p.V:(off + n) * p.V], "<f4").tobytes())
        off += n
    return b"".join(parts)


def _smx1_walk_other(b: bytes, pos: int, kind: int, M: int, K: int, V: int, G: int) -> bool:
    """True if the payload of another kind is corrupt (decode_container,
    src/container.cpp:158-238: kind 0 dense, 1 mask, 2 vector-wise
    read_vector_wise_payload :90-115, 4 block-wise)."""
    n = len(b)

    def u32():
        nonlocal pos
        if n - pos < 4:
            raise ValueError
        v = int.from_bytes(b[pos:pos + 4], "little")
        pos += 4
        return v

    def skip_f32s(count):
        nonlocal pos
        if count > (n - pos) // 4:
            raise ValueError
        pos += 4 * count
    try:
        if kind == 0:
            start = pos
            skip_f32s(M * K)
            if pos != n:
                return True
            vals = np.frombuffer(b, "<u4", M * K, start)
            return bool(np.any((vals & 0x7F800000) == 0x7F800000))
        if kind == 1:
            nbytes = (M * K + 7) // 8
            if pos + nbytes > n:
                return True
            return pos + nbytes != n
        if kind == 2:
            if V == 0 or V * G != M:
                return True
            for _ in range(G):
                ng = u32()
                if ng > K:
                    return True
                prev = 0
                for j in range(ng):
                    c = u32()
                    if c >= K or (j > 0 and c <= prev):
                        return True
                    prev = c
                skip_f32s(ng * V)
            return pos != n
        # kind 4
        if V == 0 or M % V or K % V:
            return True
        nb = u32()
        if pos + nb * 8 > n:
            return True
        prev = None
        for _ in range(nb):
            br, bc = u32(), u32()
            if br >= M // V or bc >= K // V:
                return True
            if prev is not None and (br, bc) <= prev:
                return True
            prev = (br, bc)
        skip_f32s((nb * V * V) % (1 << 64))
        return pos != n
    except ValueError:
        return True


def smx1_decode(b: bytes) -> tuple[int, "Packed | None"]:
    """decode_container + as_shflbw (src/container.cpp:147-215, :90-124,
    :126-134): (status, matrix).  Status codes as include/shflbw_cu.h:
    3 BadParams (another kind), 7 BadMagic, 8 UnsupportedVersion,
    9 CorruptPayload.  Other kinds are walked with the reference's checks
    (_smx1_walk_other): corrupt -> CorruptPayload, valid -> as_shflbw's
    BadParams."""
    if len(b) < 4 or b[:4] != SMX1_MAGIC:
        return 7, None
    pos = 4

    def u32s(n):
        nonlocal pos
        if n > (len(b) - pos) // 4:
            raise ValueError
        v = np.frombuffer(b, "<u4", n, pos).astype(np.uint32)
        pos += 4 * n
        return v
    try:
        version = int(u32s(1)[0])
        if version != 1:
            return 8, None
        kind, M, K, V, G = (int(x) for x in u32s(5))
        if kind in (0, 1, 2, 4):  # decoded and validated first, then as_shflbw's BadParams
            return (9 if _smx1_walk_other(b, pos, kind, M, K, V, G) else 3), None
        if kind != 3:
            return 9, None
        ri = u32s(M)
        seen = np.zeros(M, bool)
        if np.any(ri >= M):
            return 9, None
        seen[ri] = True
        if not seen.all():
            return 9, None
        if V == 0 or V * G != M:
            return 9, None
        gn, cols, vals = [], [], []
        for _ in range(G):
            n = int(u32s(1)[0])
            if n > K:
                return 9, None
            c = u32s(n)
            if n and (np.any(c >= K) or np.any(np.diff(c.astype(np.int64)) <= 0)):
                return 9, None
            gn.append(n)
            cols.append(c)
            vals.append(u32s(n * V).view(np.float32))
        if pos != len(b):
            return 9, None
    except ValueError:
        return 9, None
    return 0, Packed(M, K, V, ri.copy(), np.array(gn, np.uint32),
                     np.concatenate(cols).astype(np.uint32) if cols else np.zeros(0, np.uint32),
                     np.concatenate(vals).astype(np.float32) if vals else np.zeros(0, np.float32))


def _nz(a: np.ndarray) -> np.ndarray:
    """ctypes ndpointer rejects size-0 arrays' null data; give a 1-element dummy."""
    a = np.ascontiguousarray(a)
    if a.size == 0:
        return np.zeros(1, a.dtype)
    return a.reshape(-1)
