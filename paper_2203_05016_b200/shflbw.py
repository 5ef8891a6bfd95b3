"""Python mirror of the reference's hot-path interface, on device tensors.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/shflbw/{errors,formats,spmm}.hpp):

    compress_shflbw(dense, mask, v)          formats.hpp:98-99
    validate_pattern(mask, "shfl_bw", v)     formats.hpp:91-92
    decompress(a)                            formats.hpp:102-104
    spmm_execute(a, b, cfg=None, threads=1)  spmm.hpp:28-29
    conv2d(w, x, geo, cfg=None, threads=1)   spmm.hpp:87-89
    conv_output_size(x_shape, geo)           spmm.hpp:93-94

Every call goes through the C ABI (include/shflbw_cu.h) into the sm_100a
kernels; tensors are torch CUDA tensors and work is queued on torch's
current stream.  ``threads`` is accepted and ignored, as on any GPU build
(results never depend on it, include/shflbw/spmm.hpp:24-27).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L


class Error(RuntimeError):
    """shflbw::Error (include/shflbw/errors.hpp:9-11)."""


class ShapeMismatch(Error):
    pass


class NonConformantMask(Error):
    pass


class BadParams(Error):
    pass


class BadGeometry(Error):
    pass


class BadMagic(Error):
    """Container errors (include/shflbw/errors.hpp:29-40)."""


class UnsupportedVersion(Error):
    pass


class CorruptPayload(Error):
    pass


_ERRORS = {L.SHAPE_MISMATCH: ShapeMismatch, L.NONCONFORMANT_MASK: NonConformantMask,
           L.BAD_PARAMS: BadParams, L.BAD_GEOMETRY: BadGeometry, L.BAD_MAGIC: BadMagic,
           L.UNSUPPORTED_VERSION: UnsupportedVersion, L.CORRUPT_PAYLOAD: CorruptPayload}


def _lib():
    return L.load()


def _check(status: int) -> None:
    if status != L.OK:
        msg = _lib().shflbw_cu_last_error().decode(errors="replace")
        raise _ERRORS.get(status, Error)(msg)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


_DT = {torch.float32: L.F32, torch.bfloat16: L.BF16, torch.float16: L.F16}
_TORCH = {v: k for k, v in _DT.items()}


def _dt(t: torch.dtype) -> int:
    if t not in _DT:
        raise BadParams(f"unsupported dtype {t}")
    return _DT[t]


@dataclass
class TileConfig:
    """include/shflbw/spmm.hpp:13-22.  Validated like the reference
    (src/spmm.cpp:11-19); the GPU kernels pick their own tiles, results do
    not depend on it."""
    t_m: int = 64
    t_n: int = 16
    t_k: int = 8
    regfile_size: int = 4096
    pipe_stage: int = 2
    meta_prefetch_stage: int = 4

    def validate(self) -> None:
        if self.t_m == 0 or self.t_n == 0 or self.t_k == 0:
            raise BadParams("tile sizes must be positive")
        if self.t_m * self.t_n > self.regfile_size:
            raise BadParams("T_M * T_N exceeds the register-file budget")
        if self.pipe_stage < 2:
            raise BadParams("pipe_stage must be >= 2")
        if self.meta_prefetch_stage < 1:
            raise BadParams("meta_prefetch_stage must be >= 1")


@dataclass
class ConvGeometry:
    """include/shflbw/spmm.hpp:76-81"""
    r: int = 1
    s: int = 1
    stride: int = 1
    pad: int = 0


class ShflBWMatrix:
    """Device-resident Shfl-BW matrix (struct shflbw_cu_matrix)."""

    def __init__(self, cm: L.CuMatrix):
        self._m = cm
        self._ref = C.byref(cm)

    def __del__(self):
        try:
            if self._m.owns:
                _lib().shflbw_cu_matrix_free(C.byref(self._m))
        except Exception:
            pass

    @property
    def rows(self) -> int:
        return self._m.rows

    @property
    def cols(self) -> int:
        return self._m.cols

    @property
    def vector_size(self) -> int:
        return self._m.v

    v = vector_size

    def group_count(self) -> int:
        return self._m.groups

    @property
    def dtype(self) -> torch.dtype:
        return _TORCH[self._m.dtype]

    @property
    def total_cols(self) -> int:
        return int(self._m.total_cols)

    @property
    def ptr(self):
        return self._ref


    def to_host(self):
        """-> (row_indices u32[M], group_ncols u32[G], cols u32[sum n_g],
        values f32[V*sum n_g]) in the reference's layout."""
        M, G, V = self.rows, self.group_count(), self.v
        ri = np.zeros(max(M, 1), np.uint32)
        gn = np.zeros(max(G, 1), np.uint32)
        cap = max(self.total_cols, 1)
        cols = np.zeros(cap, np.uint32)
        vals = np.zeros(cap * V, np.float32)
        _check(_lib().shflbw_cu_matrix_download(self.ptr, ri.ctypes.data, gn.ctypes.data, cols.ctypes.data,
                                                vals.ctypes.data, _stream()))
        nnzc = int(gn[:G].sum())
        return ri[:M], gn[:G], cols[:nnzc], vals[: nnzc * V]

    def raw(self):
        """-> (group_ptr i32[G+1], col_idx i32[total], values u16[total*V] (u32 bit patterns for F32
        matrices)): the device layout."""
        G, V, T = self.group_count(), self.v, self.total_cols
        gp = np.zeros(G + 1, np.int32)
        ci = np.zeros(max(T, 1), np.int32)
        vv = np.zeros(max(T * V, 1), np.uint32 if self.dtype == torch.float32 else np.uint16)
        _check(_lib().shflbw_cu_matrix_export_raw(self.ptr, gp.ctypes.data, ci.ctypes.data, vv.ctypes.data,
                                                  _stream()))
        return gp, ci[:T], vv[: T * V]

    @property
    def row_indices_ptr(self) -> int:
        return self._m.row_indices


def _dev_u8(mask: torch.Tensor) -> torch.Tensor:
    if not (isinstance(mask, torch.Tensor) and mask.is_cuda):
        raise BadParams("mask must be a CUDA tensor")
    if mask.dtype == torch.bool:
        mask = mask.to(torch.uint8)
    if mask.dtype != torch.uint8 or mask.dim() != 2:
        raise BadParams("mask must be a 2-D uint8/bool CUDA tensor")
    return mask.contiguous()


def validate_pattern(mask: torch.Tensor, pattern: str = "shfl_bw", v: int = 1):
    """-> (pass, fail_row).  Only the shfl_bw pattern is on the hot path."""
    if pattern not in ("shfl_bw", "shflbw"):
        raise BadParams(f"pattern {pattern!r} is not provided by the GPU library")
    mask = _dev_u8(mask)
    M, K = mask.shape
    p, fr = C.c_int32(0), C.c_uint32(0)
    _check(_lib().shflbw_cu_validate(mask.data_ptr(), M, K, v, C.byref(p), C.byref(fr), _stream()))
    return bool(p.value), int(fr.value)


def compress_shflbw(dense: torch.Tensor, mask: torch.Tensor, v: int,
                    dtype: torch.dtype = torch.bfloat16) -> ShflBWMatrix:
    """Build the device Shfl-BW matrix; values rounded to `dtype` (RNE)."""
    if not (isinstance(dense, torch.Tensor) and dense.is_cuda and dense.dim() == 2):
        raise BadParams("dense must be a 2-D CUDA tensor")
    mask = _dev_u8(mask)
    if tuple(dense.shape) != tuple(mask.shape):
        raise ShapeMismatch("compress_shflbw: dense and mask shapes differ")
    dense = dense.contiguous()
    M, K = mask.shape
    cm = L.CuMatrix()
    fr = C.c_uint32(0)
    st = _lib().shflbw_cu_compress(dense.data_ptr(), _dt(dense.dtype), mask.data_ptr(), M, K, v, _dt(dtype),
                                   C.byref(cm), C.byref(fr), _stream())
    _check(st)
    return ShflBWMatrix(cm)


def compress_shflbw_async(dense: torch.Tensor, mask: torch.Tensor, v: int,
                          dtype: torch.dtype = torch.bfloat16, out: "ShflBWMatrix | None" = None,
                          status: torch.Tensor | None = None):
    """The converter without a host synchronisation (shflbw_cu_compress_async,
    graph-capturable): -> (matrix, status) with status a device int32[4]
    {code, fail_row, total columns, widest group}.  The matrix is usable by
    SpMM / conv work enqueued after it; finalize(matrix, status) raises the
    reference's exception for a bad mask and sets the exact sizes."""
    if not (isinstance(dense, torch.Tensor) and dense.is_cuda and dense.dim() == 2):
        raise BadParams("dense must be a 2-D CUDA tensor")
    mask = _dev_u8(mask)
    if tuple(dense.shape) != tuple(mask.shape):
        raise ShapeMismatch("compress_shflbw: dense and mask shapes differ")
    dense = dense.contiguous()
    M, K = mask.shape
    if status is None:
        status = torch.zeros(4, dtype=torch.int32, device=dense.device)
    m = out if out is not None else ShflBWMatrix(L.CuMatrix())
    _check(_lib().shflbw_cu_compress_async(dense.data_ptr(), _dt(dense.dtype), mask.data_ptr(), M, K, v, _dt(dtype),
                                           m.ptr, status.data_ptr(), _stream()))
    m._keep = (dense, mask)  # inputs must outlive the enqueued conversion
    return m, status


def finalize(a: ShflBWMatrix, status: torch.Tensor) -> None:
    """Read an asynchronous conversion's status (one synchronisation): raises
    NonConformantMask "(row N)" / BadParams / Error, else fixes the sizes."""
    fr = C.c_uint32(0)
    _check(_lib().shflbw_cu_matrix_finalize(a.ptr, status.data_ptr(), C.byref(fr), _stream()))


def upload(M: int, K: int, V: int, row_indices, group_ncols, cols, values,
           dtype: torch.dtype = torch.bfloat16) -> ShflBWMatrix:
    """A host (reference-layout) ShflBWMatrix -> device."""
    ri = np.ascontiguousarray(row_indices, np.uint32)
    gn = np.ascontiguousarray(group_ncols, np.uint32)
    cc = np.ascontiguousarray(cols, np.uint32)
    vv = np.ascontiguousarray(values, np.float32)
    cm = L.CuMatrix()
    _check(_lib().shflbw_cu_matrix_upload(M, K, V, ri.ctypes.data, gn.ctypes.data, cc.ctypes.data,
                                          vv.ctypes.data, _dt(dtype), C.byref(cm), _stream()))
    torch.cuda.current_stream().synchronize()
    return ShflBWMatrix(cm)


def decompress(a: ShflBWMatrix) -> torch.Tensor:
    out = torch.empty((a.rows, a.cols), dtype=torch.float32, device="cuda")
    _check(_lib().shflbw_cu_decompress(a.ptr, out.data_ptr(), _stream()))
    return out


def _check_b(a: ShflBWMatrix, b: torch.Tensor) -> torch.Tensor:
    if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dim() == 2):
        raise BadParams("B must be a 2-D CUDA tensor")
    if b.shape[0] != a.cols:
        raise ShapeMismatch("spmm: A columns != B rows")
    if b.dtype != a.dtype:
        b = b.to(a.dtype)
    if b.stride(1) != 1:
        b = b.contiguous()
    return b


def spmm_execute(a: ShflBWMatrix, b: torch.Tensor, cfg: TileConfig | None = None, threads: int = 1,
                 out_dtype: torch.dtype = torch.float32, out: torch.Tensor | None = None,
                 permuted_output: bool = False) -> torch.Tensor:
    """C = decompress(a) @ b with the permuted write-back (src/spmm.cpp:76-146).

    permuted_output=True skips the write-back permutation: row i of the
    result is logical row a.row_indices[i] (group order), the input a layer
    folded with fold_input_permutation(next, a) consumes directly."""
    if cfg is not None:  # the default TileConfig is valid by construction
        cfg.validate()
    b = _check_b(a, b)
    N = b.shape[1]
    if out is None:
        out = torch.zeros((a.rows, N), dtype=out_dtype, device=b.device)
    if permuted_output:
        st = _lib().shflbw_cu_spmm_groups(a.ptr, 0, a.group_count(), b.data_ptr(), b.shape[0], N, b.stride(0),
                                          out.data_ptr(), _DT[out.dtype], out.stride(0), 1,
                                          torch.cuda.current_stream().cuda_stream)
    else:
        st = _lib().shflbw_cu_spmm(a.ptr, b.data_ptr(), b.shape[0], N, b.stride(0), out.data_ptr(),
                                   _DT[out.dtype], out.stride(0), torch.cuda.current_stream().cuda_stream)
    if st:
        _check(st)
    return out


# ---------------------------------------------------------------- pruning (§8 f3)

@dataclass
class PruneConfig:
    """include/shflbw/pruning.hpp:27-37"""
    alpha: float = 0.5
    beta_factor: float = 2.0
    v: int = 1
    kmeans_max_iters: int = 50
    seed: int = 0
    restarts: int = 4

    def beta(self) -> float:
        return min(1.0, self.beta_factor * self.alpha)

    def _c(self) -> "L.PruneConfigC":
        return L.PruneConfigC(self.alpha, self.beta_factor, self.v, self.kmeans_max_iters, self.seed,
                              self.restarts, 0)


@dataclass
class PruneResult:
    """mask [M, K] uint8, permutation [M] int32 (grouped position -> original
    row), kept_score (include/shflbw/pruning.hpp:39-45)."""
    mask: torch.Tensor
    permutation: torch.Tensor
    kept_score: float


def _scores(scores: torch.Tensor) -> torch.Tensor:
    if not (isinstance(scores, torch.Tensor) and scores.is_cuda and scores.dim() == 2):
        raise BadParams("scores must be a 2-D CUDA tensor")
    return scores.to(torch.float32).contiguous()


def importance_scores(weights: torch.Tensor) -> torch.Tensor:
    """|weights| (src/pruning.cpp:61-66)."""
    w = weights.to(torch.float32).contiguous()
    out = torch.empty_like(w)
    _check(_lib().shflbw_cu_importance_scores(w.data_ptr(), w.numel(), out.data_ptr(), _stream()))
    return out


def kept_score(scores: torch.Tensor, mask: torch.Tensor) -> float:
    """sum of scores under the mask, in the reference's order (src/pruning.cpp:68-75)."""
    s, m = _scores(scores), _dev_u8(mask)
    if tuple(s.shape) != tuple(m.shape):
        raise ShapeMismatch("kept_score: shapes differ")
    out = C.c_double(0.0)
    _check(_lib().shflbw_cu_kept_score(s.data_ptr(), m.data_ptr(), s.shape[0], s.shape[1], C.byref(out), _stream()))
    return out.value


def prune_unstructured(scores: torch.Tensor, keep_ratio: float) -> torch.Tensor:
    s = _scores(scores)
    out = torch.empty(s.shape, dtype=torch.uint8, device=s.device)
    _check(_lib().shflbw_cu_prune_unstructured(s.data_ptr(), s.shape[0], s.shape[1], keep_ratio, out.data_ptr(),
                                               _stream()))
    return out


def prune_vectorwise(scores: torch.Tensor, v: int, alpha: float) -> torch.Tensor:
    s = _scores(scores)
    out = torch.empty(s.shape, dtype=torch.uint8, device=s.device)
    _check(_lib().shflbw_cu_prune_vectorwise(s.data_ptr(), s.shape[0], s.shape[1], v, alpha, out.data_ptr(),
                                             _stream()))
    return out


def kmeans_row_grouping(mask: torch.Tensor, scores: torch.Tensor, cfg: PruneConfig) -> torch.Tensor:
    s, m = _scores(scores), _dev_u8(mask)
    if tuple(s.shape) != tuple(m.shape):
        raise ShapeMismatch("kmeans_row_grouping: mask and scores differ")
    out = torch.empty(s.shape[0], dtype=torch.int32, device=s.device)
    c = cfg._c()
    _check(_lib().shflbw_cu_kmeans_row_grouping(m.data_ptr(), s.data_ptr(), s.shape[0], s.shape[1], C.byref(c),
                                                out.data_ptr(), _stream()))
    return out


def prune_shflbw(scores: torch.Tensor, cfg: PruneConfig) -> PruneResult:
    """The Shfl-BW pruner (src/pruning.cpp:339-362) on the GPU."""
    s = _scores(scores)
    mask = torch.empty(s.shape, dtype=torch.uint8, device=s.device)
    perm = torch.empty(s.shape[0], dtype=torch.int32, device=s.device)
    kept = C.c_double(0.0)
    c = cfg._c()
    _check(_lib().shflbw_cu_prune_shflbw(s.data_ptr(), s.shape[0], s.shape[1], C.byref(c), mask.data_ptr(),
                                         perm.data_ptr(), C.byref(kept), _stream()))
    return PruneResult(mask, perm, kept.value)


def smx1_loads(data: bytes, dtype: torch.dtype = torch.bfloat16) -> ShflBWMatrix:
    """An SMX1 kind-3 container (the reference's file format,
    include/shflbw/container.hpp:14-22) straight into the device layout;
    the reference's validation rules and error classes (BadMagic,
    UnsupportedVersion, CorruptPayload; BadParams for another kind)."""
    buf = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(bytes(data) or b"\0")
    cm = L.CuMatrix()
    _check(_lib().shflbw_cu_smx1_decode(buf, len(data), _dt(dtype), C.byref(cm), _stream()))
    return ShflBWMatrix(cm)


def smx1_load(path, dtype: torch.dtype = torch.bfloat16) -> ShflBWMatrix:
    """read_container(path) + as_shflbw, into the device layout."""
    with open(path, "rb") as f:
        return smx1_loads(f.read(), dtype)


def smx1_dumps(a: ShflBWMatrix) -> bytes:
    """encode_container(ShflBWMatrix) of a device matrix (values widened to
    f32, so an F32 matrix round-trips byte-identically)."""
    n = C.c_uint64(0)
    _check(_lib().shflbw_cu_smx1_encode(a.ptr, None, 0, C.byref(n), _stream()))
    buf = (C.c_uint8 * max(n.value, 1))()
    _check(_lib().shflbw_cu_smx1_encode(a.ptr, buf, n.value, C.byref(n), _stream()))
    return bytes(buf[: n.value])


def smx1_dump(a: ShflBWMatrix, path) -> None:
    """write_container(ShflBWMatrix, path)."""
    with open(path, "wb") as f:
        f.write(smx1_dumps(a))


def conv_prepare(w: ShflBWMatrix, geo: "ConvGeometry | int") -> ShflBWMatrix:
    """A copy of conv weight `w` in conv order for filter width S = geo.s
    (shflbw_cu_conv_prepare): per group, columns ordered by filter column s
    with each s-run padded to a multiple of 4.  conv2d then fetches 128-byte
    activation rows (64/N adjacent output positions) for stride-1 convs with
    batch N in {16, 32}; results stay within the 1e-5 tolerance (only the
    fp32 summation order differs).  One-time cost, like a filter reorder."""
    S = geo if isinstance(geo, int) else geo.s
    cm = L.CuMatrix()
    _check(_lib().shflbw_cu_conv_prepare(w.ptr, S, C.byref(cm), _stream()))
    return ShflBWMatrix(cm)


def fold_input_permutation(a: ShflBWMatrix, producer) -> ShflBWMatrix:
    """Remap a's column indices so it consumes the group-ordered output of
    `producer` (a ShflBWMatrix run with permuted_output=True, or a device
    int32 tensor of its row_indices).  In place; results stay bit-identical
    to the unpermuted chain."""
    if isinstance(producer, ShflBWMatrix):
        if producer.rows != a.cols:
            raise ShapeMismatch(f"producer rows {producer.rows} != consumer cols {a.cols}")
        rows_ptr = producer._m.row_indices
    else:
        if not (isinstance(producer, torch.Tensor) and producer.is_cuda and producer.dtype == torch.int32
                and producer.dim() == 1 and producer.is_contiguous()):
            raise BadParams("producer must be a ShflBWMatrix or a contiguous CUDA int32 vector")
        if producer.numel() != a.cols:
            raise ShapeMismatch(f"producer rows {producer.numel()} != consumer cols {a.cols}")
        rows_ptr = producer.data_ptr()
    _check(_lib().shflbw_cu_fold_input_permutation(a.ptr, rows_ptr, _stream()))
    return a


def spmm_groups(a: ShflBWMatrix, g_begin: int, g_end: int, b: torch.Tensor, out: torch.Tensor,
                compact: bool) -> torch.Tensor:
    """One shard's groups (src/spmm.cpp:93-144); compact=True writes
    group-ordered rows out[(g - g_begin)*V + r]."""
    b = _check_b(a, b)
    _check(_lib().shflbw_cu_spmm_groups(a.ptr, g_begin, g_end, b.data_ptr(), b.shape[0], b.shape[1],
                                        b.stride(0), out.data_ptr(), _dt(out.dtype), out.stride(0),
                                        int(compact), _stream()))
    return out


def spmm_groups_peers(a: ShflBWMatrix, g_begin: int, g_end: int, b: torch.Tensor, outs,
                      dtype: torch.dtype | None = None, ldc: int | None = None) -> None:
    """One shard's groups with the all-gather fused into the epilogue: every
    finished row is stored at its row_indices position into each full-size
    buffer of `outs` (this GPU's C first, then the peers' C mapped over
    P2P / CUDA IPC).  `outs`: bf16 / f16 tensors of equal dtype and stride,
    or raw device pointers (then `dtype` and `ldc` are required)."""
    b = _check_b(a, b)
    outs = list(outs)
    if not outs:
        raise BadParams("spmm_groups_peers: no destination")
    if all(isinstance(o, torch.Tensor) for o in outs):
        if any(o.dtype != outs[0].dtype or o.stride(0) != outs[0].stride(0) for o in outs):
            raise BadParams("spmm_groups_peers: destinations differ in dtype or stride")
        dtype, ldc = outs[0].dtype, outs[0].stride(0)
        outs = [o.data_ptr() for o in outs]
    elif dtype is None or ldc is None:
        raise BadParams("spmm_groups_peers: raw pointers need dtype and ldc")
    ptrs = (C.c_void_p * len(outs))(*[int(o) for o in outs])
    _check(_lib().shflbw_cu_spmm_groups_peers(a.ptr, g_begin, g_end, b.data_ptr(), b.shape[0], b.shape[1],
                                              b.stride(0), ptrs, len(outs), _dt(dtype), ldc, _stream()))


def spmm_groups_multicast(a: ShflBWMatrix, g_begin: int, g_end: int, b: torch.Tensor, mc_ptr: int,
                          dtype: torch.dtype, ldc: int) -> None:
    """One shard's groups with the all-gather through NVLS multicast: every
    finished row is stored once at its row_indices position through
    `mc_ptr`, a multicast address bound to all ranks' full outputs
    (shflbw_cu_spmm_groups_multicast)."""
    b = _check_b(a, b)
    _check(_lib().shflbw_cu_spmm_groups_multicast(a.ptr, g_begin, g_end, b.data_ptr(), b.shape[0], b.shape[1],
                                                  b.stride(0), int(mc_ptr), _dt(dtype), ldc, _stream()))


def unpermute_rows(row_indices_ptr: int, c_perm: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    _check(_lib().shflbw_cu_unpermute_rows(row_indices_ptr, c_perm.shape[0], c_perm.shape[1],
                                           c_perm.data_ptr(), c_perm.stride(0), out.data_ptr(), out.stride(0),
                                           _dt(out.dtype), _stream()))
    return out


def conv_output_size(shape_chwn, geo: ConvGeometry):
    """(P, Q) for an input of shape (C, H, W, N) (src/spmm.cpp:177-191)."""
    _, H, W, _ = shape_chwn
    P, Q = C.c_int32(0), C.c_int32(0)
    _check(_lib().shflbw_cu_conv_output_size(H, W, geo.r, geo.s, geo.stride, geo.pad, C.byref(P), C.byref(Q)))
    return int(P.value), int(Q.value)


def conv2d(w: ShflBWMatrix, x: torch.Tensor, geo: ConvGeometry, cfg: TileConfig | None = None,
           threads: int = 1, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """Implicit-GEMM sparse conv, input [C][H][W][N] -> [K_f][P][Q][N]."""
    (cfg or TileConfig()).validate()
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dim() == 4):
        raise BadParams("input must be a 4-D CUDA tensor [C][H][W][N]")
    P, Q = conv_output_size(x.shape, geo)
    if x.dtype != w.dtype:
        x = x.to(w.dtype)
    x = x.contiguous()
    Cc, H, W, Nb = x.shape
    out = torch.zeros((w.rows, P, Q, Nb), dtype=out_dtype, device=x.device)
    _check(_lib().shflbw_cu_conv2d(w.ptr, x.data_ptr(), Cc, H, W, Nb, geo.r, geo.s, geo.stride, geo.pad,
                                   out.data_ptr(), _dt(out_dtype), _stream()))
    return out


def set_option(key: str, value: int) -> None:
    _check(_lib().shflbw_cu_set_option(key.encode(), value))


def launch_count() -> int:
    return int(_lib().shflbw_cu_launch_count())


def last_plan() -> str:
    """The kernel variant the last SpMM / conv call on this thread ran
    (shflbw_cu_last_plan): "k_spmm_tc ...", "k_spmm_persist ..." or
    "k_spmm_simt ..."."""
    return _lib().shflbw_cu_last_plan().decode()
