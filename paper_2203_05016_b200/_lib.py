"""ctypes loader for libshflbw_b200.so (the C ABI of include/shflbw_cu.h).

There is no fallback: if the library is missing, importing the package
raises, and if no sm_100 device is usable every compute call raises
``shflbw.Error``.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SBW_LIB") or os.path.join(HERE, "lib", "libshflbw_b200.so")  # SBW_LIB: A/B runs

(OK, SHAPE_MISMATCH, NONCONFORMANT_MASK, BAD_PARAMS, BAD_GEOMETRY, CUDA_ERROR, UNSUPPORTED, BAD_MAGIC,
 UNSUPPORTED_VERSION, CORRUPT_PAYLOAD) = range(10)
F32, BF16, F16 = 0, 1, 2
PAD_COLUMN = -1
K_TILE = 64


class PruneConfigC(C.Structure):
    """struct shflbw_prune_config"""
    _fields_ = [("alpha", C.c_double), ("beta_factor", C.c_double), ("v", C.c_uint32),
                ("kmeans_max_iters", C.c_uint32), ("seed", C.c_uint64), ("restarts", C.c_uint32),
                ("reserved", C.c_uint32)]


class CuMatrix(C.Structure):
    """struct shflbw_cu_matrix (include/shflbw_cu.h)."""
    _fields_ = [
        ("rows", C.c_int32), ("cols", C.c_int32), ("v", C.c_int32), ("groups", C.c_int32),
        ("dtype", C.c_int32), ("k_tile", C.c_int32), ("total_cols", C.c_int64),
        ("row_indices", C.c_void_p), ("group_ptr", C.c_void_p), ("group_ncols", C.c_void_p),
        ("col_idx", C.c_void_p), ("values", C.c_void_p), ("device", C.c_int32), ("owns", C.c_int32),
        ("max_group_cols", C.c_int32), ("reserved", C.c_int32),
    ]


# name -> (restype, argtypes); this list is also the ABI the CPU tests check
SIGNATURES = {
    "shflbw_cu_last_error": (C.c_char_p, []),
    "shflbw_cu_version": (C.c_int, []),
    "shflbw_cu_set_option": (C.c_int, [C.c_char_p, C.c_int64]),
    "shflbw_cu_launch_count": (C.c_int64, []),
    "shflbw_cu_last_plan": (C.c_char_p, []),
    "shflbw_cu_validate": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(C.c_int32), C.POINTER(C.c_uint32), C.c_void_p]),
    "shflbw_cu_compress": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                     C.c_int32, C.POINTER(CuMatrix), C.POINTER(C.c_uint32), C.c_void_p]),
    "shflbw_cu_matrix_free": (None, [C.POINTER(CuMatrix)]),
    "shflbw_cu_compress_async": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                           C.c_int32, C.POINTER(CuMatrix), C.c_void_p, C.c_void_p]),
    "shflbw_cu_matrix_finalize": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p, C.POINTER(C.c_uint32), C.c_void_p]),
    "shflbw_cu_matrix_upload": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.c_void_p, C.c_int32, C.POINTER(CuMatrix),
                                          C.c_void_p]),
    "shflbw_cu_matrix_download": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p]),
    "shflbw_cu_matrix_export_raw": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p]),
    "shflbw_cu_decompress": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p, C.c_void_p]),
    "shflbw_cu_spmm": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p, C.c_int32, C.c_int32, C.c_int64,
                                 C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    "shflbw_cu_spmm_groups_peers": (C.c_int, [C.POINTER(CuMatrix), C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                              C.c_int32, C.c_int64, C.POINTER(C.c_void_p), C.c_int32, C.c_int32,
                                              C.c_int64, C.c_void_p]),
    "shflbw_cu_spmm_groups_multicast": (C.c_int, [C.POINTER(CuMatrix), C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                                  C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_int64,
                                                  C.c_void_p]),
    "shflbw_cu_spmm_groups": (C.c_int, [C.POINTER(CuMatrix), C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                        C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_int64, C.c_int32,
                                        C.c_void_p]),
    "shflbw_cu_importance_scores": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "shflbw_cu_kept_score": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                       C.c_void_p]),
    "shflbw_cu_prune_unstructured": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_double, C.c_void_p,
                                               C.c_void_p]),
    "shflbw_cu_prune_vectorwise": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_uint32, C.c_double,
                                             C.c_void_p, C.c_void_p]),
    "shflbw_cu_kmeans_row_grouping": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                                C.c_void_p, C.c_void_p]),
    "shflbw_cu_prune_shflbw": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.POINTER(C.c_double), C.c_void_p]),
    "shflbw_cu_smx1_decode": (C.c_int, [C.c_void_p, C.c_uint64, C.c_int32, C.c_void_p, C.c_void_p]),
    "shflbw_cu_smx1_encode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64), C.c_void_p]),
    "shflbw_cu_conv_prepare": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "shflbw_cu_fold_input_permutation": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "shflbw_cu_unpermute_rows": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]),
    "shflbw_cu_conv_output_size": (C.c_int, [C.c_int32] * 6 + [C.POINTER(C.c_int32)] * 2),
    "shflbw_cu_conv2d": (C.c_int, [C.POINTER(CuMatrix), C.c_void_p] + [C.c_int32] * 8
                         + [C.c_void_p, C.c_int32, C.c_void_p]),
    "shflbw_cu_dense_matmul_f32": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_int32,
                                             C.c_void_p, C.c_void_p]),
    "shflbw_cu_stitch_tile": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_int32,
                                        C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p]),
    "shflbw_cu_tile_mma": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_void_p]),
    "shflbw_cu_convert": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p]),
    "shflbw_cu_convert_2d": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_int32, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -m paper_2203_05016_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
