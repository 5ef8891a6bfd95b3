"""B200-native Shfl-BW (arXiv 2203.05016) sparse linear / conv hot path.

The product is ``lib/libshflbw_b200.so``: hand-written sm_100a kernels
(tcgen05 + TMEM + TMA gather4) behind the C ABI of ``include/shflbw_cu.h``
and the reference-compatible C++ API of ``include/shflbw/``.  This Python
package is a thin host mirror of the reference interface over that ABI
(``shflbw``) plus the multi-GPU row-group sharding (``sharded``).
"""
from .shflbw import (BadGeometry, BadMagic, BadParams, ConvGeometry, CorruptPayload, Error, NonConformantMask,
                     ShapeMismatch, UnsupportedVersion, smx1_dump, smx1_dumps, smx1_load, smx1_loads,
                     PruneConfig, PruneResult, importance_scores, kept_score, kmeans_row_grouping,
                     prune_shflbw, prune_unstructured, prune_vectorwise,
                     ShflBWMatrix, TileConfig, compress_shflbw, compress_shflbw_async, conv2d, conv_output_size, conv_prepare,
                     decompress, finalize, fold_input_permutation, last_plan, launch_count, set_option, spmm_execute, spmm_groups, spmm_groups_multicast, spmm_groups_peers,
                     unpermute_rows, upload, validate_pattern)

__all__ = ["BadGeometry", "BadMagic", "BadParams", "ConvGeometry", "CorruptPayload", "Error", "NonConformantMask",
           "ShapeMismatch", "UnsupportedVersion", "smx1_dump", "smx1_dumps", "smx1_load", "smx1_loads",
           "PruneConfig", "PruneResult", "importance_scores", "kept_score", "kmeans_row_grouping",
           "prune_shflbw", "prune_unstructured", "prune_vectorwise",
           "ShflBWMatrix", "TileConfig", "compress_shflbw", "compress_shflbw_async", "conv2d", "conv_output_size", "conv_prepare",
           "decompress", "finalize",
           "fold_input_permutation", "last_plan", "launch_count", "set_option", "spmm_execute", "spmm_groups", "spmm_groups_multicast", "spmm_groups_peers",
           "unpermute_rows", "upload", "validate_pattern"]
