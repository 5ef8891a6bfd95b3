/*
 * shflbw_cu.h -- C ABI of the B200-native Shfl-BW hot path.
 *
 * Plain pointers and sizes only; every entry point is stream-ordered on the
 * cudaStream_t passed as `stream` (NULL = legacy default stream).  Device
 * pointers are marked [dev], host pointers [host].  All calls return a
 * status code; shflbw_cu_last_error() gives the thread-local message of the
 * last failure.  There is no CPU fallback: without a usable sm_100 device
 * every compute entry point returns SHFLBW_CUDA_ERROR.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj, see INTEGRATION.md for the binding a maintainer
 * adds on the reference side).
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (include/shflbw/errors.hpp:9-40).
 */
#ifndef SHFLBW_CU_H
#define SHFLBW_CU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* shflbw_stream_t; /* == cudaStream_t */

enum shflbw_status {
    SHFLBW_OK = 0,
    SHFLBW_SHAPE_MISMATCH = 1,     /* shflbw::ShapeMismatch     */
    SHFLBW_NONCONFORMANT_MASK = 2, /* shflbw::NonConformantMask */
    SHFLBW_BAD_PARAMS = 3,         /* shflbw::BadParams         */
    SHFLBW_BAD_GEOMETRY = 4,       /* shflbw::BadGeometry       */
    SHFLBW_CUDA_ERROR = 5,         /* shflbw::Error (runtime)   */
    SHFLBW_UNSUPPORTED = 6,        /* shflbw::Error (no kernel for this case) */
    SHFLBW_BAD_MAGIC = 7,          /* shflbw::BadMagic          (SMX1 container) */
    SHFLBW_UNSUPPORTED_VERSION = 8,/* shflbw::UnsupportedVersion (SMX1 container) */
    SHFLBW_CORRUPT_PAYLOAD = 9     /* shflbw::CorruptPayload    (SMX1 container) */
};

enum shflbw_dtype { SHFLBW_F32 = 0, SHFLBW_BF16 = 1, SHFLBW_F16 = 2 };

/* kPadColumn (include/shflbw/formats.hpp:109, 0xffffffff) as int32. */
#define SHFLBW_PAD_COLUMN (-1)
/* Every group's column list is padded to a multiple of this (the SpMM
 * kernel's K block); padding follows stitch_to_blockwise
 * (src/formats.cpp:221-250): index SHFLBW_PAD_COLUMN, value 0. */
#define SHFLBW_K_TILE 64

/*
 * Device-resident Shfl-BW matrix: the reference's ShflBWMatrix
 * (include/shflbw/formats.hpp:14-42) with each group's column-major V x n_g
 * value block stored contiguously (values[(group_ptr[g] + j) * v + r] is row r
 * of group g at column col_idx[group_ptr[g] + j]) and 16-bit values.
 */
typedef struct shflbw_cu_matrix {
    int32_t rows;        /* M (K_f for conv weights)                      */
    int32_t cols;        /* K (C*R*S for conv weights)                    */
    int32_t v;           /* V, rows per group                             */
    int32_t groups;      /* G = M / V                                     */
    int32_t dtype;       /* SHFLBW_BF16 / SHFLBW_F16: tensor cores;
                            SHFLBW_F32: exact CUDA-core path (bit-identical
                            to the reference's fp32 arithmetic)             */
    int32_t k_tile;      /* SHFLBW_K_TILE                                 */
    int64_t total_cols;  /* group_ptr[groups]                             */
    int32_t* row_indices; /* [dev] M: compressed row r -> original row    */
    int32_t* group_ptr;   /* [dev] G+1: padded column offsets              */
    int32_t* group_ncols; /* [dev] G: n_g (unpadded)                       */
    int32_t* col_idx;     /* [dev] total_cols, SHFLBW_PAD_COLUMN padding   */
    void* values;         /* [dev] total_cols * v 16-bit values            */
    int32_t device;       /* CUDA device ordinal                           */
    int32_t owns;         /* 1: free with shflbw_cu_matrix_free            */
    int32_t max_group_cols; /* max_g (group_ptr[g+1]-group_ptr[g]); 0 = unknown
                               (kernels then size pipelines from `cols`)    */
    int32_t reserved;   /* flags: SHFLBW_FOLDED                          */
} shflbw_cu_matrix;

/* shflbw_cu_matrix.reserved bit: col_idx were remapped by
 * shflbw_cu_fold_input_permutation (SpMM input in the producer's group order) */
#define SHFLBW_FOLDED 1
/* shflbw_cu_matrix.reserved bit: columns in conv order (shflbw_cu_conv_prepare);
 * bits 8..15 hold the filter width S it was prepared for */
#define SHFLBW_CONV_ORDER 2
#define SHFLBW_CONV_ORDER_S(reserved) (((reserved) >> 8) & 0xff)
/* shflbw_cu_matrix.reserved bit: built by shflbw_cu_compress_async and not yet
 * finalized -- total_cols / max_group_cols hold the allocation bounds
 * (G * roundup(K, 64) / roundup(K, 64)); every kernel reads the exact group
 * sizes from the device, so the matrix is usable as is */
#define SHFLBW_SIZE_BOUND 4
/* shflbw_cu_matrix.reserved bit: the buffers were allocated from the bound
 * (shflbw_cu_compress_async); a later compress_async of the same shape into
 * this matrix reuses them */
#define SHFLBW_BOUND_ALLOC 8
/* shflbw_cu_matrix.reserved bit: some K block is one contiguous run of 64
 * columns (block-wise patterns; set by shflbw_cu_compress / _upload): the
 * SpMM loads such blocks as TMA 2D tiles instead of row gathers */
#define SHFLBW_CONTIG_BLOCKS 16

/* ---- library ---------------------------------------------------------- */
const char* shflbw_cu_last_error(void);
int shflbw_cu_version(void);
/* Tuning / testing knobs.  Keys: "force_simt" (1: use the CUDA-core kernel
 * for every V), "split" (cluster split of V for the tcgen05 kernel, 0 =
 * auto), "stages" (pipeline depth, 0 = auto), "pdl" (1 = default:
 * programmatic dependent launch -- the SpMM prologue, which reads only the
 * sparse matrix, overlaps the previous kernel on the stream; the activation
 * B and the output C are touched only after the previous grid completes, so
 * a matrix must not be written by work still in flight when an SpMM using it
 * is enqueued -- shflbw_cu_compress / _upload return with it complete),
 * "split_mode" (cluster split kind: 0 = auto, 1 = K split with a DSMEM
 * reduction of fp32 partials, 2 = 2 x 2: V split over a CTA pair and K split
 * over two pairs, 3 = V split with multicast activation tiles; with mode 0 an
 * explicit "split" means V split), "persistent" (N = 1 or 2: the persistent
 * kernel, N CTAs per SM looping over (group, column tile) units; -1: one CTA
 * per unit; 0 = auto: persistent with 2 CTAs per SM once the units exceed
 * one such wave), "gather_warps" (4 or 8 warps issuing the TMA gathers per
 * CTA; 0 = auto: 8 for unsplit units of >= 5 K blocks), "cp_async_slabs"
 * (0..2 activation slabs filled by cp.async instead of TMA gather4),
 * "no_bulk_out" (1: per-element output stores), "strict" (1: a BF16/F16
 * matrix outside the tcgen05 envelope returns UNSUPPORTED with the reason
 * instead of running the CUDA-core kernel), "raster" (persistent unit order:
 * 0 = auto, 1 = group-major, 2 = column-tile-major), "tile_n" (output columns
 * per unit: 0 = auto, 128, or 64 = half-width units for grids that would
 * leave SMs idle), "gather_issue" (0 = auto, 1 = one elected lane per
 * warp issues its gathers, 2 = every issuing lane), "tile_loads" (0 = auto:
 * block-wise K blocks of matrices flagged SHFLBW_CONTIG_BLOCKS as 2D TMA
 * tiles, -1 = gathers only, 1 = check every K block),
 * "prefetch" (SpMM: activation rows of the first n K blocks prefetched
 * into L2 before the programmatic-launch wait; 0 = auto: half-width units
 * only, -1 = off), "pdl_trigger" (where the SpMM releases its successor
 * under PDL: 1 = at entry, -1 = after the setup, 0 = auto: at entry for
 * one-K-block CTAs), "converter_legacy" (1: the converter's sort-based class grouping instead
 * of the class table + one-CTA planner; the same output).  All variants give results
 * within the same tolerance; V split, cp.async, gather warps and persistent
 * are bit-identical to the default.
 * Unknown key: BAD_PARAMS. */
int shflbw_cu_set_option(const char* key, int64_t value);
/* Number of kernels this library launched on the calling thread so far. */
int64_t shflbw_cu_launch_count(void);
/* The kernel variant of the last SpMM / conv call on the calling thread:
 * "k_spmm_tc ..." / "k_spmm_persist ..." (tcgen05; kind, V, V per CTA,
 * cluster size and split, gather warps, stages, tiles) or "k_spmm_simt ..."
 * (the CUDA-core kernel).  Lets callers and tests prove which path ran. */
const char* shflbw_cu_last_plan(void);

/* ---- converter (replaces validate_pattern(ShflBW), src/formats.cpp:113-138,
 *      and compress_shflbw, include/shflbw/formats.hpp:98-99 /
 *      src/formats.cpp:140-181) ------------------------------------------- */

/* mask [dev] M*K bytes, each 0 or 1.  *pass = 1/0; *fail_row = smallest row of
 * the lexicographically first support class whose size is not a multiple of
 * V.  BAD_PARAMS if V == 0, V does not divide M, or a mask byte > 1.
 * Synchronises `stream`. */
int shflbw_cu_validate(const uint8_t* mask, int32_t M, int32_t K, int32_t V,
                       int32_t* pass, uint32_t* fail_row, shflbw_stream_t stream);

/* dense [dev] M*K of dense_dtype, mask [dev] M*K bytes.  Builds *out (device
 * buffers owned by the library) with values rounded to value_dtype (RNE;
 * F32 keeps them exact).
 * NONCONFORMANT_MASK sets *fail_row.  Synchronises `stream` once (sizes). */
int shflbw_cu_compress(const void* dense, int32_t dense_dtype, const uint8_t* mask,
                       int32_t M, int32_t K, int32_t V, int32_t value_dtype,
                       shflbw_cu_matrix* out, uint32_t* fail_row,
                       shflbw_stream_t stream);

/* The converter without a host synchronisation (graph-capturable, stream
 * ordered like every kernel): *out is allocated from the bound
 * G * roundup(K, 64) columns and built on `stream`; status [dev] int32[4]
 * receives {status code, fail_row, total columns, widest group}.  A
 * non-conformant mask, a mask byte > 1 or an (astronomically unlikely) row
 * hash collision is reported there instead of being returned (the pipeline
 * stays in bounds).  The matrix may be used by SpMM / conv calls enqueued
 * after it; shflbw_cu_matrix_finalize (one synchronisation, e.g. outside a
 * captured graph) returns the status code -- NONCONFORMANT_MASK with
 * *fail_row, BAD_PARAMS, CUDA_ERROR -- and sets the exact total_cols /
 * max_group_cols.  Results equal shflbw_cu_compress's.  If *out already holds
 * a bound-allocated matrix of the same M, K, V and value dtype (from an
 * earlier compress_async), its buffers are reused: a captured graph then
 * converts into the same memory on every replay. */
int shflbw_cu_compress_async(const void* dense, int32_t dense_dtype, const uint8_t* mask,
                             int32_t M, int32_t K, int32_t V, int32_t value_dtype,
                             shflbw_cu_matrix* out, int32_t* status, shflbw_stream_t stream);
int shflbw_cu_matrix_finalize(shflbw_cu_matrix* m, const int32_t* status, uint32_t* fail_row,
                              shflbw_stream_t stream);

void shflbw_cu_matrix_free(shflbw_cu_matrix* m);

/* Host ShflBWMatrix (flattened: row_indices[M], group_ncols[G], cols[sum n_g],
 * values[V*sum n_g] f32) -> device layout.  ShapeMismatch on a row index >= M
 * or a column >= K (the reference checks the former in spmm_execute,
 * src/spmm.cpp:82-86, and the latter in stitch_tile, src/spmm.cpp:50-52). */
int shflbw_cu_matrix_upload(int32_t M, int32_t K, int32_t V,
                            const uint32_t* row_indices, const uint32_t* group_ncols,
                            const uint32_t* cols, const float* values,
                            int32_t value_dtype, shflbw_cu_matrix* out,
                            shflbw_stream_t stream);

/* Device layout -> host flattened ShflBWMatrix (values widened to f32).
 * cols / values capacity: sum n_g and V*sum n_g.  Synchronises `stream`. */
int shflbw_cu_matrix_download(const shflbw_cu_matrix* m, uint32_t* row_indices,
                              uint32_t* group_ncols, uint32_t* cols, float* values,
                              shflbw_stream_t stream);

/* The raw device layout -> host: group_ptr[G+1], col_idx[total_cols],
 * values[total_cols * V] as raw 2-byte (BF16/F16) or 4-byte (F32) words (for
 * layout checks and serialisers).
 * Synchronises `stream`. */
int shflbw_cu_matrix_export_raw(const shflbw_cu_matrix* m, int32_t* group_ptr, int32_t* col_idx,
                                void* values, shflbw_stream_t stream);

/* decompress(ShflBWMatrix), src/formats.cpp:195-206: dense [dev] M*K f32. */
int shflbw_cu_decompress(const shflbw_cu_matrix* m, float* dense, shflbw_stream_t stream);

/* ---- SpMM (replaces spmm_execute, include/shflbw/spmm.hpp:28-29 /
 *      src/spmm.cpp:76-146) ---------------------------------------------- */

/* C[row_indices[g*V+r]][n] = sum_j values[g][j][r] * B[col_idx[g][j]][n].
 * B [dev] K_b x N, row stride ldb elements, dtype == a->dtype.  BF16/F16
 * matrices run the tcgen05 kernel (V in {16,32,64,128}, ldb % 8 == 0) or the
 * exact CUDA-core kernel; F32 matrices run the CUDA-core kernel, bit-identical
 * to spmm_execute.
 * C [dev] M x N, row stride ldc, c_dtype F32 or BF16/F16.
 * ShapeMismatch if K_b != a->cols.  Asynchronous. */
int shflbw_cu_spmm(const shflbw_cu_matrix* a, const void* B, int32_t K_b, int32_t N,
                   int64_t ldb, void* C, int32_t c_dtype, int64_t ldc,
                   shflbw_stream_t stream);

/* One shard's share: groups [g_begin, g_end) (the reference's per-worker
 * run_groups range, src/spmm.cpp:93-144).  compact = 0 writes through
 * row_indices into the full C; compact = 1 writes group-ordered rows
 * C[(g - g_begin)*V + r] (input of an all-gather + shflbw_cu_unpermute_rows). */
int shflbw_cu_spmm_groups(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end,
                          const void* B, int32_t K_b, int32_t N, int64_t ldb, void* C,
                          int32_t c_dtype, int64_t ldc, int32_t compact,
                          shflbw_stream_t stream);

/* The row-sharded SpMM with the all-gather fused into its epilogue (SURVEY.md
 * §8(e)): groups [g_begin, g_end) computed once, each finished output row
 * stored at its row_indices position into every buffer of C_dst[0..n_dst)
 * -- this GPU's full C and the peer GPUs' full C through P2P mappings
 * (cudaIpcOpenMemHandle / cudaDeviceEnablePeerAccess) -- with the same
 * 16-byte stores, so the transfer overlaps the remaining tiles' math and no
 * collective or unpermute pass follows.  The caller orders the consumers
 * after every rank's call (a cross-GPU barrier).  bf16 / f16 output, the
 * tcgen05 path (else UNSUPPORTED); n_dst in 1..8; buffers 16-byte aligned
 * with the same ldc. */
int shflbw_cu_spmm_groups_peers(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end,
                                const void* B, int32_t K_b, int32_t N, int64_t ldb,
                                void* const* C_dst, int32_t n_dst, int32_t c_dtype,
                                int64_t ldc, shflbw_stream_t stream);

/* The same with the gather through NVLink SHARP (NVLS) multicast: C_mc is a
 * multicast address bound to every rank's full C (e.g. torch symmetric
 * memory's multicast_ptr, or cuMulticastCreate + cuMulticastBindMem +
 * cuMemMap); each finished 16-byte row chunk is ONE multimem.st that the
 * NVSwitch replicates into all GPUs' outputs (the P2P variant above issues P
 * stores).  bf16 / f16 output, the tcgen05 path, same ordering contract. */
int shflbw_cu_spmm_groups_multicast(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end,
                                    const void* B, int32_t K_b, int32_t N, int64_t ldb,
                                    void* C_mc, int32_t c_dtype, int64_t ldc,
                                    shflbw_stream_t stream);

/* Conv weight layout (cf. a library's one-time filter reorder): *out = a copy
 * of w whose columns are, per group, ordered by filter column s = c % S
 * (ascending c within each s) with every s-run padded to a multiple of 4 by
 * pad columns (index SHFLBW_PAD_COLUMN, zero values).  shflbw_cu_conv2d then
 * fetches each activation row as 64/Nb adjacent output positions x Nb
 * (128 bytes) instead of one position (Nb*2 bytes) when stride = 1,
 * Nb in {16, 32} and 64/Nb divides Q.  Same values, so conv2d (and spmm) stay
 * within the 1e-5 tolerance; only the fp32 summation order changes.
 * matrix_download rejects the result (its columns are not ascending).
 * S in 1..32.  Synchronises `stream`. */
int shflbw_cu_conv_prepare(const shflbw_cu_matrix* w, int32_t S, shflbw_cu_matrix* out,
                           shflbw_stream_t stream);

/* Permutation folding (the paper's layout fusion,
 * PAPER.md:181-183).  A layer whose SpMM wrote group-ordered rows
 * (shflbw_cu_spmm_groups over all groups with compact = 1: row i holds logical
 * row producer_rows[i], producer_rows = that layer's row_indices) feeds the
 * next layer `a` directly once a's column indices are remapped through the
 * inverse permutation, col -> i with producer_rows[i] == col.  No un-permute
 * pass, and under sharding no scatter after the all-gather.  Rewrites
 * a->col_idx in place; values and accumulation order are unchanged, so every
 * result is bit-identical to the unfolded chain.  producer_rows [dev] holds
 * a->cols entries and must be a permutation of 0..a->cols-1 (else
 * BAD_PARAMS, matrix unchanged).  Sets SHFLBW_FOLDED in a->reserved; conv2d
 * and matrix_download reject folded matrices (decompress returns the weight
 * over the folded input order, W[:, producer_rows]).  Synchronises `stream`. */
int shflbw_cu_fold_input_permutation(shflbw_cu_matrix* a, const int32_t* producer_rows,
                                     shflbw_stream_t stream);

/* ---- pruning: the converter's upstream producer (
 *      include/shflbw/pruning.hpp:27-94, src/pruning.cpp) ------------------
 * Importance scores are M x K f32 [dev], finite and >= 0 (else BAD_PARAMS,
 * the ImportanceMatrix ctor, src/pruning.cpp:35-44).  Masks are M x K bytes
 * [dev] (0/1).  Every result is identical to the reference's: the integer
 * and index work is exact and every double sum runs in the reference's
 * order with separately rounded operations. */
typedef struct shflbw_prune_config {
    double alpha;              /* target non-zero ratio, (0, 1]             */
    double beta_factor;        /* beta = min(1, beta_factor * alpha)        */
    uint32_t v;                /* group size, divides M                     */
    uint32_t kmeans_max_iters; /* >= 1                                      */
    uint64_t seed;
    uint32_t restarts;         /* >= 1                                      */
    uint32_t reserved;
} shflbw_prune_config;

/* scores[i] = |w[i]| (importance_scores, src/pruning.cpp:61-66). */
int shflbw_cu_importance_scores(const float* w, int64_t n, float* scores, shflbw_stream_t stream);
/* *out = sum of scores where mask (kept_score, src/pruning.cpp:68-75), in the
 * reference's linear order.  Synchronises `stream`. */
int shflbw_cu_kept_score(const float* scores, const uint8_t* mask, int32_t M, int32_t K, double* out,
                         shflbw_stream_t stream);
/* Top llround(keep_ratio*M*K) entries, ties to the lower linear index
 * (prune_unstructured, src/pruning.cpp:77-92). */
int shflbw_cu_prune_unstructured(const float* scores, int32_t M, int32_t K, double keep_ratio,
                                 uint8_t* mask, shflbw_stream_t stream);
/* Per group of V consecutive rows, the llround(alpha*K) columns with the
 * largest score sums (prune_vectorwise, src/pruning.cpp:94-121). */
int shflbw_cu_prune_vectorwise(const float* scores, int32_t M, int32_t K, uint32_t V, double alpha,
                               uint8_t* mask, shflbw_stream_t stream);
/* Balanced K-Means row grouping of `mask` with `restarts` seeds, scored by
 * the vector-wise prune of the permuted scores (kmeans_row_grouping,
 * src/pruning.cpp:183-337): order[i] = original row at grouped position i. */
int shflbw_cu_kmeans_row_grouping(const uint8_t* mask, const float* scores, int32_t M, int32_t K,
                                  const shflbw_prune_config* cfg, uint32_t* order, shflbw_stream_t stream);
/* prune_shflbw (src/pruning.cpp:339-362): mask [dev] M x K, permutation
 * [dev] M, *kept_score.  Synchronises `stream`. */
int shflbw_cu_prune_shflbw(const float* scores, int32_t M, int32_t K, const shflbw_prune_config* cfg,
                           uint8_t* mask, uint32_t* permutation, double* kept_score, shflbw_stream_t stream);

/* ---- SMX1 container <-> device layout (the reference's
 *      on-disk format, include/shflbw/container.hpp:14-22) ------------------ */

/* bytes [host] = a whole SMX1 file.  Kind 3 (Shfl-BW): validated with the
 * reference's rules (decode_container + as_shflbw, src/container.cpp:147-215,
 * :90-134) and uploaded into *out with values rounded to value_dtype (F32
 * keeps them exact).  BAD_MAGIC / UNSUPPORTED_VERSION / CORRUPT_PAYLOAD as the
 * reference; another valid kind (0, 1, 2, 4) -> BAD_PARAMS without walking its
 * payload.  Synchronises `stream`. */
int shflbw_cu_smx1_decode(const void* bytes, uint64_t nbytes, int32_t value_dtype,
                          shflbw_cu_matrix* out, shflbw_stream_t stream);
/* *m -> SMX1 kind-3 bytes (encode_container, src/container.cpp:141-145):
 * *nbytes = the file size; bytes [host] == NULL is a size query.  Values are
 * written as f32 (exact widening of bf16/f16), so a matrix decoded with F32
 * values re-encodes byte-identically.  Folded / conv-ordered matrices:
 * BAD_PARAMS.  Synchronises `stream`. */
int shflbw_cu_smx1_encode(const shflbw_cu_matrix* m, void* bytes, uint64_t capacity,
                          uint64_t* nbytes, shflbw_stream_t stream);

/* C[row_indices[r]][:] = C_perm[r][:] for r < M (2- or 4-byte elements);
 * rows with row_indices[r] < 0 (padding of an all-gathered buffer) are skipped. */
int shflbw_cu_unpermute_rows(const int32_t* row_indices, int32_t M, int32_t N,
                             const void* C_perm, int64_t ld_perm, void* C, int64_t ldc,
                             int32_t dtype, shflbw_stream_t stream);

/* ---- sparse convolution (replaces conv2d, include/shflbw/spmm.hpp:87-89 /
 *      src/spmm.cpp:193-291, and conv_output_size, src/spmm.cpp:177-191) ---- */

int shflbw_cu_conv_output_size(int32_t H, int32_t W, int32_t R, int32_t S,
                               int32_t stride, int32_t pad, int32_t* P, int32_t* Q);

/* input [dev] [C][H][W][Nb] (dtype == w->dtype); out [dev] [K_f][P][Q][Nb] of
 * out_dtype.  Weights are K_f x C*R*S; column c decodes to
 * (c / (R*S), (c % (R*S)) / S, c % S).  BadGeometry as the reference. */
int shflbw_cu_conv2d(const shflbw_cu_matrix* w, const void* input, int32_t C, int32_t H,
                     int32_t W, int32_t Nb, int32_t R, int32_t S, int32_t stride,
                     int32_t pad, void* out, int32_t out_dtype, shflbw_stream_t stream);

/* ---- the reference's public helpers, on the device ------------------------ */

/* spmm_dense_oracle (src/spmm.cpp:148-161): C = A*B, fp32, each product
 * rounded then added, k ascending (bit-identical to the reference loop).
 * A [dev] MxK, B [dev] KxN, C [dev] MxN. */
int shflbw_cu_dense_matmul_f32(const float* A, int32_t M, int32_t K, const float* B, int32_t N,
                               float* C, shflbw_stream_t stream);

/* stitch_tile (src/spmm.cpp:37-58): staging [dev] t_k x t_n row-major gets
 * the rows of B [dev] named by group_cols[chunk_begin..+t_k) [dev], zero past
 * the list or B's edge; ShapeMismatch if a named row >= B_rows (synchronises). */
int shflbw_cu_stitch_tile(const uint32_t* group_cols, int64_t ncols, int64_t chunk_begin,
                          int64_t t_k, const float* B, int32_t B_rows, int32_t B_cols,
                          int64_t slice_begin, int64_t t_n, float* staging,
                          shflbw_stream_t stream);

/* tile_mma (src/spmm.cpp:60-74): acc [dev] v_rows x t_n += a_tile (column-major
 * v_rows x k_len) * b_tile (k_len x t_n), products added one k at a time. */
int shflbw_cu_tile_mma(float* acc, const float* a_tile, const float* b_tile, int64_t v_rows,
                       int64_t k_len, int64_t t_n, shflbw_stream_t stream);

/* ---- utilities ---------------------------------------------------------- */

/* dst[i] = (dst_dtype) src[i], RNE; src_dtype/dst_dtype any of F32/BF16/F16. */
int shflbw_cu_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype,
                      int64_t n, shflbw_stream_t stream);
/* Pitched form: dst[r*ld_dst + c] = (dst_dtype) src[r*ld_src + c] for r < rows,
 * c < cols (one launch; e.g. an fp32 host matrix into a 16-byte aligned
 * 16-bit operand). */
int shflbw_cu_convert_2d(const void* src, int32_t src_dtype, int64_t ld_src, void* dst,
                         int32_t dst_dtype, int64_t ld_dst, int64_t rows, int64_t cols,
                         shflbw_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SHFLBW_CU_H */
