/*
 * shflbw_oracle.h -- CPU restatement of the reference Shfl-BW hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2203_05016_b200/) links, loads or calls this code.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it,
 * and only as the checker.
 *
 * Parity is pinned two ways:
 *   1. the fixtures under tests/golden/ were produced by the reference itself
 *      (oracle/_ref/libshflbw_ref.so, compiled from /root/reference/proj/src
 *      by oracle/Makefile) and tests/test_oracle.py checks this restatement
 *      against them;
 *   2. when oracle/_ref is built, tests compare the two directly.
 *
 * Conventions: all matrices are row-major.  A compressed matrix is the
 * reference's ShflBWMatrix (include/shflbw/formats.hpp:14-42) flattened:
 *   row_indices[M]        original row of compressed row r
 *   group_ncols[G]        n_g, columns kept by group g
 *   cols[sum n_g]         per-group strictly increasing column lists, concatenated
 *   values[V * sum n_g]   per-group column-major V x n_g blocks, concatenated
 */
#ifndef SHFLBW_ORACLE_H
#define SHFLBW_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: same numbering as include/shflbw_cu.h. */
#define ORC_OK 0
#define ORC_SHAPE_MISMATCH 1
#define ORC_NONCONFORMANT_MASK 2
#define ORC_BAD_PARAMS 3
#define ORC_BAD_GEOMETRY 4

/* std::mt19937_64 (the reference seeds it directly, include/shflbw/rng.hpp). */
typedef struct orc_rng {
    uint64_t state[312];
    int pos;
} orc_rng;

void orc_rng_seed(orc_rng* g, uint64_t seed);
uint64_t orc_rng_next(orc_rng* g);
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* g);
double orc_uniform01(orc_rng* g);
float orc_uniform_float(orc_rng* g, float lo, float hi);
void orc_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out);
void orc_fill_uniform(orc_rng* g, size_t n, float lo, float hi, float* out);

/* tests/test_helpers.hpp generators */
void orc_random_vector_wise_mask(uint32_t m, uint32_t k, uint32_t v,
                                 uint32_t cols_per_group, orc_rng* g,
                                 uint8_t* mask);
void orc_random_permutation(uint32_t m, orc_rng* g, uint32_t* perm);
void orc_random_shflbw_mask(uint32_t m, uint32_t k, uint32_t v,
                            uint32_t cols_per_group, orc_rng* g,
                            uint8_t* mask);

/* validate_pattern(ShflBW): pass=1/0, fail_row = front of the first failing
 * support class in lexicographic order. */
int orc_validate_shflbw(const uint8_t* mask, uint32_t M, uint32_t K, uint32_t V,
                        int* pass, uint32_t* fail_row);

/* compress_shflbw.  cols and values must hold M*K entries (upper bound). */
int orc_compress(const float* dense, const uint8_t* mask, uint32_t M, uint32_t K,
                 uint32_t V, uint32_t* row_indices, uint32_t* group_ncols,
                 uint32_t* cols, float* values, uint32_t* fail_row);

/* decompress(ShflBWMatrix) */
void orc_decompress(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                    const uint32_t* group_ncols, const uint32_t* cols,
                    const float* values, float* dense);

/* spmm_execute, in the reference's pinned reduction order. */
int orc_spmm(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
             const uint32_t* group_ncols, const uint32_t* cols,
             const float* values, const float* B, uint32_t B_rows, uint32_t N,
             float* C);
/* spmm_execute restricted to groups [g_begin, g_end) (one worker's share). */
void orc_spmm_groups(uint32_t M, uint32_t V, const uint32_t* row_indices,
                     const uint32_t* group_ncols, const uint32_t* cols,
                     const float* values, const float* B, uint32_t N,
                     uint32_t g_begin, uint32_t g_end, float* C);

void orc_spmm_dense(const float* A, uint32_t M, uint32_t K, const float* B,
                    uint32_t N, float* C);
double orc_rel_frobenius(const float* x, const float* y, size_t n);

int orc_conv_output_size(uint32_t H, uint32_t W, uint32_t R, uint32_t S,
                         uint32_t stride, uint32_t pad, uint32_t* P, uint32_t* Q);
int orc_conv2d(uint32_t Kf, uint32_t Kcols, uint32_t V, const uint32_t* row_indices,
               const uint32_t* group_ncols, const uint32_t* cols,
               const float* values, const float* input, uint32_t C, uint32_t H,
               uint32_t W, uint32_t Nb, uint32_t R, uint32_t S, uint32_t stride,
               uint32_t pad, float* out);
/* direct conv with double accumulation (tests/test_conv.cpp:14-42 oracle) */
int orc_conv_direct(const float* w_dense, uint32_t Kf, const float* input,
                    uint32_t C, uint32_t H, uint32_t W, uint32_t Nb, uint32_t R,
                    uint32_t S, uint32_t stride, uint32_t pad, float* out);

/* stitch_to_blockwise: tiles of tile_width, kPadColumn padding. Returns the
 * number of tiles written (tile_cols: ntiles*tile_width, tile_vals:
 * ntiles*tile_width*V, tile_group: ntiles). */
int orc_stitch_to_blockwise(uint32_t V, uint32_t G, const uint32_t* group_ncols,
                            const uint32_t* cols, const float* values,
                            uint32_t tile_width, uint32_t* tile_cols,
                            float* tile_vals, uint32_t* tile_group);

/* 16-bit conversions, round-to-nearest-even. */
uint16_t orc_f32_to_bf16(float x);
float orc_bf16_to_f32(uint16_t h);
uint16_t orc_f32_to_f16(float x);
float orc_f16_to_f32(uint16_t h);
/* round every element through bf16 (dtype 1) or fp16 (dtype 2) in place */
void orc_round16(float* x, size_t n, int dtype);

/* The device packed layout (include/shflbw_cu.h, shflbw_cu_matrix): each
 * group's column list padded to a multiple of k_tile with kPadColumn (-1)
 * and zero values, values as 16-bit (dtype 1 = bf16, 2 = fp16).
 * group_ptr[G+1] = prefix sum of padded counts.  Returns total padded cols. */
int64_t orc_pack_device(uint32_t M, uint32_t V, const uint32_t* group_ncols,
                        const uint32_t* cols, const float* values, uint32_t k_tile,
                        int dtype, int32_t* group_ptr, int32_t* col_idx,
                        uint16_t* vals16);

#ifdef __cplusplus
}
#endif
#endif
