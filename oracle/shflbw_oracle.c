/*
 * shflbw_oracle.c -- CPU restatement of the reference Shfl-BW hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see shflbw_oracle.h).  Built with
 * -ffp-contract=off, like the reference (/root/reference/proj/CMakeLists.txt:12-16),
 * so every float product is rounded before it is added.
 *
 * Each function cites the reference code it restates; paths are relative to
 * /root/reference/proj.
 */
#include "shflbw_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Random numbers: std::mt19937_64 as seeded by include/shflbw/rng.hpp:14-24 */
/* ------------------------------------------------------------------------ */

enum { MT_N = 312, MT_M = 156 };
static const uint64_t MT_MATRIX_A = 0xB5026F5AA96619E9ULL;
static const uint64_t MT_UPPER = 0xFFFFFFFF80000000ULL;
static const uint64_t MT_LOWER = 0x000000007FFFFFFFULL;

void orc_rng_seed(orc_rng* g, uint64_t seed) {
    g->state[0] = seed;
    for (int i = 1; i < MT_N; ++i) {
        const uint64_t prev = g->state[i - 1];
        g->state[i] = 6364136223846793005ULL * (prev ^ (prev >> 62)) + (uint64_t)i;
    }
    g->pos = MT_N;
}

static void mt_twist(orc_rng* g) {
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t y = (g->state[i] & MT_UPPER) | (g->state[(i + 1) % MT_N] & MT_LOWER);
        uint64_t next = g->state[(i + MT_M) % MT_N] ^ (y >> 1);
        if (y & 1ULL) next ^= MT_MATRIX_A;
        g->state[i] = next;
    }
    g->pos = 0;
}

uint64_t orc_rng_next(orc_rng* g) {
    if (g->pos >= MT_N) mt_twist(g);
    uint64_t z = g->state[g->pos++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

orc_rng* orc_rng_new(uint64_t seed) {
    orc_rng* g = (orc_rng*)malloc(sizeof(orc_rng));
    if (g) orc_rng_seed(g, seed);
    return g;
}

void orc_rng_free(orc_rng* g) { free(g); }

/* include/shflbw/rng.hpp:14-16 */
double orc_uniform01(orc_rng* g) {
    return (double)(orc_rng_next(g) >> 11) * 0x1.0p-53;
}

/* include/shflbw/rng.hpp:18-20 (float arithmetic, no contraction) */
float orc_uniform_float(orc_rng* g, float lo, float hi) {
    const float u = (float)orc_uniform01(g);
    const float span = hi - lo;
    const float scaled = u * span;
    return lo + scaled;
}

void orc_fill_uniform(orc_rng* g, size_t n, float lo, float hi, float* out) {
    for (size_t i = 0; i < n; ++i) out[i] = orc_uniform_float(g, lo, hi);
}

/* src/rng.cpp:6-12 */
void orc_random_dense(uint32_t rows, uint32_t cols, uint64_t seed, float* out) {
    orc_rng g;
    orc_rng_seed(&g, seed);
    orc_fill_uniform(&g, (size_t)rows * cols, -1.0f, 1.0f, out);
}

/* tests/test_helpers.hpp:17-32: every V-row group keeps the same
 * cols_per_group columns, chosen by a partial Fisher-Yates shuffle. */
void orc_random_vector_wise_mask(uint32_t m, uint32_t k, uint32_t v,
                                 uint32_t cols_per_group, orc_rng* g,
                                 uint8_t* mask) {
    memset(mask, 0, (size_t)m * k);
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (k ? k : 1));
    for (uint32_t grp = 0; (uint64_t)grp * v < m; ++grp) {
        for (uint32_t c = 0; c < k; ++c) order[c] = c;
        for (uint32_t j = 0; j < cols_per_group; ++j) {
            const uint32_t pick = j + (uint32_t)(orc_rng_next(g) % (uint64_t)(k - j));
            const uint32_t tmp = order[j];
            order[j] = order[pick];
            order[pick] = tmp;
        }
        for (uint32_t j = 0; j < cols_per_group; ++j)
            for (uint32_t i = 0; i < v; ++i) {
                const uint64_t r = (uint64_t)grp * v + i;
                if (r < m) mask[r * k + order[j]] = 1;
            }
    }
    free(order);
}

/* tests/test_helpers.hpp:34-41 */
void orc_random_permutation(uint32_t m, orc_rng* g, uint32_t* perm) {
    for (uint32_t i = 0; i < m; ++i) perm[i] = i;
    for (uint32_t i = 0; i + 1 < m; ++i) {
        const uint32_t pick = i + (uint32_t)(orc_rng_next(g) % (uint64_t)(m - i));
        const uint32_t tmp = perm[i];
        perm[i] = perm[pick];
        perm[pick] = tmp;
    }
}

/* tests/test_helpers.hpp:44-55: a vector-wise mask whose rows are scattered
 * by a random permutation (row r of the VW mask lands on row perm[r]). */
void orc_random_shflbw_mask(uint32_t m, uint32_t k, uint32_t v,
                            uint32_t cols_per_group, orc_rng* g, uint8_t* mask) {
    uint8_t* vw = (uint8_t*)malloc((size_t)m * k + 1);
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (m + 1));
    orc_random_vector_wise_mask(m, k, v, cols_per_group, g, vw);
    orc_random_permutation(m, g, perm);
    for (uint32_t r = 0; r < m; ++r)
        memcpy(mask + (size_t)perm[r] * k, vw + (size_t)r * k, k);
    free(perm);
    free(vw);
}

/* ------------------------------------------------------------------------ */
/* Support classes (src/formats.cpp:40-46).  The reference keys a std::map  */
/* by the whole mask row, so classes come out in lexicographic byte order,  */
/* members ascending.  Restated as a stable sort of row ids by (row bytes,  */
/* row id); equal-byte runs are the classes.                                */
/* ------------------------------------------------------------------------ */

typedef struct {
    const uint8_t* mask;
    uint32_t K;
} row_order_ctx;

static int row_less(const row_order_ctx* ctx, uint32_t a, uint32_t b) {
    const int c = memcmp(ctx->mask + (size_t)a * ctx->K, ctx->mask + (size_t)b * ctx->K, ctx->K);
    if (c != 0) return c < 0;
    return a < b;
}

static void merge_sort_rows(const row_order_ctx* ctx, uint32_t* a, uint32_t* tmp, uint32_t n) {
    if (n < 2) return;
    const uint32_t h = n / 2;
    merge_sort_rows(ctx, a, tmp, h);
    merge_sort_rows(ctx, a + h, tmp, n - h);
    uint32_t i = 0, j = h, o = 0;
    while (i < h && j < n) tmp[o++] = row_less(ctx, a[j], a[i]) ? a[j++] : a[i++];
    while (i < h) tmp[o++] = a[i++];
    while (j < n) tmp[o++] = a[j++];
    memcpy(a, tmp, sizeof(uint32_t) * n);
}

/* Returns the rows in class order; *nclass and class_start[nclass+1] give runs. */
static uint32_t* support_classes(const uint8_t* mask, uint32_t M, uint32_t K,
                                 uint32_t** class_start_out, uint32_t* nclass_out) {
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (M + 1));
    uint32_t* tmp = (uint32_t*)malloc(sizeof(uint32_t) * (M + 1));
    for (uint32_t r = 0; r < M; ++r) order[r] = r;
    row_order_ctx ctx = {mask, K};
    merge_sort_rows(&ctx, order, tmp, M);
    uint32_t* starts = (uint32_t*)malloc(sizeof(uint32_t) * (M + 2));
    uint32_t nclass = 0;
    for (uint32_t i = 0; i < M; ++i) {
        if (i == 0 || memcmp(mask + (size_t)order[i] * K, mask + (size_t)order[i - 1] * K, K) != 0)
            starts[nclass++] = i;
    }
    starts[nclass] = M;
    free(tmp);
    *class_start_out = starts;
    *nclass_out = nclass;
    return order;
}

/* validate_pattern(ShflBW) = src/formats.cpp:113-125 + validate_shfl_bw
 * src/formats.cpp:85-93: every class size must be a multiple of V; the first
 * failing class (map order) reports its smallest member. */
int orc_validate_shflbw(const uint8_t* mask, uint32_t M, uint32_t K, uint32_t V,
                        int* pass, uint32_t* fail_row) {
    if (V == 0 || M % V != 0) return ORC_BAD_PARAMS;
    uint32_t* starts;
    uint32_t nclass;
    uint32_t* order = support_classes(mask, M, K, &starts, &nclass);
    *pass = 1;
    *fail_row = 0;
    for (uint32_t c = 0; c < nclass; ++c) {
        if ((starts[c + 1] - starts[c]) % V != 0) {
            *pass = 0;
            *fail_row = order[starts[c]];
            break;
        }
    }
    free(order);
    free(starts);
    return ORC_OK;
}

static int cmp_u32_pair_first(const void* a, const void* b) {
    const uint32_t x = ((const uint32_t*)a)[0], y = ((const uint32_t*)b)[0];
    return (x > y) - (x < y);
}

/* compress_shflbw, src/formats.cpp:140-181.  Classes are cut into V-row
 * chunks (ascending rows), chunks ordered by their first row; each group's
 * columns are its leader row's set bits; values[j*V+i] = dense[rows[i]][cols[j]]. */
int orc_compress(const float* dense, const uint8_t* mask, uint32_t M, uint32_t K,
                 uint32_t V, uint32_t* row_indices, uint32_t* group_ncols,
                 uint32_t* cols, float* values, uint32_t* fail_row) {
    int pass = 1;
    const int st = orc_validate_shflbw(mask, M, K, V, &pass, fail_row);
    if (st != ORC_OK) return st;
    if (!pass) return ORC_NONCONFORMANT_MASK;

    uint32_t* starts;
    uint32_t nclass;
    uint32_t* order = support_classes(mask, M, K, &starts, &nclass);
    const uint32_t G = V ? M / V : 0;
    /* (first row, position of the chunk in `order`) */
    uint32_t* chunks = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (G + 1));
    uint32_t n = 0;
    for (uint32_t c = 0; c < nclass; ++c)
        for (uint32_t i = starts[c]; i < starts[c + 1]; i += V) {
            chunks[2 * n] = order[i];
            chunks[2 * n + 1] = i;
            ++n;
        }
    qsort(chunks, n, 2 * sizeof(uint32_t), cmp_u32_pair_first);

    size_t col_off = 0;
    for (uint32_t g = 0; g < n; ++g) {
        const uint32_t* rows = order + chunks[2 * g + 1];
        const uint8_t* lead = mask + (size_t)rows[0] * K;
        uint32_t ng = 0;
        for (uint32_t c = 0; c < K; ++c)
            if (lead[c]) cols[col_off + ng++] = c;
        for (uint32_t j = 0; j < ng; ++j)
            for (uint32_t i = 0; i < V; ++i)
                values[(col_off + j) * V + i] = dense[(size_t)rows[i] * K + cols[col_off + j]];
        group_ncols[g] = ng;
        memcpy(row_indices + (size_t)g * V, rows, sizeof(uint32_t) * V);
        col_off += ng;
    }
    free(chunks);
    free(order);
    free(starts);
    return ORC_OK;
}

/* decompress(ShflBWMatrix), src/formats.cpp:195-206 */
void orc_decompress(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
                    const uint32_t* group_ncols, const uint32_t* cols,
                    const float* values, float* dense) {
    memset(dense, 0, sizeof(float) * (size_t)M * K);
    const uint32_t G = V ? M / V : 0;
    size_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        for (uint32_t j = 0; j < group_ncols[g]; ++j)
            for (uint32_t i = 0; i < V; ++i)
                dense[(size_t)row_indices[(size_t)g * V + i] * K + cols[off + j]] =
                    values[(off + j) * V + i];
        off += group_ncols[g];
    }
}

/* One worker's share of spmm_execute (src/spmm.cpp:93-126): for every output
 * element, kept columns are accumulated in ascending k starting from 0.0f --
 * the order tile_mma pins (src/spmm.cpp:60-74), independent of t_n/t_k.  The
 * accumulated V rows are written to rows row_indices[g*V + v]
 * (src/spmm.cpp:115-123). */
void orc_spmm_groups(uint32_t M, uint32_t V, const uint32_t* row_indices,
                     const uint32_t* group_ncols, const uint32_t* cols,
                     const float* values, const float* B, uint32_t N,
                     uint32_t g_begin, uint32_t g_end, float* C) {
    (void)M;
    size_t off = 0;
    for (uint32_t g = 0; g < g_begin; ++g) off += group_ncols[g];
    float* acc = (float*)malloc(sizeof(float) * ((size_t)N + 1));
    for (uint32_t g = g_begin; g < g_end; ++g) {
        const uint32_t ng = group_ncols[g];
        for (uint32_t vi = 0; vi < V; ++vi) {
            for (uint32_t j = 0; j < N; ++j) acc[j] = 0.0f;
            for (uint32_t t = 0; t < ng; ++t) {
                const float a = values[(off + t) * V + vi];
                const float* brow = B + (size_t)cols[off + t] * N;
                for (uint32_t j = 0; j < N; ++j) {
                    const float prod = a * brow[j];
                    acc[j] = acc[j] + prod;
                }
            }
            memcpy(C + (size_t)row_indices[(size_t)g * V + vi] * N, acc, sizeof(float) * N);
        }
        off += ng;
    }
    free(acc);
}

/* spmm_execute, src/spmm.cpp:76-146 (checks at src/spmm.cpp:80-86). */
int orc_spmm(uint32_t M, uint32_t K, uint32_t V, const uint32_t* row_indices,
             const uint32_t* group_ncols, const uint32_t* cols,
             const float* values, const float* B, uint32_t B_rows, uint32_t N,
             float* C) {
    if (K != B_rows) return ORC_SHAPE_MISMATCH;
    for (uint32_t r = 0; r < M; ++r)
        if (row_indices[r] >= M) return ORC_SHAPE_MISMATCH;
    memset(C, 0, sizeof(float) * (size_t)M * N);
    orc_spmm_groups(M, V, row_indices, group_ncols, cols, values, B, N, 0, V ? M / V : 0, C);
    return ORC_OK;
}

/* spmm_dense_oracle, src/spmm.cpp:148-161 */
void orc_spmm_dense(const float* A, uint32_t M, uint32_t K, const float* B,
                    uint32_t N, float* C) {
    for (uint32_t i = 0; i < M; ++i)
        for (uint32_t j = 0; j < N; ++j) {
            float acc = 0.0f;
            for (uint32_t k = 0; k < K; ++k) {
                const float prod = A[(size_t)i * K + k] * B[(size_t)k * N + j];
                acc = acc + prod;
            }
            C[(size_t)i * N + j] = acc;
        }
}

/* relative_frobenius_error, src/spmm.cpp:163-175 */
double orc_rel_frobenius(const float* x, const float* y, size_t n) {
    double num = 0.0, den = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double d = (double)x[i] - (double)y[i];
        num += d * d;
        den += (double)y[i] * (double)y[i];
    }
    if (den == 0.0) return num == 0.0 ? 0.0 : INFINITY;
    return sqrt(num) / sqrt(den);
}

/* conv_output_size, src/spmm.cpp:177-191 */
int orc_conv_output_size(uint32_t H, uint32_t W, uint32_t R, uint32_t S,
                         uint32_t stride, uint32_t pad, uint32_t* P, uint32_t* Q) {
    if (R == 0 || S == 0 || stride == 0) return ORC_BAD_GEOMETRY;
    const int64_t span_h = (int64_t)H + 2 * (int64_t)pad - (int64_t)R;
    const int64_t span_w = (int64_t)W + 2 * (int64_t)pad - (int64_t)S;
    if (span_h < 0 || span_w < 0 || span_h % stride != 0 || span_w % stride != 0)
        return ORC_BAD_GEOMETRY;
    *P = (uint32_t)(span_h / stride + 1);
    *Q = (uint32_t)(span_w / stride + 1);
    return ORC_OK;
}

/* conv2d, src/spmm.cpp:193-291.  Sparse column c decodes to
 * (ch, r, s) = (c / RS, (c % RS) / S, c % S); flat output column
 * jj = (p*Q + q)*Nb + n; out-of-image taps stage 0.0f and still enter the sum
 * (src/spmm.cpp:250-255). */
int orc_conv2d(uint32_t Kf, uint32_t Kcols, uint32_t V, const uint32_t* row_indices,
               const uint32_t* group_ncols, const uint32_t* cols,
               const float* values, const float* input, uint32_t C, uint32_t H,
               uint32_t W, uint32_t Nb, uint32_t R, uint32_t S, uint32_t stride,
               uint32_t pad, float* out) {
    uint32_t P = 0, Q = 0;
    const int st = orc_conv_output_size(H, W, R, S, stride, pad, &P, &Q);
    if (st != ORC_OK) return st;
    if ((uint64_t)Kcols != (uint64_t)C * R * S) return ORC_BAD_GEOMETRY;
    for (uint32_t r = 0; r < Kf; ++r)
        if (row_indices[r] >= Kf) return ORC_BAD_GEOMETRY;
    const uint32_t RS = R * S;
    const size_t flat = (size_t)P * Q * Nb;
    const uint32_t G = V ? Kf / V : 0;
    memset(out, 0, sizeof(float) * (size_t)Kf * flat);
    float* acc = (float*)malloc(sizeof(float) * (flat + 1));
    size_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = group_ncols[g];
        for (uint32_t vi = 0; vi < V; ++vi) {
            for (size_t jj = 0; jj < flat; ++jj) acc[jj] = 0.0f;
            for (uint32_t t = 0; t < ng; ++t) {
                const uint32_t col = cols[off + t];
                const uint32_t ch = col / RS, fr = (col % RS) / S, fs = col % S;
                const float a = values[(off + t) * V + vi];
                for (size_t jj = 0; jj < flat; ++jj) {
                    const uint32_t n = (uint32_t)(jj % Nb);
                    const size_t pq = jj / Nb;
                    const uint32_t q = (uint32_t)(pq % Q), p = (uint32_t)(pq / Q);
                    const int64_t h = (int64_t)p * stride + fr - (int64_t)pad;
                    const int64_t w = (int64_t)q * stride + fs - (int64_t)pad;
                    float x = 0.0f;
                    if (h >= 0 && h < (int64_t)H && w >= 0 && w < (int64_t)W)
                        x = input[(((size_t)ch * H + (size_t)h) * W + (size_t)w) * Nb + n];
                    const float prod = a * x;
                    acc[jj] = acc[jj] + prod;
                }
            }
            memcpy(out + (size_t)row_indices[(size_t)g * V + vi] * flat, acc, sizeof(float) * flat);
        }
        off += ng;
    }
    free(acc);
    return ORC_OK;
}

/* direct convolution with double accumulation, tests/test_conv.cpp:14-42 */
int orc_conv_direct(const float* w_dense, uint32_t Kf, const float* input,
                    uint32_t C, uint32_t H, uint32_t W, uint32_t Nb, uint32_t R,
                    uint32_t S, uint32_t stride, uint32_t pad, float* out) {
    uint32_t P = 0, Q = 0;
    const int st = orc_conv_output_size(H, W, R, S, stride, pad, &P, &Q);
    if (st != ORC_OK) return st;
    const size_t crs = (size_t)C * R * S;
    for (uint32_t f = 0; f < Kf; ++f)
        for (uint32_t p = 0; p < P; ++p)
            for (uint32_t q = 0; q < Q; ++q)
                for (uint32_t n = 0; n < Nb; ++n) {
                    double acc = 0.0;
                    for (uint32_t ci = 0; ci < C; ++ci)
                        for (uint32_t r = 0; r < R; ++r)
                            for (uint32_t s = 0; s < S; ++s) {
                                const int64_t h = (int64_t)p * stride + r - (int64_t)pad;
                                const int64_t w = (int64_t)q * stride + s - (int64_t)pad;
                                if (h < 0 || h >= (int64_t)H || w < 0 || w >= (int64_t)W) continue;
                                acc += (double)w_dense[(size_t)f * crs + ((size_t)ci * R + r) * S + s] *
                                       (double)input[(((size_t)ci * H + (size_t)h) * W + (size_t)w) * Nb + n];
                            }
                    out[(((size_t)f * P + p) * Q + q) * Nb + n] = (float)acc;
                }
    return ORC_OK;
}

/* stitch_to_blockwise, src/formats.cpp:221-250 (kPadColumn = 0xffffffff,
 * include/shflbw/formats.hpp:109) */
int orc_stitch_to_blockwise(uint32_t V, uint32_t G, const uint32_t* group_ncols,
                            const uint32_t* cols, const float* values,
                            uint32_t tile_width, uint32_t* tile_cols,
                            float* tile_vals, uint32_t* tile_group) {
    if (tile_width == 0) return -ORC_BAD_PARAMS;
    int ntiles = 0;
    size_t off = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = group_ncols[g];
        for (uint32_t begin = 0; begin < ng; begin += tile_width) {
            const uint32_t avail = ng - begin < tile_width ? ng - begin : tile_width;
            uint32_t* tc = tile_cols + (size_t)ntiles * tile_width;
            float* tv = tile_vals + (size_t)ntiles * tile_width * V;
            for (uint32_t j = 0; j < tile_width; ++j) tc[j] = 0xffffffffu;
            memset(tv, 0, sizeof(float) * (size_t)tile_width * V);
            for (uint32_t j = 0; j < avail; ++j) {
                tc[j] = cols[off + begin + j];
                for (uint32_t i = 0; i < V; ++i) tv[(size_t)j * V + i] = values[(off + begin + j) * V + i];
            }
            tile_group[ntiles++] = g;
        }
        off += ng;
    }
    return ntiles;
}

/* ------------------------------------------------------------------------ */
/* 16-bit conversions (round to nearest even)                               */
/* ------------------------------------------------------------------------ */

uint16_t orc_f32_to_bf16(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu))
        return (uint16_t)((u >> 16) | 0x0040u); /* quiet NaN */
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

float orc_bf16_to_f32(uint16_t h) {
    const uint32_t u = (uint32_t)h << 16;
    float x;
    memcpy(&x, &u, 4);
    return x;
}

uint16_t orc_f32_to_f16(float x) {
    const _Float16 h = (_Float16)x;
    uint16_t u;
    memcpy(&u, &h, 2);
    return u;
}

float orc_f16_to_f32(uint16_t u) {
    _Float16 h;
    memcpy(&h, &u, 2);
    return (float)h;
}

void orc_round16(float* x, size_t n, int dtype) {
    for (size_t i = 0; i < n; ++i)
        x[i] = dtype == 2 ? orc_f16_to_f32(orc_f32_to_f16(x[i])) : orc_bf16_to_f32(orc_f32_to_bf16(x[i]));
}

/* Device packed layout: stitch_to_blockwise's padding rule (zero values,
 * kPadColumn indices) applied with tile_width = k_tile, concatenated. */
int64_t orc_pack_device(uint32_t M, uint32_t V, const uint32_t* group_ncols,
                        const uint32_t* cols, const float* values, uint32_t k_tile,
                        int dtype, int32_t* group_ptr, int32_t* col_idx,
                        uint16_t* vals16) {
    const uint32_t G = V ? M / V : 0;
    int64_t out = 0;
    size_t off = 0;
    group_ptr[0] = 0;
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = group_ncols[g];
        const uint32_t padded = (ng + k_tile - 1) / k_tile * k_tile;
        for (uint32_t j = 0; j < padded; ++j) {
            col_idx[out + j] = j < ng ? (int32_t)cols[off + j] : -1;
            for (uint32_t i = 0; i < V; ++i) {
                const float x = j < ng ? values[(off + j) * V + i] : 0.0f;
                vals16[(out + j) * V + i] = dtype == 2 ? orc_f32_to_f16(x) : orc_f32_to_bf16(x);
            }
        }
        out += padded;
        off += ng;
        group_ptr[g + 1] = (int32_t)out;
    }
    return out;
}
