// capi.cu -- the extern "C" boundary (include/shflbw_cu.h): argument checks
// with the reference's error semantics, kernel dispatch, status plumbing.
#include <atomic>
#include <cstring>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace sbw {

namespace {
thread_local std::string g_error;
thread_local std::string g_plan;
thread_local int64_t g_launches = 0;
std::atomic<int64_t> g_force_simt{0}, g_split{0}, g_stages{0}, g_pdl{1}, g_cps{0}, g_trace{0}, g_nobulk{0}, g_split_mode{0}, g_persist{0}, g_gw{0}, g_strict{0}, g_raster{0}, g_tile_n{0}, g_issue{0}, g_tiles{0}, g_conv_legacy{0}, g_prefetch{0}, g_trigger{0};
}  // namespace

void set_error(const std::string& msg) { g_error = msg; }
void set_plan(const std::string& plan) { g_plan = plan; }
int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return SHFLBW_CUDA_ERROR;
}
void count_launch(int n) { g_launches += n; }

int64_t option(const char* key) {
    if (!std::strcmp(key, "force_simt")) return g_force_simt.load();
    if (!std::strcmp(key, "split")) return g_split.load();
    if (!std::strcmp(key, "stages")) return g_stages.load();
    if (!std::strcmp(key, "pdl")) return g_pdl.load();
    if (!std::strcmp(key, "cp_async_slabs")) return g_cps.load();
    if (!std::strcmp(key, "trace")) return g_trace.load();
    if (!std::strcmp(key, "no_bulk_out")) return g_nobulk.load();
    if (!std::strcmp(key, "split_mode")) return g_split_mode.load();
    if (!std::strcmp(key, "persistent")) return g_persist.load();
    if (!std::strcmp(key, "gather_warps")) return g_gw.load();
    if (!std::strcmp(key, "strict")) return g_strict.load();
    if (!std::strcmp(key, "raster")) return g_raster.load();
    if (!std::strcmp(key, "tile_n")) return g_tile_n.load();
    if (!std::strcmp(key, "gather_issue")) return g_issue.load();
    if (!std::strcmp(key, "tile_loads")) return g_tiles.load();
    if (!std::strcmp(key, "converter_legacy")) return g_conv_legacy.load();
    if (!std::strcmp(key, "prefetch")) return g_prefetch.load();
    if (!std::strcmp(key, "pdl_trigger")) return g_trigger.load();
    return 0;
}

namespace {

int check_matrix(const shflbw_cu_matrix* a) {
    if (!a || !a->row_indices || !a->group_ptr || !a->group_ncols)
        return fail(SHFLBW_BAD_PARAMS, "null shflbw_cu_matrix");
    if (a->v <= 0 || a->rows % a->v != 0 || a->groups != a->rows / a->v)
        return fail(SHFLBW_BAD_PARAMS, "inconsistent shflbw_cu_matrix (V, M, G)");
    if (a->dtype != SHFLBW_BF16 && a->dtype != SHFLBW_F16 && a->dtype != SHFLBW_F32)
        return fail(SHFLBW_BAD_PARAMS, "matrix dtype must be BF16, F16 or F32");
    return SHFLBW_OK;
}

int check_compute_matrix(const shflbw_cu_matrix* a) { return check_matrix(a); }

int check_out_dtype(int dt) {
    if (dt != SHFLBW_F32 && dt != SHFLBW_BF16 && dt != SHFLBW_F16)
        return fail(SHFLBW_BAD_PARAMS, "output dtype must be F32, BF16 or F16");
    return SHFLBW_OK;
}

int run_spmm(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
             cudaStream_t s) {
    if (g_end <= g_begin || b.N == 0) return SHFLBW_OK;
    if (!option("force_simt") && a->dtype != SHFLBW_F32) {  // fp32: the exact CUDA-core path
        const int st = spmm_tc(a, g_begin, g_end, b, c, s);
        // strict: a 16-bit matrix outside the tcgen05 envelope is an error
        // (the message names the reason), not a silent CUDA-core fallback
        if (st != SHFLBW_UNSUPPORTED || option("strict")) return st;
    }
    if (c.n_extra > 0 || c.multicast)
        return fail(SHFLBW_UNSUPPORTED, "spmm with peer / multicast destinations: needs the tcgen05 path (bf16/f16 "
                                        "matrix, V in {16, 32, 64, 128}, 16-byte aligned rows)");
    return spmm_simt(a, g_begin, g_end, b, c, s);
}

int spmm_groups_impl(const shflbw_cu_matrix* a, int g_begin, int g_end, const void* B, int K_b, int N,
                     int64_t ldb, void* C, int c_dtype, int64_t ldc, int compact, cudaStream_t s,
                     void* const* extra = nullptr, int n_extra = 0, int multicast = 0) {
    if (int st = check_compute_matrix(a)) return st;
    if (int st = check_out_dtype(c_dtype)) return st;
    if (K_b != a->cols) return fail(SHFLBW_SHAPE_MISMATCH, "spmm: A columns != B rows");
    if (N < 0 || ldb < N || ldc < N) return fail(SHFLBW_BAD_PARAMS, "spmm: bad N / leading dimensions");
    if (g_begin < 0 || g_end > a->groups || g_begin > g_end)
        return fail(SHFLBW_BAD_PARAMS, "spmm: group range outside [0, G]");
    if ((N > 0 && (a->rows > 0) && (!B || !C))) return fail(SHFLBW_BAD_PARAMS, "spmm: null B or C");
    Operand b;
    b.kind = 0;
    b.ptr = B;
    b.ldb = ldb;
    b.K = K_b;
    b.N = N;
    OutSpec c;
    c.ptr = C;
    c.dtype = c_dtype;
    c.ldc = ldc;
    c.compact = compact;
    if (n_extra < 0 || n_extra > kMaxPeers - 1) return fail(SHFLBW_BAD_PARAMS, "spmm: 0..7 peer destinations");
    for (int d = 0; d < n_extra; ++d) {
        if (!extra[d]) return fail(SHFLBW_BAD_PARAMS, "spmm: null peer destination");
        c.extra[d] = extra[d];
    }
    c.n_extra = n_extra;
    c.multicast = multicast;
    return run_spmm(a, g_begin, g_end, b, c, s);
}

}  // namespace
}  // namespace sbw

using namespace sbw;

extern "C" {

const char* shflbw_cu_last_error(void) { return g_error.c_str(); }

int shflbw_cu_version(void) { return 10000; }

int shflbw_cu_set_option(const char* key, int64_t value) {
    if (!key) return fail(SHFLBW_BAD_PARAMS, "null option key");
    if (!std::strcmp(key, "force_simt")) g_force_simt = value;
    else if (!std::strcmp(key, "split")) g_split = value;
    else if (!std::strcmp(key, "stages")) {
        // the epilogue stages its output tile in >= 2 pipeline slots
        if (value != 0 && (value < 2 || value > 32)) return fail(SHFLBW_BAD_PARAMS, "stages must be 0 (auto) or 2..32");
        g_stages = value;
    }
    else if (!std::strcmp(key, "pdl")) g_pdl = value;
    else if (!std::strcmp(key, "cp_async_slabs")) g_cps = value;
    else if (!std::strcmp(key, "trace")) g_trace = value;
    else if (!std::strcmp(key, "no_bulk_out")) g_nobulk = value;
    else if (!std::strcmp(key, "split_mode")) g_split_mode = value;
    else if (!std::strcmp(key, "persistent")) g_persist = value;
    else if (!std::strcmp(key, "gather_warps")) g_gw = value;
    else if (!std::strcmp(key, "strict")) g_strict = value;
    else if (!std::strcmp(key, "raster")) g_raster = value;
    else if (!std::strcmp(key, "tile_n")) g_tile_n = value;
    else if (!std::strcmp(key, "gather_issue")) g_issue = value;
    else if (!std::strcmp(key, "tile_loads")) g_tiles = value;
    else if (!std::strcmp(key, "converter_legacy")) g_conv_legacy = value;
    else if (!std::strcmp(key, "prefetch")) g_prefetch = value;
    else if (!std::strcmp(key, "pdl_trigger")) g_trigger = value;
    else return fail(SHFLBW_BAD_PARAMS, std::string("unknown option ") + key);
    return SHFLBW_OK;
}

int64_t shflbw_cu_launch_count(void) { return g_launches; }

const char* shflbw_cu_last_plan(void) { return g_plan.c_str(); }

int shflbw_cu_validate(const uint8_t* mask, int32_t M, int32_t K, int32_t V, int32_t* pass,
                       uint32_t* fail_row, shflbw_stream_t stream) {
    if (!pass || !fail_row) return fail(SHFLBW_BAD_PARAMS, "null output pointer");
    return validate_impl(mask, M, K, V, pass, fail_row, reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_compress(const void* dense, int32_t dense_dtype, const uint8_t* mask, int32_t M, int32_t K,
                       int32_t V, int32_t value_dtype, shflbw_cu_matrix* out, uint32_t* fail_row,
                       shflbw_stream_t stream) {
    if (!out) return fail(SHFLBW_BAD_PARAMS, "null output matrix");
    return compress_impl(dense, dense_dtype, mask, M, K, V, value_dtype, out, fail_row,
                         reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_compress_async(const void* dense, int32_t dense_dtype, const uint8_t* mask, int32_t M, int32_t K,
                             int32_t V, int32_t value_dtype, shflbw_cu_matrix* out, int32_t* status,
                             shflbw_stream_t stream) {
    if (!out || !status) return fail(SHFLBW_BAD_PARAMS, "null output matrix or status");
    return compress_async_impl(dense, dense_dtype, mask, M, K, V, value_dtype, out, status,
                               reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_matrix_finalize(shflbw_cu_matrix* m, const int32_t* status, uint32_t* fail_row,
                              shflbw_stream_t stream) {
    if (!m || !status) return fail(SHFLBW_BAD_PARAMS, "null matrix or status");
    return finalize_impl(m, status, fail_row, reinterpret_cast<cudaStream_t>(stream));
}

void shflbw_cu_matrix_free(shflbw_cu_matrix* m) { free_matrix(m); }

int shflbw_cu_matrix_upload(int32_t M, int32_t K, int32_t V, const uint32_t* row_indices,
                            const uint32_t* group_ncols, const uint32_t* cols, const float* values,
                            int32_t value_dtype, shflbw_cu_matrix* out, shflbw_stream_t stream) {
    if (!out) return fail(SHFLBW_BAD_PARAMS, "null output matrix");
    return upload_impl(M, K, V, row_indices, group_ncols, cols, values, value_dtype, out,
                       reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_matrix_download(const shflbw_cu_matrix* m, uint32_t* row_indices, uint32_t* group_ncols,
                              uint32_t* cols, float* values, shflbw_stream_t stream) {
    if (int st = check_matrix(m)) return st;
    if (m->reserved & SHFLBW_FOLDED) return fail(SHFLBW_BAD_PARAMS, "matrix has a folded input permutation");
    if (m->reserved & SHFLBW_CONV_ORDER)
        return fail(SHFLBW_BAD_PARAMS, "matrix is in conv order (shflbw_cu_conv_prepare); download the original");
    return download_impl(m, row_indices, group_ncols, cols, values, reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_matrix_export_raw(const shflbw_cu_matrix* m, int32_t* group_ptr, int32_t* col_idx,
                                void* values, shflbw_stream_t stream) {
    if (int st = check_matrix(m)) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SBW_CUDA(cudaMemcpyAsync(group_ptr, m->group_ptr, sizeof(int32_t) * (m->groups + 1), cudaMemcpyDeviceToHost, s));
    if (m->total_cols > 0) {
        SBW_CUDA(cudaMemcpyAsync(col_idx, m->col_idx, sizeof(int32_t) * m->total_cols, cudaMemcpyDeviceToHost, s));
        SBW_CUDA(cudaMemcpyAsync(values, m->values, static_cast<size_t>(dtype_bytes(m->dtype)) * m->total_cols * m->v,
                                 cudaMemcpyDeviceToHost, s));
    }
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int shflbw_cu_decompress(const shflbw_cu_matrix* m, float* dense, shflbw_stream_t stream) {
    if (int st = check_matrix(m)) return st;
    return decompress_impl(m, dense, reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_spmm(const shflbw_cu_matrix* a, const void* B, int32_t K_b, int32_t N, int64_t ldb, void* C,
                   int32_t c_dtype, int64_t ldc, shflbw_stream_t stream) {
    if (int st = check_matrix(a)) return st;
    return spmm_groups_impl(a, 0, a->groups, B, K_b, N, ldb, C, c_dtype, ldc, 0,
                            reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_spmm_groups(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end, const void* B,
                          int32_t K_b, int32_t N, int64_t ldb, void* C, int32_t c_dtype, int64_t ldc,
                          int32_t compact, shflbw_stream_t stream) {
    return spmm_groups_impl(a, g_begin, g_end, B, K_b, N, ldb, C, c_dtype, ldc, compact,
                            reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_spmm_groups_peers(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end, const void* B,
                                int32_t K_b, int32_t N, int64_t ldb, void* const* C_dst, int32_t n_dst,
                                int32_t c_dtype, int64_t ldc, shflbw_stream_t stream) {
    if (!C_dst || n_dst < 1 || n_dst > kMaxPeers) return fail(SHFLBW_BAD_PARAMS, "spmm_groups_peers: 1..8 destinations");
    if (c_dtype == SHFLBW_F32) return fail(SHFLBW_UNSUPPORTED, "spmm_groups_peers: 16-bit output only");
    return spmm_groups_impl(a, g_begin, g_end, B, K_b, N, ldb, C_dst[0], c_dtype, ldc, 0,
                            reinterpret_cast<cudaStream_t>(stream), C_dst + 1, n_dst - 1);
}

int shflbw_cu_spmm_groups_multicast(const shflbw_cu_matrix* a, int32_t g_begin, int32_t g_end, const void* B,
                                    int32_t K_b, int32_t N, int64_t ldb, void* C_mc, int32_t c_dtype, int64_t ldc,
                                    shflbw_stream_t stream) {
    if (c_dtype == SHFLBW_F32) return fail(SHFLBW_UNSUPPORTED, "spmm_groups_multicast: 16-bit output only");
    if (!C_mc || (reinterpret_cast<uintptr_t>(C_mc) & 15)) return fail(SHFLBW_BAD_PARAMS, "spmm_groups_multicast: null or unaligned address");
    return spmm_groups_impl(a, g_begin, g_end, B, K_b, N, ldb, C_mc, c_dtype, ldc, 0,
                            reinterpret_cast<cudaStream_t>(stream), nullptr, 0, 1);
}

int shflbw_cu_unpermute_rows(const int32_t* row_indices, int32_t M, int32_t N, const void* C_perm,
                             int64_t ld_perm, void* C, int64_t ldc, int32_t dtype, shflbw_stream_t stream) {
    if (int st = check_out_dtype(dtype)) return st;
    return unpermute_impl(row_indices, M, N, C_perm, ld_perm, C, ldc, dtype,
                          reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_conv_output_size(int32_t H, int32_t W, int32_t R, int32_t S, int32_t stride, int32_t pad,
                               int32_t* P, int32_t* Q) {
    // conv_output_size, src/spmm.cpp:177-191
    if (R <= 0 || S <= 0 || stride <= 0 || H < 0 || W < 0 || pad < 0)
        return fail(SHFLBW_BAD_GEOMETRY, "filter sizes and stride must be positive");
    const int64_t sh = static_cast<int64_t>(H) + 2 * static_cast<int64_t>(pad) - R;
    const int64_t sw = static_cast<int64_t>(W) + 2 * static_cast<int64_t>(pad) - S;
    if (sh < 0 || sw < 0 || sh % stride != 0 || sw % stride != 0)
        return fail(SHFLBW_BAD_GEOMETRY,
                    "input size, padding, filter and stride do not produce a whole output grid");
    if (P) *P = static_cast<int32_t>(sh / stride + 1);
    if (Q) *Q = static_cast<int32_t>(sw / stride + 1);
    return SHFLBW_OK;
}

int shflbw_cu_conv2d(const shflbw_cu_matrix* w, const void* input, int32_t C, int32_t H, int32_t W,
                     int32_t Nb, int32_t R, int32_t S, int32_t stride, int32_t pad, void* out,
                     int32_t out_dtype, shflbw_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (int st = check_compute_matrix(w)) return st;
    if (int st = check_out_dtype(out_dtype)) return st;
    if (w->reserved & SHFLBW_FOLDED) return fail(SHFLBW_BAD_PARAMS, "conv2d: matrix has a folded input permutation");
    int32_t P = 0, Q = 0;
    if (int st = shflbw_cu_conv_output_size(H, W, R, S, stride, pad, &P, &Q)) return st;
    if (static_cast<int64_t>(w->cols) != static_cast<int64_t>(C) * R * S)
        return fail(SHFLBW_BAD_GEOMETRY, "weight columns != C*R*S");
    if (Nb < 0 || C < 0) return fail(SHFLBW_BAD_GEOMETRY, "negative tensor extent");
    const int64_t flat = static_cast<int64_t>(P) * Q * Nb;
    if (flat > 0x7fffffff) return fail(SHFLBW_UNSUPPORTED, "conv: P*Q*N exceeds 2^31");
    if (flat == 0 || w->rows == 0) return SHFLBW_OK;
    if (R == 1 && S == 1 && stride == 1 && pad == 0) {
        // 1x1 conv is exactly the SpMM on the [C][H*W*N] view (the reference's
        // own identity, tests/test_conv.cpp:88-99), same kernel, same bits
        return spmm_groups_impl(w, 0, w->groups, input, C, static_cast<int>(flat), flat, out, out_dtype, flat,
                                0, s);
    }
    Operand b;
    // 128-byte activation rows when the weight is in conv order for this S
    const int ppb = Nb > 0 ? 64 / Nb : 0;  // output positions per 64-element row
    // (an output width Q that is not a multiple of ppb runs on a padded
    // position grid, spmm_sm100.cu)
    const bool wide = (w->reserved & SHFLBW_CONV_ORDER) && SHFLBW_CONV_ORDER_S(w->reserved) == S && stride == 1 &&
                      (Nb == 16 || Nb == 32) && ppb > 0 && (static_cast<int64_t>(C) * H < (1LL << 31));
    b.kind = wide ? 2 : 1;
    b.ptr = input;
    b.K = w->cols;
    b.N = static_cast<int>(flat);
    b.C = C;
    b.H = H;
    b.W = W;
    b.Nb = Nb;
    b.R = R;
    b.S = S;
    b.stride = stride;
    b.pad = pad;
    b.P = P;
    b.Q = Q;
    OutSpec c;
    c.ptr = out;
    c.dtype = out_dtype;
    c.ldc = flat;
    c.compact = 0;
    return run_spmm(w, 0, w->groups, b, c, s);
}

int shflbw_cu_conv_prepare(const shflbw_cu_matrix* w, int32_t S, shflbw_cu_matrix* out, shflbw_stream_t stream) {
    if (int st = check_matrix(w)) return st;
    if (!out) return fail(SHFLBW_BAD_PARAMS, "conv_prepare: out is null");
    if (S < 1 || w->cols % S != 0) return fail(SHFLBW_BAD_GEOMETRY, "conv_prepare: S must divide the weight columns");
    return conv_prepare_impl(w, S, out, reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n,
                      shflbw_stream_t stream) {
    if (check_out_dtype(src_dtype) || check_out_dtype(dst_dtype)) return SHFLBW_BAD_PARAMS;
    return convert_impl(src, src_dtype, dst, dst_dtype, n, reinterpret_cast<cudaStream_t>(stream));
}

int shflbw_cu_convert_2d(const void* src, int32_t src_dtype, int64_t ld_src, void* dst, int32_t dst_dtype,
                         int64_t ld_dst, int64_t rows, int64_t cols, shflbw_stream_t stream) {
    if (check_out_dtype(src_dtype) || check_out_dtype(dst_dtype)) return SHFLBW_BAD_PARAMS;
    if (rows < 0 || cols < 0 || ld_src < cols || ld_dst < cols)
        return fail(SHFLBW_BAD_PARAMS, "convert_2d: bad extents / leading dimensions");
    return convert_2d_impl(src, src_dtype, ld_src, dst, dst_dtype, ld_dst, rows, cols,
                           reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
