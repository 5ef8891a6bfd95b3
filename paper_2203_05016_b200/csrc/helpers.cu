// helpers.cu -- device versions of the reference's public helper routines
// (not on the timed path, but part of the API surface a drop-in must offer):
//   spmm_dense_oracle  src/spmm.cpp:148-161
//   stitch_tile        src/spmm.cpp:37-58
//   tile_mma           src/spmm.cpp:60-74
// All three keep the reference's fp32 arithmetic exactly: every product is
// rounded, then added (__fmul_rn / __fadd_rn never contract to FMA), k
// ascending -- so their results are bit-identical to the reference's.
#include "common.cuh"
#include "internal.h"

namespace sbw {
namespace {

__global__ void k_dense_matmul(const float* __restrict__ A, int M, int K, const float* __restrict__ B,
                               int N, float* __restrict__ C) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= N) return;
    float acc = 0.0f;
    const float* a = A + static_cast<int64_t>(i) * K;
    for (int k = 0; k < K; ++k) acc = __fadd_rn(acc, __fmul_rn(a[k], B[static_cast<int64_t>(k) * N + j]));
    C[static_cast<int64_t>(i) * N + j] = acc;
}

__global__ void k_stitch_tile(const uint32_t* __restrict__ cols, int64_t k_len, int64_t chunk_begin,
                              const float* __restrict__ B, int B_rows, int B_cols, int64_t slice_begin,
                              int64_t n_len, int64_t t_n, int64_t t_k, float* __restrict__ out,
                              uint32_t* __restrict__ flag) {
    const int64_t total = t_k * t_n;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = idx / t_n, j = idx % t_n;
        float x = 0.0f;
        if (t < k_len) {
            const uint32_t row = cols[chunk_begin + t];
            if (row >= static_cast<uint32_t>(B_rows)) {
                atomicOr(flag, 1u);
            } else if (j < n_len) {
                x = B[static_cast<int64_t>(row) * B_cols + slice_begin + j];
            }
        }
        out[idx] = x;
    }
}

__global__ void k_tile_mma(float* __restrict__ acc, const float* __restrict__ a_tile,
                           const float* __restrict__ b_tile, int64_t v_rows, int64_t k_len, int64_t t_n) {
    const int64_t total = v_rows * t_n;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t vi = idx / t_n, j = idx % t_n;
        float x = acc[idx];
        for (int64_t t = 0; t < k_len; ++t) x = __fadd_rn(x, __fmul_rn(a_tile[t * v_rows + vi], b_tile[t * t_n + j]));
        acc[idx] = x;
    }
}

// permutation folding (shflbw_cu_fold_input_permutation)
__global__ void k_invert_perm(const int32_t* __restrict__ perm, int n, int32_t* __restrict__ inv,
                              uint32_t* __restrict__ flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int32_t p = perm[i];
        if (p < 0 || p >= n) atomicOr(flag, 1u);
        else if (atomicExch(&inv[p], i) != -1) atomicOr(flag, 2u);  // duplicate entry
    }
}

__global__ void k_fold_cols(int32_t* __restrict__ col_idx, int64_t total, const int32_t* __restrict__ inv) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < total;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t c = col_idx[j];
        if (c >= 0) col_idx[j] = inv[c];  // pad entries (-1) stay pads
    }
}

int blocks_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return static_cast<int>(b < 1 ? 1 : (b > 65536 ? 65536 : b));
}

}  // namespace
}  // namespace sbw

using namespace sbw;

extern "C" {

int shflbw_cu_dense_matmul_f32(const float* A, int32_t M, int32_t K, const float* B, int32_t N, float* C,
                               shflbw_stream_t stream) {
    if (M < 0 || K < 0 || N < 0) return fail(SHFLBW_BAD_PARAMS, "negative extent");
    if (M == 0 || N == 0) return SHFLBW_OK;
    if (M > 65535) return fail(SHFLBW_UNSUPPORTED, "dense oracle: M > 65535");
    dim3 grid((N + 127) / 128, M);
    k_dense_matmul<<<grid, 128, 0, reinterpret_cast<cudaStream_t>(stream)>>>(A, M, K, B, N, C);
    SBW_LAUNCHED("k_dense_matmul");
    return SHFLBW_OK;
}

int shflbw_cu_stitch_tile(const uint32_t* group_cols, int64_t ncols, int64_t chunk_begin, int64_t t_k,
                          const float* B, int32_t B_rows, int32_t B_cols, int64_t slice_begin, int64_t t_n,
                          float* staging, shflbw_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (t_k < 0 || t_n < 0 || chunk_begin < 0 || slice_begin < 0) return fail(SHFLBW_BAD_PARAMS, "negative extent");
    const int64_t k_len = chunk_begin < ncols ? (t_k < ncols - chunk_begin ? t_k : ncols - chunk_begin) : 0;
    const int64_t n_len = slice_begin < B_cols ? (t_n < B_cols - slice_begin ? t_n : B_cols - slice_begin) : 0;
    if (t_k * t_n == 0) return SHFLBW_OK;
    uint32_t* flag = nullptr;
    SBW_CUDA(cudaMallocAsync(&flag, sizeof(uint32_t), s));
    SBW_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), s));
    k_stitch_tile<<<blocks_for(t_k * t_n), 256, 0, s>>>(group_cols, k_len, chunk_begin, B, B_rows, B_cols,
                                                        slice_begin, n_len, t_n, t_k, staging, flag);
    SBW_LAUNCHED("k_stitch_tile");
    uint32_t h = 0;
    SBW_CUDA(cudaMemcpyAsync(&h, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaFreeAsync(flag, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    if (h) return fail(SHFLBW_SHAPE_MISMATCH, "stitch_tile: column index exceeds B rows");
    return SHFLBW_OK;
}

int shflbw_cu_tile_mma(float* acc, const float* a_tile, const float* b_tile, int64_t v_rows, int64_t k_len,
                       int64_t t_n, shflbw_stream_t stream) {
    if (v_rows < 0 || k_len < 0 || t_n < 0) return fail(SHFLBW_BAD_PARAMS, "negative extent");
    if (v_rows * t_n == 0) return SHFLBW_OK;
    k_tile_mma<<<blocks_for(v_rows * t_n), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(acc, a_tile, b_tile,
                                                                                            v_rows, k_len, t_n);
    SBW_LAUNCHED("k_tile_mma");
    return SHFLBW_OK;
}

}  // extern "C"

int shflbw_cu_fold_input_permutation(shflbw_cu_matrix* a, const int32_t* producer_rows, shflbw_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!a || !a->group_ptr || a->cols < 0) return fail(SHFLBW_BAD_PARAMS, "fold: invalid matrix");
    if (a->reserved & SHFLBW_FOLDED) return fail(SHFLBW_BAD_PARAMS, "fold: input permutation already folded");
    const int n = a->cols;
    if (n > 0 && !producer_rows) return fail(SHFLBW_BAD_PARAMS, "fold: producer_rows is null");
    if (n > 0) {
        int32_t* inv = nullptr;
        uint32_t* flag = nullptr;
        SBW_CUDA(cudaMallocAsync(&inv, static_cast<size_t>(n) * sizeof(int32_t), s));
        SBW_CUDA(cudaMallocAsync(&flag, sizeof(uint32_t), s));
        SBW_CUDA(cudaMemsetAsync(inv, 0xff, static_cast<size_t>(n) * sizeof(int32_t), s));
        SBW_CUDA(cudaMemsetAsync(flag, 0, sizeof(uint32_t), s));
        k_invert_perm<<<blocks_for(n), 256, 0, s>>>(producer_rows, n, inv, flag);
        SBW_LAUNCHED("k_invert_perm");
        uint32_t h = 0;
        SBW_CUDA(cudaMemcpyAsync(&h, flag, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SBW_CUDA(cudaStreamSynchronize(s));
        if (!h && a->total_cols > 0) {
            k_fold_cols<<<blocks_for(a->total_cols), 256, 0, s>>>(a->col_idx, a->total_cols, inv);
            SBW_LAUNCHED("k_fold_cols");
        }
        SBW_CUDA(cudaFreeAsync(inv, s));
        SBW_CUDA(cudaFreeAsync(flag, s));
        SBW_CUDA(cudaStreamSynchronize(s));
        if (h) return fail(SHFLBW_BAD_PARAMS, "fold: producer_rows is not a permutation of 0..cols-1");
    }
    a->reserved = (a->reserved | SHFLBW_FOLDED) & ~SHFLBW_CONTIG_BLOCKS;
    return SHFLBW_OK;
}
