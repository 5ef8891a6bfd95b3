// internal.h -- entry points shared between the translation units of
// libshflbw_b200.so (not part of the public ABI; see include/shflbw_cu.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "shflbw_cu.h"

namespace sbw {

// convert.cu
int validate_impl(const uint8_t* mask, int M, int K, int V, int32_t* pass, uint32_t* fail_row,
                  cudaStream_t s);
int compress_impl(const void* dense, int dense_dtype, const uint8_t* mask, int M, int K, int V,
                  int value_dtype, shflbw_cu_matrix* out, uint32_t* fail_row, cudaStream_t s);
int compress_async_impl(const void* dense, int dense_dtype, const uint8_t* mask, int M, int K, int V,
                        int value_dtype, shflbw_cu_matrix* out, int32_t* status, cudaStream_t s);
int finalize_impl(shflbw_cu_matrix* m, const int32_t* status, uint32_t* fail_row, cudaStream_t s);
int upload_impl(int M, int K, int V, const uint32_t* row_indices, const uint32_t* group_ncols,
                const uint32_t* cols, const float* values, int value_dtype, shflbw_cu_matrix* out,
                cudaStream_t s);
int download_impl(const shflbw_cu_matrix* m, uint32_t* row_indices, uint32_t* group_ncols,
                  uint32_t* cols, float* values, cudaStream_t s);
int decompress_impl(const shflbw_cu_matrix* m, float* dense, cudaStream_t s);
int conv_prepare_impl(const shflbw_cu_matrix* w, int S, shflbw_cu_matrix* out, cudaStream_t s);
int convert_impl(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t s);
int convert_2d_impl(const void* src, int sdt, int64_t ld_src, void* dst, int ddt, int64_t ld_dst, int64_t rows,
                    int64_t cols, cudaStream_t s);
int scan_exclusive(const int* in, int* out, int n, int* total_dev, cudaStream_t s);
// keep the default stream-ordered pool's memory across synchronisations (convert.cu)
void retain_pool();
int radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* keys_tmp, uint32_t* vals_tmp, int n,
                     cudaStream_t s);
void free_matrix(shflbw_cu_matrix* m);

// Where the "B" operand rows come from.
//   kind 0 (SpMM): row c of B, element n at B[c * ldb + n]
//   kind 1 (conv): implicit im2col of a [C][H][W][Nb] tensor; sparse column
//                  c = (ch, r, s), flat output column n = (p*Q + q)*Nb + nb
//   kind 2 (conv, 128-byte rows): as kind 1 for a matrix in conv order
//                  (shflbw_cu_conv_prepare), stride 1, Nb in {16, 32} and
//                  64/Nb | Q: each activation row fetched is 64/Nb adjacent
//                  output positions x Nb from the [C*H][W*Nb] view
struct Operand {
    int kind = 0;
    const void* ptr = nullptr;
    int64_t ldb = 0;  // kind 0
    int K = 0;        // rows of B / C*R*S
    int N = 0;        // flat output columns
    // kind 1 geometry
    int C = 0, H = 0, W = 0, Nb = 0, R = 1, S = 1, stride = 1, pad = 0, P = 0, Q = 0;
};

constexpr int kMaxPeers = 8;  // output destinations (the fused all-gather)

struct OutSpec {
    void* ptr = nullptr;
    int dtype = SHFLBW_F32;
    int64_t ldc = 0;
    int compact = 0;  // 1: row (g - g_begin)*V + r instead of row_indices
    // further destinations that receive identical row stores (peer GPUs' C
    // through P2P mappings: the all-gather fused into the epilogue)
    void* extra[kMaxPeers - 1] = {};
    int n_extra = 0;
    // 1: ptr is an NVLS multicast address -- every row store is one
    // multimem.st that lands in all bound GPUs' outputs
    int multicast = 0;
};

// spmm_simt.cu: CUDA-core kernel, any V, bit-exact ascending-k order
int spmm_simt(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b,
              const OutSpec& c, cudaStream_t s);
// spmm_sm100.cu: tcgen05 kernel; returns SHFLBW_UNSUPPORTED if the case is
// outside its envelope (caller then uses spmm_simt)
int spmm_tc(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
            cudaStream_t s);
int unpermute_impl(const int32_t* row_indices, int M, int N, const void* C_perm, int64_t ld_perm,
                   void* C, int64_t ldc, int dtype, cudaStream_t s);

}  // namespace sbw
