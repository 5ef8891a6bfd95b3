// spmm_simt.cu -- CUDA-core Shfl-BW SpMM / implicit-GEMM conv for any V.
//
// Serves the V values the tcgen05 kernel does not take (the reference tests
// use V in 1..16, tests/test_spmm.cpp:118, tests/acceptance.cpp:66) and any
// shape outside its envelope.  It keeps the reference's pinned reduction
// order exactly: every output element is a chain of fmaf in ascending k from
// 0.0f, which for 16-bit operands equals the reference's separately rounded
// multiply-add (src/spmm.cpp:60-74) because each product is exact in fp32.
// Products are rounded and then added (__fmul_rn / __fadd_rn, never a fused
// FMA -- the reference builds with -ffp-contract=off), so this path is
// BIT-IDENTICAL to spmm_execute / conv2d for fp32 operands (SHFLBW_F32
// matrices, the C++ drop-in's default) as well as for bf16/fp16 ones.
//
// Block = one group x 128 output columns; thread = one output column.  The
// group's weights and column indices are staged through shared memory in
// chunks of 64 columns; the write-back goes through row_indices
// (src/spmm.cpp:115-123) or, for sharded runs, to compact group order.
#include "common.cuh"
#include "internal.h"

namespace sbw {
namespace {

constexpr int kThreads = 128;
constexpr int kJ = 64;   // columns staged per chunk
constexpr int kVC = 16;  // group rows accumulated per pass

template <int DT, int KIND>
__global__ void __launch_bounds__(kThreads) k_spmm_simt(
    const int32_t* __restrict__ row_indices, const int32_t* __restrict__ group_ptr,
    const int32_t* __restrict__ group_ncols, const int32_t* __restrict__ col_idx,
    const void* __restrict__ values, int V, int g_begin, Operand b, OutSpec c) {
    using T = typename Elem<DT>::T;
    __shared__ float w_s[kJ][kVC];
    __shared__ int64_t base_s[kJ];  // KIND 0: row offset; KIND 1: channel plane offset
    __shared__ int dr_s[kJ], ds_s[kJ];

    const int g = g_begin + blockIdx.y;
    const int n = blockIdx.x * kThreads + threadIdx.x;
    const bool live = n < b.N;
    // the padded width: pad columns (-1) are skipped wherever they sit (at the
    // end in the reference order, inside the group in conv order), so the sum
    // keeps the layout's column order exactly
    const int gp = group_ptr[g], ng = group_ptr[g + 1] - gp;
    (void)group_ncols;
    const T* vals = static_cast<const T*>(values) + static_cast<int64_t>(gp) * V;
    const T* B = static_cast<const T*>(b.ptr);

    // conv: decode this thread's output position once
    int p0 = 0, q0 = 0, nb = 0;
    if (KIND == 1 && live) {
        nb = n % b.Nb;
        const int pq = n / b.Nb;
        q0 = (pq % b.Q) * b.stride;
        p0 = (pq / b.Q) * b.stride;
    }

    for (int vc = 0; vc < V; vc += kVC) {
        const int nv = min(kVC, V - vc);
        float acc[kVC];
#pragma unroll
        for (int u = 0; u < kVC; ++u) acc[u] = 0.0f;
        for (int j0 = 0; j0 < ng; j0 += kJ) {
            const int nj = min(kJ, ng - j0);
            __syncthreads();
            for (int idx = threadIdx.x; idx < kJ * kVC; idx += kThreads) {
                const int jj = idx / kVC, u = idx % kVC;
                w_s[jj][u] = (jj < nj && u < nv)
                                 ? Elem<DT>::to_f(vals[static_cast<int64_t>(j0 + jj) * V + vc + u])
                                 : 0.0f;
            }
            for (int jj = threadIdx.x; jj < nj; jj += kThreads) {
                const int col = col_idx[gp + j0 + jj];
                if (col < 0) {
                    base_s[jj] = -1;
                } else if (KIND == 0) {
                    base_s[jj] = static_cast<int64_t>(col) * b.ldb;
                } else {
                    const int rs = b.R * b.S;
                    const int ch = col / rs, r = (col % rs) / b.S, s = col % b.S;
                    base_s[jj] = static_cast<int64_t>(ch) * b.H * b.W * b.Nb;
                    dr_s[jj] = r - b.pad;
                    ds_s[jj] = s - b.pad;
                }
            }
            __syncthreads();
            if (live) {
                for (int jj = 0; jj < nj; ++jj) {
                    if (base_s[jj] < 0) continue;  // pad column
                    float x;
                    if (KIND == 0) {
                        x = Elem<DT>::to_f(B[base_s[jj] + n]);
                    } else {
                        const int h = p0 + dr_s[jj], w = q0 + ds_s[jj];
                        x = (h >= 0 && h < b.H && w >= 0 && w < b.W)
                                ? Elem<DT>::to_f(B[base_s[jj] + (static_cast<int64_t>(h) * b.W + w) * b.Nb + nb])
                                : 0.0f;
                    }
#pragma unroll
                    for (int u = 0; u < kVC; ++u) acc[u] = __fadd_rn(acc[u], __fmul_rn(w_s[jj][u], x));
                }
            }
        }
        if (live) {
            for (int u = 0; u < nv; ++u) {
                const int64_t gr = static_cast<int64_t>(g) * V + vc + u;
                const int64_t row = c.compact ? static_cast<int64_t>(g - g_begin) * V + vc + u
                                              : static_cast<int64_t>(row_indices[gr]);
                store_from_f32(c.ptr, c.dtype, row * c.ldc + n, acc[u]);
            }
        }
    }
}

template <int DT>
int launch(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
           cudaStream_t s) {
    dim3 grid((b.N + kThreads - 1) / kThreads, g_end - g_begin);
    if (b.kind == 0)
        k_spmm_simt<DT, 0><<<grid, kThreads, 0, s>>>(a->row_indices, a->group_ptr, a->group_ncols,
                                                     a->col_idx, a->values, a->v, g_begin, b, c);
    else
        k_spmm_simt<DT, 1><<<grid, kThreads, 0, s>>>(a->row_indices, a->group_ptr, a->group_ncols,
                                                     a->col_idx, a->values, a->v, g_begin, b, c);
    SBW_LAUNCHED("k_spmm_simt");
    return SHFLBW_OK;
}

}  // namespace

int spmm_simt(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
              cudaStream_t s) {
    if (g_end <= g_begin || b.N <= 0) return SHFLBW_OK;
    if (g_end - g_begin > 65535) {  // grid.y limit: split
        for (int g0 = g_begin; g0 < g_end; g0 += 65535) {
            OutSpec cc = c;
            if (c.compact)
                cc.ptr = static_cast<char*>(c.ptr) +
                         static_cast<int64_t>(g0 - g_begin) * a->v * c.ldc * dtype_bytes(c.dtype);
            const int st = spmm_simt(a, g0, g0 + 65535 < g_end ? g0 + 65535 : g_end, b, cc, s);
            if (st) return st;
        }
        return SHFLBW_OK;
    }
    set_plan(std::string("k_spmm_simt kind=") + std::to_string(b.kind) + " v=" + std::to_string(a->v));
    if (a->dtype == SHFLBW_F32) return launch<SHFLBW_F32>(a, g_begin, g_end, b, c, s);
    return a->dtype == SHFLBW_BF16 ? launch<SHFLBW_BF16>(a, g_begin, g_end, b, c, s)
                                   : launch<SHFLBW_F16>(a, g_begin, g_end, b, c, s);
}

namespace {
template <typename U>
__global__ void k_unpermute(const int32_t* __restrict__ ri, int N, const U* __restrict__ src,
                            int64_t lds, U* __restrict__ dst, int64_t ldd) {
    const int r = blockIdx.x;
    const int64_t out_row = ri[r];
    if (out_row < 0) return;  // padding row of a sharded all-gather
    for (int n = threadIdx.x; n < N; n += blockDim.x) dst[out_row * ldd + n] = src[r * lds + n];
}
}  // namespace

int unpermute_impl(const int32_t* row_indices, int M, int N, const void* C_perm, int64_t ld_perm,
                   void* C, int64_t ldc, int dtype, cudaStream_t s) {
    if (M <= 0 || N <= 0) return SHFLBW_OK;
    if (dtype == SHFLBW_F32)
        k_unpermute<float><<<M, 256, 0, s>>>(row_indices, N, static_cast<const float*>(C_perm), ld_perm,
                                             static_cast<float*>(C), ldc);
    else
        k_unpermute<uint16_t><<<M, 256, 0, s>>>(row_indices, N, static_cast<const uint16_t*>(C_perm),
                                                ld_perm, static_cast<uint16_t*>(C), ldc);
    SBW_LAUNCHED("k_unpermute");
    return SHFLBW_OK;
}

}  // namespace sbw
