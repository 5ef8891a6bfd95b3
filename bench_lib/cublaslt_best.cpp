// cublaslt_best.cpp -- benchmark-only helper (not part of the product): the
// dense bf16/fp16 GEMM baseline through cuBLASLt with the best of its top-k
// heuristic algorithms, for bench.py's "speed-up vs cuBLAS dense" line.
//
// Row-major C[M][N] = A[M][K] * B[K][N] is run as the column-major
// C^T = B^T * A^T (m = N, n = M, k = K), fp32 accumulation, output in the
// input type.  sbw_lt_select() times every returned algorithm on the given
// buffers (CUDA events, median of `reps` after a warm-up) and keeps the
// fastest; sbw_lt_run() launches it (graph-capturable).
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

namespace {

struct Plan {
    cublasLtHandle_t h = nullptr;
    cublasLtMatmulDesc_t op = nullptr;
    cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
    std::vector<cublasLtMatmulHeuristicResult_t> algos;
    int best = -1;
    void* ws = nullptr;
    size_t ws_size = 0;
    float best_ms = 0.f;
};

Plan g;

void release() {
    if (g.la) cublasLtMatrixLayoutDestroy(g.la);
    if (g.lb) cublasLtMatrixLayoutDestroy(g.lb);
    if (g.lc) cublasLtMatrixLayoutDestroy(g.lc);
    if (g.op) cublasLtMatmulDescDestroy(g.op);
    g.la = g.lb = g.lc = nullptr;
    g.op = nullptr;
    g.algos.clear();
    g.best = -1;
}

int launch(int i, const void* A, const void* B, void* C, cudaStream_t s) {
    const float alpha = 1.f, beta = 0.f;
    // column-major: "A" operand = B^T (N x K, ld N), "B" operand = A^T (K x M, ld K)
    return cublasLtMatmul(g.h, g.op, &alpha, B, g.la, A, g.lb, &beta, C, g.lc, C, g.lc, &g.algos[i].algo, g.ws,
                          g.ws_size, s) == CUBLAS_STATUS_SUCCESS
               ? 0
               : 1;
}

}  // namespace

extern "C" {

// dtype: 1 = bf16, 2 = fp16.  Returns the number of candidate algorithms
// timed (0 on failure); *best_ms = the winner's median time per call.
int sbw_lt_select(int M, int N, int K, int dtype, const void* A, const void* B, void* C, int topk, int reps,
                  float* best_ms, cudaStream_t s) {
    if (!g.h && cublasLtCreate(&g.h) != CUBLAS_STATUS_SUCCESS) return 0;
    release();
    const cudaDataType_t t = dtype == 2 ? CUDA_R_16F : CUDA_R_16BF;
    if (!g.ws) {
        g.ws_size = 64u << 20;
        if (cudaMalloc(&g.ws, g.ws_size) != cudaSuccess) return 0;
    }
    cublasLtMatmulDescCreate(&g.op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
    cublasLtMatrixLayoutCreate(&g.la, t, N, K, N);
    cublasLtMatrixLayoutCreate(&g.lb, t, K, M, K);
    cublasLtMatrixLayoutCreate(&g.lc, t, N, M, N);
    cublasLtMatmulPreference_t pref;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &g.ws_size,
                                         sizeof(g.ws_size));
    g.algos.resize(std::max(1, topk));
    int found = 0;
    cublasLtMatmulAlgoGetHeuristic(g.h, g.op, g.la, g.lb, g.lc, g.lc, pref, topk, g.algos.data(), &found);
    cublasLtMatmulPreferenceDestroy(pref);
    g.algos.resize(found);
    if (!found) return 0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    int timed = 0;
    for (int i = 0; i < found; ++i) {
        if (g.algos[i].state != CUBLAS_STATUS_SUCCESS) continue;
        bool ok = true;
        for (int w = 0; w < 3 && ok; ++w) ok = launch(i, A, B, C, s) == 0;
        if (!ok || cudaStreamSynchronize(s) != cudaSuccess) {
            cudaGetLastError();
            continue;
        }
        std::vector<float> t_ms;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(e0, s);
            launch(i, A, B, C, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            t_ms.push_back(ms);
        }
        std::sort(t_ms.begin(), t_ms.end());
        const float med = t_ms[t_ms.size() / 2];
        ++timed;
        if (med < best) {
            best = med;
            g.best = i;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    g.best_ms = best;
    if (best_ms) *best_ms = best;
    return g.best >= 0 ? timed : 0;
}

// Launch the selected algorithm on (A, B, C) of the selected shape.
int sbw_lt_run(const void* A, const void* B, void* C, cudaStream_t s) {
    if (g.best < 0) return 1;
    return launch(g.best, A, B, C, s);
}

}  // extern "C"
