// prune.cu -- the Shfl-BW pruner on the GPU: the upstream
// producer of the converter's mask.  Replaces, with identical results,
//   importance_scores   src/pruning.cpp:61-66
//   kept_score          src/pruning.cpp:68-75
//   prune_unstructured  src/pruning.cpp:77-92
//   prune_vectorwise    src/pruning.cpp:94-121
//   kmeans_row_grouping src/pruning.cpp:183-337 (kmeans_assign, assignment_to_order)
//   prune_shflbw        src/pruning.cpp:339-362
//
// Exactness.  Integer and index work is exact by construction: Hamming
// distances between mask rows (the seeding distances are sums of 0/1
// squares, i.e. integers), stable radix sorts on monotone bit patterns
// (score / margin descending, index ascending = the reference's comparators),
// integer centroid counts.  Every floating-point sum runs in the reference's
// order with separately rounded operations (__dsub_rn / __dmul_rn /
// __dadd_rn, no FMA): centroid distances one thread per (row, cluster) over
// the columns in ascending order, column sums over the V rows in ascending
// order, kept_score over the linear index in ascending order.  The balanced
// assignment is the reference's greedy pass (rows by descending margin, each
// takes its nearest cluster with capacity left, ties to the lower cluster --
// the same choice as scanning its sorted preference list), run by one warp.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sbw {
namespace {

struct Buf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Buf() = default;
    Buf(const Buf&) = delete;
    ~Buf() {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        s = st;
        retain_pool();
        return cudaMallocAsync(&p, bytes ? bytes : 16, st);
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

int blocks(int64_t n, int per = 256) {
    const int64_t b = (n + per - 1) / per;
    return static_cast<int>(b < 1 ? 1 : (b > 1048576 ? 1048576 : b));
}

// +0.0 and -0.0 compare equal in the reference's comparators
__device__ __forceinline__ uint32_t canon(float x) { return x == 0.0f ? 0u : __float_as_uint(x); }
__device__ __forceinline__ uint64_t canon(double x) {
    return x == 0.0 ? 0ull : static_cast<uint64_t>(__double_as_longlong(x));
}

// ---- scores ----------------------------------------------------------------

__global__ void k_abs(const float* __restrict__ w, int64_t n, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = fabsf(w[i]);
}

// ImportanceMatrix ctor: finite and non-negative
__global__ void k_check_scores(const float* __restrict__ s, int64_t n, uint32_t* __restrict__ flag) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float x = s[i];
        if (!isfinite(x) || x < 0.0f) atomicOr(flag, 1u);
    }
}

// ---- kept_score: sum in linear index order ---------------------------------
// One block: each chunk of 4096 elements is compacted (order preserved) into
// shared memory, then thread 0 adds the kept values in sequence.  rows: the
// optional row map of a permuted view (element (r, c) = scores[rows[r]][c]).
constexpr int kKeptThreads = 1024;
constexpr int kKeptPer = 4;
constexpr int kKeptChunk = kKeptThreads * kKeptPer;

__global__ void __launch_bounds__(kKeptThreads) k_kept_score(const float* __restrict__ scores,
                                                             const uint8_t* __restrict__ mask,
                                                             const uint32_t* __restrict__ rows, int M, int K,
                                                             double* __restrict__ out) {
    __shared__ float kept[kKeptChunk];
    __shared__ int warp_tot[32];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const int64_t n = static_cast<int64_t>(M) * K;
    double acc = 0.0;
    for (int64_t base = 0; base < n; base += kKeptChunk) {
        float v[kKeptPer];
        int c = 0;
#pragma unroll
        for (int e = 0; e < kKeptPer; ++e) {
            const int64_t i = base + static_cast<int64_t>(t) * kKeptPer + e;
            bool m = false;
            float x = 0.0f;
            if (i < n && mask[i]) {
                m = true;
                const int64_t r = i / K, col = i - r * K;
                x = scores[(rows ? static_cast<int64_t>(rows[r]) : r) * K + col];
            }
            v[e] = x;
            c += m;
            if (!m) v[e] = __int_as_float(0x7fffffff);  // marker: skipped
        }
        // exclusive scan of the per-thread counts (thread order = linear order)
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_tot[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            int w = warp_tot[lane];
            int wi = w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, wi, o);
                if (lane >= o) wi += y;
            }
            warp_tot[lane] = wi - w;  // exclusive warp offsets
        }
        __syncthreads();
        int pos = warp_tot[wid] + incl - c;
#pragma unroll
        for (int e = 0; e < kKeptPer; ++e)
            if (__float_as_int(v[e]) != 0x7fffffff) kept[pos++] = v[e];
        // total kept in this chunk = last thread's inclusive end
        __syncthreads();
        if (t == kKeptThreads - 1) warp_tot[0] = pos;  // reuse: chunk total
        __syncthreads();
        if (t == 0) {
            const int tot = warp_tot[0];
            for (int k = 0; k < tot; ++k) acc = __dadd_rn(acc, static_cast<double>(kept[k]));
        }
        __syncthreads();
    }
    if (t == 0) *out = acc;
}

// ---- prune_unstructured ----------------------------------------------------

__global__ void k_unstructured_keys(const float* __restrict__ s, int64_t n, uint64_t* __restrict__ keys,
                                    uint32_t* __restrict__ vals) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // descending score, ascending linear index
        keys[i] = (static_cast<uint64_t>(0xffffffffu - canon(s[i])) << 32) | static_cast<uint32_t>(i);
        vals[i] = static_cast<uint32_t>(i);
    }
}

__global__ void k_mark_first(const uint32_t* __restrict__ vals, int64_t nkeep, uint8_t* __restrict__ mask) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nkeep;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        mask[vals[i]] = 1;
}

// ---- prune_vectorwise: one block per group ---------------------------------
// Column sums over the group's V rows (ascending row order, double), then a
// bitonic sort of (descending sum, ascending column) in shared memory; the
// first kcols columns are kept for every row of the group.
constexpr int kVwThreads = 1024;
constexpr int kVwMaxK = 16384;

__global__ void __launch_bounds__(kVwThreads) k_vectorwise(const float* __restrict__ scores,
                                                           const uint32_t* __restrict__ rows, int K, int V,
                                                           int kcols, int P, uint8_t* __restrict__ mask) {
    extern __shared__ __align__(16) unsigned char vw_smem[];
    uint64_t* key = reinterpret_cast<uint64_t*>(vw_smem);
    uint32_t* idx = reinterpret_cast<uint32_t*>(key + P);
    const int g = blockIdx.x;
    for (int c = threadIdx.x; c < P; c += blockDim.x) {
        uint64_t k = ~0ull;
        if (c < K) {
            double sum = 0.0;
            for (int i = 0; i < V; ++i) {
                const int64_t r = static_cast<int64_t>(g) * V + i;
                const int64_t src = rows ? static_cast<int64_t>(rows[r]) : r;
                sum = __dadd_rn(sum, static_cast<double>(scores[src * K + c]));
            }
            k = ~canon(sum);  // sums >= 0: descending
        }
        key[c] = k;
        idx[c] = static_cast<uint32_t>(c);
    }
    __syncthreads();
    // bitonic sort ascending by (key, idx)
    for (int size = 2; size <= P; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                const int j = i ^ stride;
                if (j > i) {
                    const bool up = (i & size) == 0;
                    const uint64_t ki = key[i], kj = key[j];
                    const uint32_t ii = idx[i], ij = idx[j];
                    const bool gt = ki > kj || (ki == kj && ii > ij);
                    if (gt == up) {
                        key[i] = kj;
                        key[j] = ki;
                        idx[i] = ij;
                        idx[j] = ii;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int e = threadIdx.x; e < kcols * V; e += blockDim.x) {
        const int j = e / V, i = e - j * V;
        mask[(static_cast<int64_t>(g) * V + i) * K + idx[j]] = 1;
    }
}

// ---- K-Means row grouping ----------------------------------------------------

// mask rows -> bit words (bit b of word w = column 64w + b)
__global__ void k_pack_bits(const uint8_t* __restrict__ mask, int M, int K, int W, uint64_t* __restrict__ words) {
    const int64_t total = static_cast<int64_t>(M) * W;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(t / W), w = static_cast<int>(t - static_cast<int64_t>(r) * W);
        uint64_t x = 0;
        for (int b = 0; b < 64; ++b) {
            const int c = w * 64 + b;
            if (c < K && mask[static_cast<int64_t>(r) * K + c]) x |= 1ull << b;
        }
        words[t] = x;
    }
}

__device__ __forceinline__ int hamming(const uint64_t* __restrict__ words, int W, int a, int b) {
    int d = 0;
    for (int w = 0; w < W; ++w) d += __popcll(words[static_cast<int64_t>(a) * W + w] ^ words[static_cast<int64_t>(b) * W + w]);
    return d;
}

// Farthest-point seeding (src/pruning.cpp:205-219), one block: seeds[0] = s0,
// then repeatedly the first row with the largest distance to its nearest seed.
__global__ void __launch_bounds__(1024) k_seed(const uint64_t* __restrict__ words, int M, int W, int G, int s0,
                                               int* __restrict__ nearest, int* __restrict__ seeds) {
    __shared__ int red_d[32], red_r[32];
    __shared__ int best_s;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
    if (t == 0) seeds[0] = s0;
    for (int r = t; r < M; r += blockDim.x) nearest[r] = hamming(words, W, r, s0);
    __syncthreads();
    for (int round = 1; round < G; ++round) {
        int bd = -1, br = 0x7fffffff;
        for (int r = t; r < M; r += blockDim.x) {
            const int d = nearest[r];
            if (d > bd) {  // ascending r per thread: keeps the first maximum
                bd = d;
                br = r;
            }
        }
        for (int o = 16; o; o >>= 1) {
            const int od = __shfl_xor_sync(0xffffffffu, bd, o), orr = __shfl_xor_sync(0xffffffffu, br, o);
            if (od > bd || (od == bd && orr < br)) {
                bd = od;
                br = orr;
            }
        }
        if (lane == 0) {
            red_d[wid] = bd;
            red_r[wid] = br;
        }
        __syncthreads();
        if (wid == 0) {
            bd = lane < nw ? red_d[lane] : -1;
            br = lane < nw ? red_r[lane] : 0x7fffffff;
            for (int o = 16; o; o >>= 1) {
                const int od = __shfl_xor_sync(0xffffffffu, bd, o), orr = __shfl_xor_sync(0xffffffffu, br, o);
                if (od > bd || (od == bd && orr < br)) {
                    bd = od;
                    br = orr;
                }
            }
            if (lane == 0) {
                best_s = br;
                seeds[round] = br;
            }
        }
        __syncthreads();
        const int best = best_s;
        for (int r = t; r < M; r += blockDim.x) nearest[r] = min(nearest[r], hamming(words, W, r, best));
        __syncthreads();
    }
}

__global__ void k_init_centroids(const uint64_t* __restrict__ words, const int* __restrict__ seeds, int G, int K,
                                 int W, double* __restrict__ ctr) {
    const int64_t total = static_cast<int64_t>(G) * K;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(t / K), j = static_cast<int>(t - static_cast<int64_t>(c) * K);
        ctr[t] = static_cast<double>((words[static_cast<int64_t>(seeds[c]) * W + (j >> 6)] >> (j & 63)) & 1ull);
    }
}

// dist[r][c] = sum_j (x_j - ctr_cj)^2, j ascending (src/pruning.cpp:235-243);
// thread index = c * M + r so a warp shares one centroid row
__global__ void k_dist(const uint64_t* __restrict__ words, const double* __restrict__ ctr, int M, int K, int W,
                       int G, double* __restrict__ dist) {
    const int64_t total = static_cast<int64_t>(M) * G;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(t / M), r = static_cast<int>(t - static_cast<int64_t>(c) * M);
        const uint64_t* x = words + static_cast<int64_t>(r) * W;
        const double* cj = ctr + static_cast<int64_t>(c) * K;
        double d = 0.0;
        for (int w = 0; w < W; ++w) {
            const uint64_t bits = x[w];
            const int jn = min(64, K - w * 64);
            for (int b = 0; b < jn; ++b) {
                const double diff = __dsub_rn(static_cast<double>((bits >> b) & 1ull), cj[w * 64 + b]);
                d = __dadd_rn(d, __dmul_rn(diff, diff));
            }
        }
        dist[static_cast<int64_t>(r) * G + c] = d;
    }
}

// margin = second - best with the reference's update rule
// (src/pruning.cpp:244-252); sort key: descending margin, stable by row
__global__ void k_margin(const double* __restrict__ dist, int M, int G, uint64_t* __restrict__ keys,
                         uint32_t* __restrict__ vals) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
        const double* d = dist + static_cast<int64_t>(r) * G;
        double best = 0.0, second = 0.0;
        for (int c = 0; c < G; ++c) {
            const double x = d[c];
            if (c == 0) {
                best = second = x;
            } else if (x < best) {
                second = best;
                best = x;
            } else if (c == 1 || x < second) {
                second = x;
            }
        }
        const double margin = G >= 2 ? __dsub_rn(second, best) : 0.0;
        keys[r] = ~canon(margin);
        vals[r] = static_cast<uint32_t>(r);
    }
}

// greedy balanced assignment (src/pruning.cpp:254-276), one warp: rows in
// order; each takes argmin over clusters with room of (distance, cluster)
__global__ void k_greedy(const double* __restrict__ dist, const uint32_t* __restrict__ row_order, int M, int G,
                         int V, int* __restrict__ counts, int* __restrict__ next) {
    const int lane = threadIdx.x;
    for (int c = lane; c < G; c += 32) counts[c] = 0;
    __syncwarp();
    for (int k = 0; k < M; ++k) {
        const int r = static_cast<int>(row_order[k]);
        const double* d = dist + static_cast<int64_t>(r) * G;
        double bd = 0.0;
        int bc = 0x7fffffff;
        for (int c = lane; c < G; c += 32) {
            if (counts[c] < V) {
                const double x = d[c];
                if (bc == 0x7fffffff || x < bd) {  // ascending c per lane: first minimum
                    bd = x;
                    bc = c;
                }
            }
        }
        for (int o = 16; o; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
            if (oc != 0x7fffffff && (bc == 0x7fffffff || od < bd || (od == bd && oc < bc))) {
                bd = od;
                bc = oc;
            }
        }
        if (lane == 0) {
            next[r] = bc;
            counts[bc] += 1;
        }
        __syncwarp();
    }
}

__global__ void k_count_bits(const uint64_t* __restrict__ words, const int* __restrict__ next, int M, int K, int W,
                             int* __restrict__ cnt) {
    const int64_t total = static_cast<int64_t>(M) * W;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(t / W), w = static_cast<int>(t - static_cast<int64_t>(r) * W);
        uint64_t bits = words[t];
        int* row = cnt + static_cast<int64_t>(next[r]) * K + w * 64;
        while (bits) {
            const int b = __ffsll(static_cast<long long>(bits)) - 1;
            atomicAdd(row + b, 1);
            bits &= bits - 1;
        }
    }
}

// centroid = (sum of 0/1 over the cluster's rows, an exact integer) / V
__global__ void k_centroids(const int* __restrict__ cnt, int64_t n, int V, double* __restrict__ ctr) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ctr[t] = __ddiv_rn(static_cast<double>(cnt[t]), static_cast<double>(V));
}

__global__ void k_changed(const int* __restrict__ next, int* __restrict__ assign, int M, uint32_t* __restrict__ flag) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) {
        if (next[r] != assign[r]) atomicOr(flag, 1u);
        assign[r] = next[r];
    }
}

// assignment_to_order (src/pruning.cpp:281-293): clusters in order of their
// first row, rows ascending inside; one thread, O(M + G).  `order` doubles as
// the rank -> cluster table until the final pass overwrites it.
__global__ void k_order(const int* __restrict__ assign, int M, int G, int* __restrict__ rank,
                        int* __restrict__ size, uint32_t* __restrict__ order) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int c = 0; c < G; ++c) {
        rank[c] = -1;
        size[c] = 0;
    }
    int nr = 0;
    for (int r = 0; r < M; ++r) {
        const int c = assign[r];
        if (rank[c] < 0) {
            rank[c] = nr;
            order[nr] = static_cast<uint32_t>(c);  // rank -> cluster
            ++nr;
        }
        size[c] += 1;
    }
    int off = 0;
    for (int k = 0; k < nr; ++k) {  // size[] becomes each cluster's start offset
        const int c = static_cast<int>(order[k]);
        const int sz = size[c];
        size[c] = off;
        off += sz;
    }
    for (int r = 0; r < M; ++r) order[size[assign[r]]++] = static_cast<uint32_t>(r);
}

// shuffled[perm[r]] = permuted_mask[r] (src/pruning.cpp:346-351)
__global__ void k_unpermute_mask(const uint8_t* __restrict__ pm, const uint32_t* __restrict__ perm, int M, int K,
                                 uint8_t* __restrict__ out) {
    const int64_t total = static_cast<int64_t>(M) * K;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / K, c = t - r * K;
        out[static_cast<int64_t>(perm[r]) * K + c] = pm[t];
    }
}

__global__ void k_iota(uint32_t* __restrict__ p, int M) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < M; r += gridDim.x * blockDim.x) p[r] = r;
}

// ---- host pieces --------------------------------------------------------------

int64_t keep_count(double ratio, int64_t total) { return static_cast<int64_t>(std::llround(ratio * double(total))); }

int check_scores(const float* scores, int64_t n, cudaStream_t s) {
    if (n == 0) return SHFLBW_OK;
    if (!scores) return fail(SHFLBW_BAD_PARAMS, "scores is null");
    Buf flag;
    SBW_CUDA(flag.alloc(4, s));
    SBW_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
    k_check_scores<<<blocks(n), 256, 0, s>>>(scores, n, flag.as<uint32_t>());
    SBW_LAUNCHED("k_check_scores");
    uint32_t h = 0;
    SBW_CUDA(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    if (h) return fail(SHFLBW_BAD_PARAMS, "ImportanceMatrix: scores must be finite and non-negative");
    return SHFLBW_OK;
}

int kept_score_impl(const float* scores, const uint8_t* mask, const uint32_t* rows, int M, int K, double* out,
                    cudaStream_t s) {
    Buf d;
    SBW_CUDA(d.alloc(sizeof(double), s));
    k_kept_score<<<1, kKeptThreads, 0, s>>>(scores, mask, rows, M, K, d.as<double>());
    SBW_LAUNCHED("k_kept_score");
    SBW_CUDA(cudaMemcpyAsync(out, d.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int vectorwise_impl(const float* scores, const uint32_t* rows, int M, int K, int V, double alpha, uint8_t* mask,
                    cudaStream_t s) {
    if (V <= 0 || M % V != 0) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    if (!(alpha > 0.0) || alpha > 1.0) return fail(SHFLBW_BAD_PARAMS, "alpha must be in (0, 1]");
    if (K > kVwMaxK) return fail(SHFLBW_UNSUPPORTED, "prune_vectorwise: K > 16384");
    SBW_CUDA(cudaMemsetAsync(mask, 0, static_cast<size_t>(M) * K, s));
    if (M == 0 || K == 0) return SHFLBW_OK;
    const int kcols = static_cast<int>(keep_count(alpha, K));
    int P = 1;
    while (P < K) P <<= 1;
    const size_t smem = static_cast<size_t>(P) * 12;
    // the attribute is per device: set on every call (not a hot path)
    SBW_CUDA(cudaFuncSetAttribute(k_vectorwise, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_vectorwise<<<M / V, kVwThreads, smem, s>>>(scores, rows, K, V, kcols, P, mask);
    SBW_LAUNCHED("k_vectorwise");
    return SHFLBW_OK;
}

int validate_cfg(const shflbw_prune_config* cfg, int M) {
    if (!cfg) return fail(SHFLBW_BAD_PARAMS, "config is null");
    if (!(cfg->alpha > 0.0) || cfg->alpha > 1.0) return fail(SHFLBW_BAD_PARAMS, "alpha must be in (0, 1]");
    if (!(cfg->beta_factor > 0.0)) return fail(SHFLBW_BAD_PARAMS, "beta_factor must be positive");
    if (M == 0 || cfg->v == 0 || M % static_cast<int64_t>(cfg->v) != 0)
        return fail(SHFLBW_BAD_PARAMS, "V must divide M, M >= 1");
    if (cfg->restarts == 0) return fail(SHFLBW_BAD_PARAMS, "restarts must be >= 1");
    if (cfg->kmeans_max_iters == 0) return fail(SHFLBW_BAD_PARAMS, "kmeans_max_iters must be >= 1");
    return SHFLBW_OK;
}

int grouping_impl(const uint8_t* mask, const float* scores, int M, int K, const shflbw_prune_config* cfg,
                  uint32_t* order_out, cudaStream_t s) {
    const int V = static_cast<int>(cfg->v), G = M / V, W = K > 0 ? (K + 63) / 64 : 1;
    Buf words, nearest, seeds, ctr, dist, keys, vals, keys2, vals2, counts, next, assign, cnt, flag, rank, fill,
        order, vmask;
    SBW_CUDA(words.alloc(sizeof(uint64_t) * M * W, s));
    SBW_CUDA(nearest.alloc(sizeof(int) * M, s));
    SBW_CUDA(seeds.alloc(sizeof(int) * G, s));
    SBW_CUDA(ctr.alloc(sizeof(double) * G * std::max(K, 1), s));
    SBW_CUDA(dist.alloc(sizeof(double) * M * G, s));
    SBW_CUDA(keys.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(vals.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(keys2.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(vals2.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(counts.alloc(sizeof(int) * G, s));
    SBW_CUDA(next.alloc(sizeof(int) * M, s));
    SBW_CUDA(assign.alloc(sizeof(int) * M, s));
    SBW_CUDA(cnt.alloc(sizeof(int) * G * std::max(K, 1), s));
    SBW_CUDA(flag.alloc(4, s));
    SBW_CUDA(rank.alloc(sizeof(int) * G, s));
    SBW_CUDA(fill.alloc(sizeof(int) * G, s));
    SBW_CUDA(order.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(vmask.alloc(static_cast<size_t>(M) * std::max(K, 1), s));
    k_pack_bits<<<blocks(static_cast<int64_t>(M) * W), 256, 0, s>>>(mask, M, K, W, words.as<uint64_t>());
    SBW_LAUNCHED("k_pack_bits");
    double best_score = -1.0;
    for (uint32_t restart = 0; restart < cfg->restarts; ++restart) {
        std::mt19937_64 rng(cfg->seed + restart);  // src/pruning.cpp:205-207
        const int s0 = static_cast<int>(rng() % static_cast<uint64_t>(M));
        k_seed<<<1, 1024, 0, s>>>(words.as<uint64_t>(), M, W, G, s0, nearest.as<int>(), seeds.as<int>());
        SBW_LAUNCHED("k_seed");
        k_init_centroids<<<blocks(static_cast<int64_t>(G) * K), 256, 0, s>>>(words.as<uint64_t>(), seeds.as<int>(),
                                                                            G, K, W, ctr.as<double>());
        SBW_LAUNCHED("k_init_centroids");
        SBW_CUDA(cudaMemsetAsync(assign.p, 0xff, sizeof(int) * M, s));  // no row assigned yet
        for (uint32_t iter = 0; iter < cfg->kmeans_max_iters; ++iter) {
            k_dist<<<blocks(static_cast<int64_t>(M) * G), 256, 0, s>>>(words.as<uint64_t>(), ctr.as<double>(), M, K,
                                                                      W, G, dist.as<double>());
            SBW_LAUNCHED("k_dist");
            k_margin<<<blocks(M), 256, 0, s>>>(dist.as<double>(), M, G, keys.as<uint64_t>(), vals.as<uint32_t>());
            SBW_LAUNCHED("k_margin");
            if (int st = radix_sort_pairs(keys.as<uint64_t>(), vals.as<uint32_t>(), keys2.as<uint64_t>(),
                                          vals2.as<uint32_t>(), M, s))
                return st;
            k_greedy<<<1, 32, 0, s>>>(dist.as<double>(), vals.as<uint32_t>(), M, G, V, counts.as<int>(),
                                      next.as<int>());
            SBW_LAUNCHED("k_greedy");
            SBW_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * G * std::max(K, 1), s));
            k_count_bits<<<blocks(static_cast<int64_t>(M) * W), 256, 0, s>>>(words.as<uint64_t>(), next.as<int>(), M,
                                                                            K, W, cnt.as<int>());
            SBW_LAUNCHED("k_count_bits");
            k_centroids<<<blocks(static_cast<int64_t>(G) * K), 256, 0, s>>>(cnt.as<int>(), static_cast<int64_t>(G) * K,
                                                                           V, ctr.as<double>());
            SBW_LAUNCHED("k_centroids");
            SBW_CUDA(cudaMemsetAsync(flag.p, 0, 4, s));
            k_changed<<<blocks(M), 256, 0, s>>>(next.as<int>(), assign.as<int>(), M, flag.as<uint32_t>());
            SBW_LAUNCHED("k_changed");
            uint32_t changed = 0;
            SBW_CUDA(cudaMemcpyAsync(&changed, flag.p, 4, cudaMemcpyDeviceToHost, s));
            SBW_CUDA(cudaStreamSynchronize(s));
            if (!changed) break;
        }
        k_order<<<1, 1, 0, s>>>(assign.as<int>(), M, G, rank.as<int>(), fill.as<int>(), order.as<uint32_t>());
        SBW_LAUNCHED("k_order");
        // score: kept_score(permuted, prune_vectorwise(permuted, v, alpha))
        if (int st = vectorwise_impl(scores, order.as<uint32_t>(), M, K, V, cfg->alpha, vmask.as<uint8_t>(), s))
            return st;
        double sc = 0.0;
        if (int st = kept_score_impl(scores, vmask.as<uint8_t>(), order.as<uint32_t>(), M, K, &sc, s)) return st;
        if (sc > best_score) {
            best_score = sc;
            SBW_CUDA(cudaMemcpyAsync(order_out, order.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToDevice, s));
        }
    }
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int unstructured_impl(const float* scores, int M, int K, double keep_ratio, uint8_t* mask, cudaStream_t s) {
    if (!(keep_ratio > 0.0) || keep_ratio > 1.0) return fail(SHFLBW_BAD_PARAMS, "keep_ratio must be in (0, 1]");
    const int64_t n = static_cast<int64_t>(M) * K;
    if (n >= (1LL << 31)) return fail(SHFLBW_UNSUPPORTED, "prune_unstructured: M*K >= 2^31");
    SBW_CUDA(cudaMemsetAsync(mask, 0, static_cast<size_t>(n), s));
    if (n == 0) return SHFLBW_OK;
    const int64_t nkeep = keep_count(keep_ratio, n);
    Buf keys, vals, keys2, vals2;
    SBW_CUDA(keys.alloc(sizeof(uint64_t) * n, s));
    SBW_CUDA(vals.alloc(sizeof(uint32_t) * n, s));
    SBW_CUDA(keys2.alloc(sizeof(uint64_t) * n, s));
    SBW_CUDA(vals2.alloc(sizeof(uint32_t) * n, s));
    k_unstructured_keys<<<blocks(n), 256, 0, s>>>(scores, n, keys.as<uint64_t>(), vals.as<uint32_t>());
    SBW_LAUNCHED("k_unstructured_keys");
    if (int st = radix_sort_pairs(keys.as<uint64_t>(), vals.as<uint32_t>(), keys2.as<uint64_t>(),
                                  vals2.as<uint32_t>(), static_cast<int>(n), s))
        return st;
    if (nkeep > 0) {
        k_mark_first<<<blocks(nkeep), 256, 0, s>>>(vals.as<uint32_t>(), nkeep, mask);
        SBW_LAUNCHED("k_mark_first");
    }
    return SHFLBW_OK;
}

}  // namespace
}  // namespace sbw

using namespace sbw;

extern "C" {

int shflbw_cu_importance_scores(const float* w, int64_t n, float* scores, shflbw_stream_t stream) {
    if (n < 0 || (n > 0 && (!w || !scores))) return fail(SHFLBW_BAD_PARAMS, "importance_scores: bad arguments");
    if (n == 0) return SHFLBW_OK;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    k_abs<<<blocks(n), 256, 0, s>>>(w, n, scores);
    SBW_LAUNCHED("k_abs");
    return SHFLBW_OK;
}

int shflbw_cu_kept_score(const float* scores, const uint8_t* mask, int32_t M, int32_t K, double* out,
                         shflbw_stream_t stream) {
    if (M < 0 || K < 0 || !out) return fail(SHFLBW_BAD_PARAMS, "kept_score: bad arguments");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (int st = check_scores(scores, static_cast<int64_t>(M) * K, s)) return st;
    return kept_score_impl(scores, mask, nullptr, M, K, out, s);
}

int shflbw_cu_prune_unstructured(const float* scores, int32_t M, int32_t K, double keep_ratio, uint8_t* mask,
                                 shflbw_stream_t stream) {
    if (M < 0 || K < 0) return fail(SHFLBW_BAD_PARAMS, "prune_unstructured: negative extent");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (int st = check_scores(scores, static_cast<int64_t>(M) * K, s)) return st;
    return unstructured_impl(scores, M, K, keep_ratio, mask, s);
}

int shflbw_cu_prune_vectorwise(const float* scores, int32_t M, int32_t K, uint32_t V, double alpha, uint8_t* mask,
                               shflbw_stream_t stream) {
    if (M < 0 || K < 0) return fail(SHFLBW_BAD_PARAMS, "prune_vectorwise: negative extent");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (int st = check_scores(scores, static_cast<int64_t>(M) * K, s)) return st;
    if (V == 0 || V > 0x7fffffffu) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    return vectorwise_impl(scores, nullptr, M, K, static_cast<int>(V), alpha, mask, s);
}

int shflbw_cu_kmeans_row_grouping(const uint8_t* mask, const float* scores, int32_t M, int32_t K,
                                  const shflbw_prune_config* cfg, uint32_t* order, shflbw_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!cfg || cfg->v == 0 || M < 0 || M % static_cast<int64_t>(cfg->v) != 0)
        return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    if (int st = validate_cfg(cfg, M)) return st;
    if (int st = check_scores(scores, static_cast<int64_t>(M) * K, s)) return st;
    return grouping_impl(mask, scores, M, K, cfg, order, s);
}

int shflbw_cu_prune_shflbw(const float* scores, int32_t M, int32_t K, const shflbw_prune_config* cfg, uint8_t* mask,
                           uint32_t* permutation, double* kept_score, shflbw_stream_t stream) {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (M < 0 || K < 0 || !kept_score) return fail(SHFLBW_BAD_PARAMS, "prune_shflbw: bad arguments");
    if (int st = validate_cfg(cfg, M)) return st;
    if (int st = check_scores(scores, static_cast<int64_t>(M) * K, s)) return st;
    const int64_t n = static_cast<int64_t>(M) * K;
    Buf beta_mask, perm, pmask, shuffled, identity;
    SBW_CUDA(beta_mask.alloc(n, s));
    SBW_CUDA(perm.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(pmask.alloc(n, s));
    SBW_CUDA(shuffled.alloc(n, s));
    SBW_CUDA(identity.alloc(n, s));
    const double beta = std::min(1.0, cfg->beta_factor * cfg->alpha);  // PruneConfig::beta
    int st;
    if ((st = unstructured_impl(scores, M, K, beta, beta_mask.as<uint8_t>(), s))) return st;
    if ((st = grouping_impl(beta_mask.as<uint8_t>(), scores, M, K, cfg, perm.as<uint32_t>(), s))) return st;
    const int V = static_cast<int>(cfg->v);
    if ((st = vectorwise_impl(scores, perm.as<uint32_t>(), M, K, V, cfg->alpha, pmask.as<uint8_t>(), s))) return st;
    if (n > 0) {
        k_unpermute_mask<<<blocks(n), 256, 0, s>>>(pmask.as<uint8_t>(), perm.as<uint32_t>(), M, K,
                                                   shuffled.as<uint8_t>());
        SBW_LAUNCHED("k_unpermute_mask");
    }
    double shuffled_score = 0.0, identity_score = 0.0;
    if ((st = kept_score_impl(scores, shuffled.as<uint8_t>(), nullptr, M, K, &shuffled_score, s))) return st;
    if ((st = vectorwise_impl(scores, nullptr, M, K, V, cfg->alpha, identity.as<uint8_t>(), s))) return st;
    if ((st = kept_score_impl(scores, identity.as<uint8_t>(), nullptr, M, K, &identity_score, s))) return st;
    // safety net: never lose to the identity-permutation vector-wise prune
    if (identity_score >= shuffled_score) {
        SBW_CUDA(cudaMemcpyAsync(mask, identity.p, static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
        k_iota<<<blocks(M), 256, 0, s>>>(permutation, M);
        SBW_LAUNCHED("k_iota");
        *kept_score = identity_score;
    } else {
        SBW_CUDA(cudaMemcpyAsync(mask, shuffled.p, static_cast<size_t>(n), cudaMemcpyDeviceToDevice, s));
        SBW_CUDA(cudaMemcpyAsync(permutation, perm.p, sizeof(uint32_t) * M, cudaMemcpyDeviceToDevice, s));
        *kept_score = shuffled_score;
    }
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

}  // extern "C"
