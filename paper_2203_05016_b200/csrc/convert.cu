// convert.cu -- K1: Shfl-BW format converter on the GPU.
//
// Replaces validate_pattern(ShflBW) + compress_shflbw
// (/root/reference/proj/src/formats.cpp:85-93, 113-125, 140-181).
//
// The reference groups rows by exact mask-row equality with a std::map keyed
// by the whole row (src/formats.cpp:40-46), cuts each class into V-row chunks
// of ascending rows and orders the chunks by first row.  Here (M <= 32768):
//
//   K1 k_pack_rows   one warp per row: the mask row becomes 64-bit words with
//                    column 0 as the MSB of word 0 (so unsigned word order is
//                    the reference's lexicographic byte order), popcount and
//                    a 64-bit hash; bytes > 1 are flagged (SparsityMask's
//                    constructor rejects them, src/matrix.cpp:24-31).  The
//                    hash claims a slot of an open-addressing class table;
//                    the slot keeps the class's smallest row and its size.
//   K2 k_class_check every row against its class representative (smallest
//                    row) word by word -- a hash collision is detected
//                    exactly and the host retries with another seed, so the
//                    grouping is exact, not probabilistic.
//   K3 k_plan        one CTA: rows ordered by (representative, row) -- a
//                    shared-memory LSD sort for M <= 4096, per-1024-row chunk
//                    ranks (k_chunk_rank, k_chunk_prefix) above; rank in
//                    class, leaders = ranks that are multiples of V, group
//                    number = exclusive scan of the leaders in row order (the
//                    reference's group order), row_indices, n_g, group_ptr.
//   K4 k_pack_group  per (group, 64-column block): the column list from the
//                    leader's words, values gathered, rounded to bf16/fp16
//                    (RNE) and written column-major (V contiguous).
//
// Larger M (and option "converter_legacy"): the sort-based pipeline -- a
// stable radix sort of (hash, row) pairs makes equal rows runs (k_runs checks
// adjacent rows exactly), then k_assign / k_pack_cols / k_pack_values.
//
// A failing class is reported like the reference: the lexicographically
// smallest failing support class (word-wise argmin over run heads) gives its
// smallest row as fail_row.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sbw {

namespace {

constexpr int kRadixTile = 2048;  // items per block (256 threads x 8)
constexpr int kScanTile = 2048;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}

// per-word term of a row hash (summed over the row's words): a bijection of
// the word keyed by (seed, word index) -- two 64-bit multiplies, not two full
// mix64 rounds (the hash was 60 % of k_pack_rows16's instructions); the row
// sum is finalised with mix64 before it indexes the class table
__device__ __forceinline__ uint64_t word_hash(uint64_t word, int w, uint64_t seed) {
    uint64_t x = (word ^ seed) + 0x632BE59BD9B4E019ULL * static_cast<uint64_t>(w + 1);
    x *= 0x9E3779B97F4A7C15ULL;
    x ^= x >> 32;
    x *= 0xD6E8FEB86659FD93ULL;
    return x ^ (x >> 29);
}

// flags[0]: mask byte > 1, flags[1]: hash collision, flags[2]: failing class,
// flags[3]: upload range error
// Class table (hash planner, M <= kPlanMax): open addressing over P = 2^k >=
// 2M slots; a row's 64-bit hash claims a slot (atomicCAS), the slot keeps the
// class's smallest row (atomicMin) and its size (atomicAdd from 0xffffffff).
// The table is reset by one 0xff memset.  Equal rows always share a slot;
// rows of different classes sharing one are caught by k_class_check.
struct ClassTable {
    uint64_t* key = nullptr;
    uint32_t* minrow = nullptr;
    uint32_t* cnt = nullptr;
    uint32_t* slot = nullptr;  // [M] slot of each row
    uint32_t mask = 0;
};

__device__ __forceinline__ void table_insert(const ClassTable& t, uint64_t h, uint32_t r) {
    h = mix64(h);
    if (h == ~0ull) h = ~1ull;  // ~0 marks an empty slot
    uint32_t s = static_cast<uint32_t>(h) & t.mask;
    for (;;) {
        const unsigned long long prev =
            atomicCAS(reinterpret_cast<unsigned long long*>(t.key + s), ~0ull, static_cast<unsigned long long>(h));
        if (prev == ~0ull || prev == h) break;
        s = (s + 1) & t.mask;
    }
    atomicMin(t.minrow + s, r);
    atomicAdd(t.cnt + s, 1u);
    t.slot[r] = s;
}

__global__ void k_pack_rows(const uint8_t* __restrict__ mask, int M, int K, int W,
                            uint64_t seed, uint64_t* __restrict__ words,
                            int* __restrict__ popc, uint64_t* __restrict__ keys,
                            uint32_t* __restrict__ vals, uint32_t* __restrict__ flags, ClassTable tab) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (r >= M) return;
    const uint8_t* row = mask + static_cast<int64_t>(r) * K;
    uint64_t h = 0;
    int pc = 0;
    bool bad = false;
    for (int w = 0; w < W; ++w) {
        const int c0 = w * 64;
        const uint8_t b0 = (c0 + lane < K) ? row[c0 + lane] : 0;
        const uint8_t b1 = (c0 + 32 + lane < K) ? row[c0 + 32 + lane] : 0;
        bad |= (b0 > 1) | (b1 > 1);
        const uint32_t hi = __brev(__ballot_sync(0xffffffffu, b0 != 0));
        const uint32_t lo = __brev(__ballot_sync(0xffffffffu, b1 != 0));
        const uint64_t word = (static_cast<uint64_t>(hi) << 32) | lo;
        if (lane == (w & 31)) words[static_cast<int64_t>(r) * W + w] = word;
        pc += __popc(hi) + __popc(lo);
        h += word_hash(word, w, seed);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags[0], 1u);
    if (lane == 0) {
        popc[r] = pc;
        if (tab.key) {
            table_insert(tab, h, static_cast<uint32_t>(r));
        } else {
            keys[r] = h;
            vals[r] = static_cast<uint32_t>(r);
        }
    }
}

// Same, 16 mask bytes per lane load (K % 16 == 0, 16-byte aligned mask): a
// warp covers 512 columns per load; lane l's 16 bytes become bits
// 15..0 of its pattern, four consecutive lanes' patterns one 64-bit word
// (column 0 = MSB, as k_pack_rows).
__global__ void __launch_bounds__(256, 8) k_pack_rows16(const uint8_t* __restrict__ mask, int M, int K, int W, uint64_t seed,
                              uint64_t* __restrict__ words, int* __restrict__ popc, uint64_t* __restrict__ keys,
                              uint32_t* __restrict__ vals, uint32_t* __restrict__ flags, ClassTable tab) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (r >= M) return;
    const uint4* row = reinterpret_cast<const uint4*>(mask + static_cast<int64_t>(r) * K);
    const int nchunk = K / 16;
    uint64_t h = 0;
    int pc = 0;
    bool bad = false;
    // the row's 16-byte chunks are loaded 4 warp-rounds at a time (2 KB per
    // warp in flight) before they are decoded: the decode and the shuffles
    // otherwise expose one load latency per 512 columns
    constexpr int kBatch = 4;
    for (int cb = 0; cb < nchunk; cb += 32 * kBatch) {
        uint4 qb[kBatch];
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int c = cb + 32 * b + lane;
            qb[b] = c < nchunk ? __ldcs(row + c) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int b = 0; b < kBatch; ++b) {
            const int c0 = cb + 32 * b;
            if (c0 >= nchunk) break;
            const uint4 q = qb[b];
            // bytes are 0/1 (anything else is flagged and the mask rejected):
            // (x & 0x01010101) * 0x08040201 gathers the 4 bytes' low bits into
            // bits 27..24, first byte (lowest column) highest
            bad |= ((q.x | q.y | q.z | q.w) & 0xFEFEFEFEu) != 0;
            const uint32_t n0 = ((q.x & 0x01010101u) * 0x08040201u) >> 24;
            const uint32_t n1 = ((q.y & 0x01010101u) * 0x08040201u) >> 24;
            const uint32_t n2 = ((q.z & 0x01010101u) * 0x08040201u) >> 24;
            const uint32_t n3 = ((q.w & 0x01010101u) * 0x08040201u) >> 24;
            const uint32_t pat = (n0 << 12) | (n1 << 8) | (n2 << 4) | n3;
            const uint32_t p1 = __shfl_down_sync(0xffffffffu, pat, 1);
            const uint32_t p2 = __shfl_down_sync(0xffffffffu, pat, 2);
            const uint32_t p3 = __shfl_down_sync(0xffffffffu, pat, 3);
            const int w = (c0 + lane) / 4;  // word of lanes 4q..4q+3
            if ((lane & 3) == 0 && w < W) {
                const uint64_t word = (static_cast<uint64_t>(pat) << 48) | (static_cast<uint64_t>(p1) << 32) |
                                      (static_cast<uint64_t>(p2) << 16) | p3;
                words[static_cast<int64_t>(r) * W + w] = word;
                pc += __popcll(word);
                h += word_hash(word, w, seed);
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        h += __shfl_xor_sync(0xffffffffu, h, o);
        pc += __shfl_xor_sync(0xffffffffu, pc, o);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags[0], 1u);
    if (lane == 0) {
        popc[r] = pc;
        if (tab.key) {
            table_insert(tab, h, static_cast<uint32_t>(r));
        } else {
            keys[r] = h;
            vals[r] = static_cast<uint32_t>(r);
        }
    }
}

// Re-hash with another seed (collision retry): one warp per row.
__global__ void k_hash_rows(const uint64_t* __restrict__ words, int M, int W, uint64_t seed,
                            uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (r >= M) return;
    uint64_t h = 0;
    for (int w = lane; w < W; w += 32) h += word_hash(words[static_cast<int64_t>(r) * W + w], w, seed);
    for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0) {
        keys[r] = h;
        vals[r] = static_cast<uint32_t>(r);
    }
}

// ---- stable LSD radix sort of (u64 key, u32 value), 8-bit digits ---------

// Small-n sort (n <= kSmallSort) in one CTA: bitonic network over (key,
// original position) in shared memory -- the exact order of the stable LSD
// radix sort (ascending key, ties in input order), in one launch instead of
// 8 x (histogram, scan, scatter).
constexpr int kSmallSort = 4096;

__global__ void __launch_bounds__(1024) k_sort_small(uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                     int n, int P) {
    extern __shared__ __align__(16) unsigned char sm_sort[];
    uint64_t* k = reinterpret_cast<uint64_t*>(sm_sort);
    uint32_t* v = reinterpret_cast<uint32_t*>(k + P);
    uint32_t* pos = v + P;
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const bool live = i < n;
        k[i] = live ? keys[i] : ~0ull;
        v[i] = live ? vals[i] : 0u;
        pos[i] = static_cast<uint32_t>(i);
    }
    __syncthreads();
    for (int kk = 2; kk <= P; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            // pair t of the P / 2 compare-exchanges of this step: i = lower
            // index (bit j clear), ixj = i + j -- no idle half of the threads
            for (int t = threadIdx.x; t < (P >> 1); t += blockDim.x) {
                const int i = ((t & ~(j - 1)) << 1) | (t & (j - 1));
                const int ixj = i | j;
                {
                    const bool up = (i & kk) == 0;
                    const uint64_t ka = k[i], kb = k[ixj];
                    const uint32_t pa = pos[i], pb = pos[ixj];
                    const bool b_lt_a = kb < ka || (kb == ka && pb < pa);
                    if (b_lt_a == up) {
                        k[i] = kb;
                        k[ixj] = ka;
                        pos[i] = pb;
                        pos[ixj] = pa;
                        const uint32_t tv = v[i];
                        v[i] = v[ixj];
                        v[ixj] = tv;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        keys[i] = k[i];
        vals[i] = v[i];
    }
}

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int n, int shift,
                             int* __restrict__ hist, int nblocks) {
    __shared__ int cnt[256];
    cnt[threadIdx.x] = 0;
    __syncthreads();
    const int base = blockIdx.x * kRadixTile;
    for (int i = threadIdx.x; i < kRadixTile; i += 256) {
        const int idx = base + i;
        if (idx < n) atomicAdd(&cnt[(keys[idx] >> shift) & 0xFF], 1);
    }
    __syncthreads();
    hist[threadIdx.x * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void k_radix_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                uint64_t* __restrict__ kout, uint32_t* __restrict__ vout, int n,
                                int shift, const int* __restrict__ offs, int nblocks) {
    __shared__ int warp_cnt[8][256];
    __shared__ int base_cnt[256];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int w = 0; w < 8; ++w) warp_cnt[w][tid] = 0;
    base_cnt[tid] = offs[tid * nblocks + blockIdx.x];
    __syncthreads();
    const unsigned lt_mask = (1u << lane) - 1u;
    for (int round = 0; round < kRadixTile / 256; ++round) {
        const int idx = blockIdx.x * kRadixTile + round * 256 + tid;
        const bool valid = idx < n;
        uint64_t k = 0;
        uint32_t v = 0;
        int d = 256;  // sentinel digit for padding lanes
        if (valid) {
            k = kin[idx];
            v = vin[idx];
            d = static_cast<int>((k >> shift) & 0xFF);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int rank = __popc(peers & lt_mask);
        if (valid && rank == 0) warp_cnt[warp][d] = __popc(peers);
        __syncthreads();
        {   // digit `tid`: exclusive prefix over warps plus running base
            int run = base_cnt[tid];
            for (int w = 0; w < 8; ++w) {
                const int c = warp_cnt[w][tid];
                warp_cnt[w][tid] = run;
                run += c;
            }
            base_cnt[tid] = run;
        }
        __syncthreads();
        if (valid) {
            const int pos = warp_cnt[warp][d] + rank;
            kout[pos] = k;
            vout[pos] = v;
        }
        __syncthreads();
        for (int w = 0; w < 8; ++w) warp_cnt[w][tid] = 0;
        __syncthreads();
    }
}

// ---- exclusive scan (int32 sum) ------------------------------------------

__global__ void k_scan_block(const int* __restrict__ in, int* __restrict__ out, int n,
                             int* __restrict__ block_sums) {
    __shared__ int s[256];
    const int tid = threadIdx.x;
    const int base = blockIdx.x * kScanTile + tid * 8;
    int v[8];
    int sum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        v[i] = (base + i < n) ? in[base + i] : 0;
        sum += v[i];
    }
    s[tid] = sum;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        const int t = tid >= o ? s[tid - o] : 0;
        __syncthreads();
        s[tid] += t;
        __syncthreads();
    }
    int run = s[tid] - sum;  // exclusive prefix of this thread
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (base + i < n) out[base + i] = run;
        run += v[i];
    }
    if (tid == 255 && block_sums) block_sums[blockIdx.x] = s[255];
}

__global__ void k_scan_add(int* __restrict__ out, int n, const int* __restrict__ block_offs) {
    const int idx = blockIdx.x * kScanTile + threadIdx.x;
    const int add = block_offs[blockIdx.x];
    for (int i = 0; i < kScanTile; i += 256)
        if (idx + i < n) out[idx + i] += add;
}

__global__ void k_total(const int* __restrict__ in, const int* __restrict__ ex, int n,
                        int* __restrict__ total) {
    *total = n ? ex[n - 1] + in[n - 1] : 0;
}

// out[0] = max(in[0..n)), single block
__global__ void k_max(const int* __restrict__ in, int n, int* __restrict__ out) {
    __shared__ int s[256];
    int m = 0;
    for (int i = threadIdx.x; i < n; i += 256) m = max(m, in[i]);
    s[threadIdx.x] = m;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) s[threadIdx.x] = max(s[threadIdx.x], s[threadIdx.x + o]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = s[0];
}

// ---- runs / groups ---------------------------------------------------------

__device__ __forceinline__ int lower_bound_u64(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int upper_bound_u64(const uint64_t* a, int n, uint64_t x) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_runs(const uint64_t* __restrict__ skeys, const uint32_t* __restrict__ srows,
                       const uint64_t* __restrict__ words, int M, int W, int V,
                       int* __restrict__ rank_out, int* __restrict__ lead_by_row,
                       int* __restrict__ fail_head, uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const uint64_t k = skeys[i];
    const int rs = lower_bound_u64(skeys, M, k);
    const int re = upper_bound_u64(skeys, M, k);
    const int rank = i - rs;
    if (rank > 0) {  // exact check against the previous row of the run
        const uint64_t* a = words + static_cast<int64_t>(srows[i]) * W;
        const uint64_t* b = words + static_cast<int64_t>(srows[i - 1]) * W;
        for (int w = 0; w < W; ++w)
            if (a[w] != b[w]) {
                atomicOr(&flags[1], 1u);
                break;
            }
    }
    rank_out[i] = rank;
    lead_by_row[srows[i]] = (rank % V == 0) ? 1 : 0;
    const bool failing = ((re - rs) % V) != 0;
    fail_head[i] = (failing && rank == 0) ? 1 : 0;
    if (failing && rank == 0) atomicOr(&flags[2], 1u);
}

// lexicographically smallest failing class -> its smallest row
__global__ void k_fail_argmin(const int* __restrict__ fail_head, const uint32_t* __restrict__ srows,
                              const uint64_t* __restrict__ words, int M, int W,
                              uint32_t* __restrict__ fail_row) {
    __shared__ int best[1024];
    const int tid = threadIdx.x;
    auto less = [&](int a, int b) {  // rows a, b; -1 = none
        if (b < 0) return a >= 0;
        if (a < 0) return false;
        const uint64_t* x = words + static_cast<int64_t>(a) * W;
        const uint64_t* y = words + static_cast<int64_t>(b) * W;
        for (int w = 0; w < W; ++w)
            if (x[w] != y[w]) return x[w] < y[w];
        return a < b;
    };
    int mine = -1;
    for (int i = tid; i < M; i += blockDim.x)
        if (fail_head[i] && less(static_cast<int>(srows[i]), mine)) mine = static_cast<int>(srows[i]);
    best[tid] = mine;
    __syncthreads();
    for (int o = blockDim.x / 2; o; o >>= 1) {
        if (tid < o && less(best[tid + o], best[tid])) best[tid] = best[tid + o];
        __syncthreads();
    }
    if (tid == 0) *fail_row = static_cast<uint32_t>(best[0] < 0 ? 0 : best[0]);
}

__global__ void k_assign(const uint32_t* __restrict__ srows, const int* __restrict__ rank,
                         const int* __restrict__ gid_by_row, const int* __restrict__ popc, int M,
                         int V, int ktile, int32_t* __restrict__ row_indices,
                         int32_t* __restrict__ group_leader, int32_t* __restrict__ group_ncols,
                         int* __restrict__ padded) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int slot = rank[i] % V;
    const int lead_row = static_cast<int>(srows[i - slot]);
    const int g = gid_by_row[lead_row];
    // a non-conformant mask has more than M / V leaders: the asynchronous
    // converter runs on anyway (its status reports the failure), in bounds
    if (g >= M / V) return;
    row_indices[static_cast<int64_t>(g) * V + slot] = static_cast<int32_t>(srows[i]);
    if (slot == 0) {
        const int n = popc[lead_row];
        group_leader[g] = lead_row;
        group_ncols[g] = n;
        padded[g] = (n + ktile - 1) / ktile * ktile;
    }
}

// column list of group g: ascending set bits of the leader row, padded.
__global__ void k_pack_cols(const uint64_t* __restrict__ words, int W,
                            const int32_t* __restrict__ group_leader,
                            const int32_t* __restrict__ group_ptr,
                            const int32_t* __restrict__ group_ncols, int32_t* __restrict__ col_idx) {
    __shared__ int s[128];
    const int g = blockIdx.x, tid = threadIdx.x;
    const uint64_t* lw = words + static_cast<int64_t>(group_leader[g]) * W;
    const int wpt = (W + 127) / 128;
    const int w0 = tid * wpt, w1 = min(W, w0 + wpt);
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popcll(lw[w]);
    s[tid] = cnt;
    __syncthreads();
    for (int o = 1; o < 128; o <<= 1) {
        const int t = tid >= o ? s[tid - o] : 0;
        __syncthreads();
        s[tid] += t;
        __syncthreads();
    }
    int out = group_ptr[g] + s[tid] - cnt;
    for (int w = w0; w < w1; ++w) {
        uint64_t x = lw[w];
        while (x) {
            const int b = __clzll(x);  // MSB first = ascending column
            col_idx[out++] = w * 64 + b;
            x &= ~(0x8000000000000000ULL >> b);
        }
    }
    const int ng = group_ncols[g], pend = group_ptr[g + 1] - group_ptr[g];
    for (int j = ng + tid; j < pend; j += 128) col_idx[group_ptr[g] + j] = SHFLBW_PAD_COLUMN;
}

// values[(gp + j) * V + v] = round16(dense[row_v][col_j]); pad columns -> 0.
template <int DT>
__global__ void k_pack_values(const void* __restrict__ dense, int dense_dtype, int K, int V,
                              int jc, const int32_t* __restrict__ row_indices,
                              const int32_t* __restrict__ group_ptr,
                              const int32_t* __restrict__ group_ncols,
                              const int32_t* __restrict__ col_idx, void* __restrict__ values) {
    using T = typename Elem<DT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* tile = reinterpret_cast<T*>(smem_raw);  // [jc][V]
    const int g = blockIdx.y;
    const int j0 = blockIdx.x * jc;
    const int gp = group_ptr[g];
    const int padded = group_ptr[g + 1] - gp;
    if (j0 >= padded) return;
    const int ng = group_ncols[g];
    const int total = jc * V;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int v = idx / jc, jj = idx % jc;  // jj fastest: same row, ascending columns
        const int j = j0 + jj;
        float x = 0.0f;
        if (j < ng) {
            const int64_t row = row_indices[static_cast<int64_t>(g) * V + v];
            x = load_as_f32(dense, dense_dtype, row * K + col_idx[gp + j]);
        }
        tile[jj * V + v] = Elem<DT>::from_f(x);
    }
    __syncthreads();
    T* dst = static_cast<T*>(values) + static_cast<int64_t>(gp + j0) * V;
    const int lim = min(jc, padded - j0) * V;
    for (int idx = threadIdx.x; idx < lim; idx += blockDim.x) dst[idx] = tile[idx];
}

// ---- upload / download / decompress --------------------------------------

__global__ void k_upload_groups(const int32_t* __restrict__ gn, int G, int V, int K, int ktile,
                                int* __restrict__ padded, uint32_t* __restrict__ flags) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= G) return;
    const int n = gn[g];
    if (n < 0 || n > K) atomicOr(&flags[3], 1u);
    padded[g] = (n + ktile - 1) / ktile * ktile;
}

__global__ void k_check_rows(const int32_t* __restrict__ ri, int M, uint32_t* __restrict__ flags) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < M && (ri[i] < 0 || ri[i] >= M)) atomicOr(&flags[0], 1u);
}

template <int DT>
__global__ void k_upload_values(const uint32_t* __restrict__ cols_in, const float* __restrict__ vals_in,
                                const int* __restrict__ src_off, const int32_t* __restrict__ group_ptr,
                                const int32_t* __restrict__ group_ncols, int V, int K,
                                int32_t* __restrict__ col_idx, void* __restrict__ values,
                                uint32_t* __restrict__ flags) {
    using T = typename Elem<DT>::T;
    const int g = blockIdx.y;
    const int gp = group_ptr[g], padded = group_ptr[g + 1] - gp, ng = group_ncols[g];
    const int64_t so = src_off[g];
    T* dst = static_cast<T*>(values);
    const int64_t total = static_cast<int64_t>(padded) * V;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(idx / V), v = static_cast<int>(idx % V);
        const float x = j < ng ? vals_in[(so + j) * V + v] : 0.0f;
        dst[(static_cast<int64_t>(gp) + j) * V + v] = Elem<DT>::from_f(x);
        if (v == 0) {
            int32_t c = SHFLBW_PAD_COLUMN;
            if (j < ng) {
                const uint32_t cu = cols_in[so + j];
                if (cu >= static_cast<uint32_t>(K) ||
                    (j > 0 && cols_in[so + j - 1] >= cu)) atomicOr(&flags[1], 1u);
                c = static_cast<int32_t>(cu);
            }
            col_idx[gp + j] = c;
        }
    }
}

template <int DT>
__global__ void k_download_values(const int32_t* __restrict__ col_idx, const void* __restrict__ values,
                                  const int* __restrict__ dst_off, const int32_t* __restrict__ group_ptr,
                                  const int32_t* __restrict__ group_ncols, int V,
                                  uint32_t* __restrict__ cols_out, float* __restrict__ vals_out) {
    const int g = blockIdx.y;
    const int gp = group_ptr[g], ng = group_ncols[g];
    const int64_t dof = dst_off[g];
    const int64_t total = static_cast<int64_t>(ng) * V;
    const auto* src = static_cast<const typename Elem<DT>::T*>(values);
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(idx / V), v = static_cast<int>(idx % V);
        vals_out[(dof + j) * V + v] = Elem<DT>::to_f(src[(static_cast<int64_t>(gp) + j) * V + v]);
        if (v == 0) cols_out[dof + j] = static_cast<uint32_t>(col_idx[gp + j]);
    }
}

template <int DT>
__global__ void k_decompress(const int32_t* __restrict__ row_indices, const int32_t* __restrict__ group_ptr,
                             const int32_t* __restrict__ group_ncols, const int32_t* __restrict__ col_idx,
                             const void* __restrict__ values, int V, int K, float* __restrict__ dense) {
    const int g = blockIdx.y;
    const int gp = group_ptr[g], width = group_ptr[g + 1] - gp;  // pads (-1) may sit anywhere (conv order)
    const auto* src = static_cast<const typename Elem<DT>::T*>(values);
    const int64_t total = static_cast<int64_t>(width) * V;
    (void)group_ncols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(idx / V), v = static_cast<int>(idx % V);
        const int c = col_idx[gp + j];
        if (c < 0) continue;
        const int64_t row = row_indices[static_cast<int64_t>(g) * V + v];
        dense[row * K + c] = Elem<DT>::to_f(src[(static_cast<int64_t>(gp) + j) * V + v]);
    }
}

// conv_prepare: per group, count the columns of each filter column s = c % S
// (c = (ch*R + r)*S + s) and size the group for s-runs padded to quads
__global__ void k_conv_widths(const int32_t* __restrict__ group_ptr, const int32_t* __restrict__ col_idx, int S,
                              int* __restrict__ widths) {
    __shared__ int cnt[32];
    const int g = blockIdx.x;
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int j = group_ptr[g] + threadIdx.x; j < group_ptr[g + 1]; j += blockDim.x) {
        const int c = col_idx[j];
        if (c >= 0) atomicAdd(&cnt[c % S], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int w = 0;
        for (int x = 0; x < S; ++x) w += (cnt[x] + 3) / 4 * 4;
        widths[g] = (w + SHFLBW_K_TILE - 1) / SHFLBW_K_TILE * SHFLBW_K_TILE;
    }
}

// one block per group: thread 0 assigns every column its slot (s-runs in
// ascending s, ascending c within a run -- a stable partition), then the
// block copies the V values of each column
template <int DT>
__global__ void k_conv_scatter(const int32_t* __restrict__ gp_in, const int32_t* __restrict__ col_in,
                               const void* __restrict__ val_in, const int32_t* __restrict__ gp_out, int S, int V,
                               int32_t* __restrict__ col_out, void* __restrict__ val_out, int32_t* __restrict__ slot) {
    __shared__ int start[33];
    const int g = blockIdx.x;
    const int b0 = gp_in[g], b1 = gp_in[g + 1], o0 = gp_out[g];
    if (threadIdx.x == 0) {
        int cnt[32];
        for (int x = 0; x < S; ++x) cnt[x] = 0;
        for (int j = b0; j < b1; ++j)
            if (col_in[j] >= 0) ++cnt[col_in[j] % S];
        start[0] = 0;
        for (int x = 0; x < S; ++x) start[x + 1] = start[x] + (cnt[x] + 3) / 4 * 4;
        for (int x = 0; x < S; ++x) cnt[x] = 0;
        for (int j = b0; j < b1; ++j) {
            const int c = col_in[j];
            if (c < 0) {
                slot[j] = -1;
                continue;
            }
            const int x = c % S;
            const int p = o0 + start[x] + cnt[x]++;
            slot[j] = p;
            col_out[p] = c;
        }
    }
    __syncthreads();
    using T = typename Elem<DT>::T;
    const T* src = static_cast<const T*>(val_in);
    T* dst = static_cast<T*>(val_out);
    const int64_t total = static_cast<int64_t>(b1 - b0) * V;
    for (int64_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const int j = b0 + static_cast<int>(idx / V), v = static_cast<int>(idx % V);
        const int p = slot[j];
        if (p >= 0) dst[static_cast<int64_t>(p) * V + v] = src[static_cast<int64_t>(j) * V + v];
    }
}

__global__ void k_convert(const void* __restrict__ src, int sdt, void* __restrict__ dst, int ddt,
                          int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        store_from_f32(dst, ddt, i, load_as_f32(src, sdt, i));
}

// pitched copy-convert: one CTA row per matrix row (grid y), threads over columns
__global__ void k_convert_2d(const void* __restrict__ src, int sdt, int64_t ld_src, void* __restrict__ dst,
                             int ddt, int64_t ld_dst, int64_t rows, int64_t cols) {
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols;
             c += static_cast<int64_t>(gridDim.x) * blockDim.x)
            store_from_f32(dst, ddt, r * ld_dst + c, load_as_f32(src, sdt, r * ld_src + c));
}

// *flag |= 1 if any K block of any group is one contiguous run of 64 columns
// (block-wise patterns: the SpMM then loads those blocks as TMA 2D tiles)
__global__ void k_contig_blocks(const int32_t* __restrict__ group_ptr, const int32_t* __restrict__ col_idx,
                                uint32_t* __restrict__ flag) {
    const int g = blockIdx.x;
    for (int j = group_ptr[g] + threadIdx.x * SHFLBW_K_TILE; j < group_ptr[g + 1]; j += blockDim.x * SHFLBW_K_TILE) {
        const int first = col_idx[j], last = col_idx[j + SHFLBW_K_TILE - 1];
        if (first >= 0 && last - first == SHFLBW_K_TILE - 1) {
            atomicOr(flag, 1u);
            return;
        }
    }
}

// asynchronous converter status: [0] status code, [1] fail_row, [2] total
// columns (group_ptr[G]), [3] widest group (padded)
__global__ void k_status(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ fail_row,
                         const int32_t* __restrict__ total, const int* __restrict__ maxp,
                         int32_t* __restrict__ status) {
    const int code = flags[0] ? SHFLBW_BAD_PARAMS
                              : (flags[1] ? SHFLBW_CUDA_ERROR : (flags[2] ? SHFLBW_NONCONFORMANT_MASK : SHFLBW_OK));
    status[0] = code;
    status[1] = code == SHFLBW_NONCONFORMANT_MASK ? static_cast<int32_t>(*fail_row) : 0;
    status[2] = *total;
    status[3] = *maxp;
}

// ---- hash planner (M <= kPlanMax): class check, one-CTA plan, fused pack ----

// K2: one warp per row.  rep = the class's smallest row (the table slot's
// atomicMin); a row whose words differ from its representative's shares a
// slot with another class (a 64-bit hash collision): flags[1].
__global__ void k_class_check(const uint64_t* __restrict__ words, int M, int W, ClassTable tab,
                              uint32_t* __restrict__ rep_out, uint32_t* __restrict__ csize_out,
                              uint32_t* __restrict__ flags) {
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (r >= M) return;
    const uint32_t sl = tab.slot[r];
    const uint32_t rep = tab.minrow[sl];
    if (rep != static_cast<uint32_t>(r)) {
        bool diff = false;
        const uint64_t* a = words + static_cast<int64_t>(r) * W;
        const uint64_t* b = words + static_cast<int64_t>(rep) * W;
        for (int w = lane; w < W; w += 32) diff |= a[w] != b[w];
        if (__any_sync(0xffffffffu, diff) && lane == 0) atomicOr(&flags[1], 1u);
    }
    if (lane == 0) {
        rep_out[r] = rep;
        csize_out[r] = tab.cnt[sl] + 1u;
    }
}

constexpr int kPlanThreads = 1024;
constexpr int kPlanMax = 32768;                      // rows: 16-bit row ids, <= 32 chunks of 1024
constexpr int kPlanSmall = 4096;                     // above: chunked ranks (k_chunk_rank) instead of the CTA sort

// exclusive scan of one int per thread over a 1024-thread block; *total =
// the block sum (every thread).  `tmp` holds 33 ints.
__device__ __forceinline__ int block_scan_1024(int x, int* tmp, int* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) tmp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int v = tmp[lane];
        int wi = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        tmp[lane] = wi - v;  // exclusive warp offsets
        if (lane == 31) tmp[32] = wi;
    }
    __syncthreads();
    const int r = tmp[warp] + incl - x;
    *total = tmp[32];
    __syncthreads();
    return r;
}

// lanes whose `nb`-bit digit d equals this lane's (and whose `valid` agrees):
// ballots per bit instead of MATCH.ANY, which in k_plan stalled every warp for
// ~40 SM cycles per call (60 % of the large-FFN plan time)
__device__ __forceinline__ unsigned match_digit(uint32_t d, int nb, bool valid) {
    const unsigned vb = __ballot_sync(0xffffffffu, valid);
    unsigned m = valid ? vb : ~vb;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        if (b < nb) {
            const bool bit = (d >> b) & 1u;
            const unsigned bal = __ballot_sync(0xffffffffu, bit);
            m &= bit ? bal : ~bal;
        }
    }
    return m;
}

__device__ __noinline__ bool row_less(const uint64_t* words, int W, int a, int b) {  // -1 = none
    if (b < 0) return a >= 0;
    if (a < 0) return false;
    const uint64_t* x = words + static_cast<int64_t>(a) * W;
    const uint64_t* y = words + static_cast<int64_t>(b) * W;
    for (int w = 0; w < W; ++w)
        if (x[w] != y[w]) return x[w] < y[w];
    return a < b;
}

// dst[i] = src[i] (u32 -> u16), i < n, by a 1024-thread block: 16-byte loads,
// four per thread in flight
__device__ __forceinline__ void load_u16(const uint32_t* __restrict__ src, int n, uint16_t* dst) {
    const int tid = threadIdx.x;
    if ((n & 3) == 0) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll 1
        for (int i4 = tid; i4 < n / 4; i4 += 4 * kPlanThreads) {
            uint4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i4 + u * kPlanThreads < n / 4) q[u] = s4[i4 + u * kPlanThreads];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = 4 * (i4 + u * kPlanThreads);
                if (i < n) {
                    dst[i] = static_cast<uint16_t>(q[u].x);
                    dst[i + 1] = static_cast<uint16_t>(q[u].y);
                    dst[i + 2] = static_cast<uint16_t>(q[u].z);
                    dst[i + 3] = static_cast<uint16_t>(q[u].w);
                }
            }
        }
    } else {
        for (int i = tid; i < n; i += kPlanThreads) dst[i] = static_cast<uint16_t>(src[i]);
    }
}

// Exclusive scan over i < n of val(i) in index order, out(i, prefix) per i;
// each warp walks one contiguous segment 32 consecutive indices at a time
// (thread-contiguous ranges put the lanes of a warp 2*PT bytes apart in a
// 16-bit array: 8-way bank conflicts at PT = 16).  Returns the total.
template <class Val, class Out>
__device__ __forceinline__ int block_scan_rows(int n, Val val, Out out, int* tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = (((n + 31) >> 5) + 31) & ~31;
    const int b0 = warp * S, b1 = min(b0 + S, n);
    int sum = 0;
    for (int i = b0 + lane; i < b1; i += 32) sum += val(i);
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) tmp[warp] = sum;
    __syncthreads();
    if (warp == 0) {
        const int v = tmp[lane];
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        tmp[lane] = incl - v;
        if (lane == 31) tmp[32] = incl;
    }
    __syncthreads();
    int carry = tmp[warp];
    for (int base = b0; base < b1; base += 32) {
        const int i = base + lane;
        const int v = i < b1 ? val(i) : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (i < b1) out(i, carry + incl - v);
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    const int total = tmp[32];
    __syncthreads();
    return total;
}

// Stable LSD sort (8-bit digits) of the n element ids in `a` by key[id]
// (16-bit), per-warp digit counts and ballot ranks; 1024 threads; returns the
// buffer (a or b) holding the sorted ids.
__device__ __forceinline__ uint16_t* block_sort16(const uint16_t* key, uint16_t* a, uint16_t* b, int n, int bits,
                                                  uint16_t* wcnt, int* tmp) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int CH = (((n + 31) >> 5) + 31) & ~31;  // positions per warp (whole rounds)
    const int p0 = warp * CH, p1 = min(p0 + CH, n);
    const unsigned lt = (1u << lane) - 1u;
    uint16_t* src = a;
    uint16_t* dst = b;
    for (int sh = 0; sh < bits; sh += 8) {
        const int nb = min(8, bits - sh);
        for (int i = tid; i < 32 * 256; i += kPlanThreads) wcnt[i] = 0;
        __syncthreads();
        for (int base = p0; base < p1; base += 32) {
            const int i = base + lane;
            const bool valid = i < p1;
            const uint32_t d = valid ? (key[src[i]] >> sh) & 255u : 0u;
            const unsigned peers = match_digit(d, nb, valid);
            if (valid && (peers & lt) == 0) wcnt[warp * 256 + d] += static_cast<uint16_t>(__popc(peers));
        }
        __syncthreads();
        {   // digit-major exclusive offsets: (digit, warp)
            int tot = 0;
            if (tid < 256)
                for (int w = 0; w < 32; ++w) tot += wcnt[w * 256 + tid];
            int all;
            int run = block_scan_1024(tid < 256 ? tot : 0, tmp, &all);
            if (tid < 256)
                for (int w = 0; w < 32; ++w) {
                    const int c = wcnt[w * 256 + tid];
                    wcnt[w * 256 + tid] = static_cast<uint16_t>(run);
                    run += c;
                }
        }
        __syncthreads();
        for (int base = p0; base < p1; base += 32) {
            const int i = base + lane;
            const bool valid = i < p1;
            const uint16_t row = valid ? src[i] : 0;
            const uint32_t d = valid ? (key[row] >> sh) & 255u : 0u;
            const unsigned peers = match_digit(d, nb, valid);
            if (valid) dst[wcnt[warp * 256 + d] + __popc(peers & lt)] = row;
            __syncwarp();
            if (valid && (peers & lt) == 0) wcnt[warp * 256 + d] += static_cast<uint16_t>(__popc(peers));
            __syncwarp();
        }
        __syncthreads();
        uint16_t* t = src;
        src = dst;
        dst = t;
    }
    return src;
}

// K3a (M > kPlanSmall): one CTA per 1024-row chunk sorts its rows by
// representative; rank of each row among its class's rows in the chunk, and
// the class's row count in the chunk: cnt[chunk][rep] (zero elsewhere).
__global__ void __launch_bounds__(kPlanThreads, 1)
    k_chunk_rank(const uint32_t* __restrict__ rep_by_row, const uint32_t* __restrict__ csize, int M, int V,
                 uint16_t* __restrict__ local_rank, uint16_t* __restrict__ cnt, uint16_t* __restrict__ seg_local,
                 int* __restrict__ chunk_seg, uint32_t* __restrict__ flags) {
    __shared__ uint16_t key[kPlanThreads], a[kPlanThreads], b[kPlanThreads];
    __shared__ uint16_t wcnt[32 * 256];
    __shared__ int tmp[33];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int r0 = blockIdx.x * kPlanThreads;
    const int n = min(kPlanThreads, M - r0);
    uint16_t* crow = cnt + static_cast<int64_t>(blockIdx.x) * M;
    for (int i = tid; i < M; i += kPlanThreads) crow[i] = 0;
    int cs = 0;
    bool isrep = false;
    if (tid < n) {
        const uint32_t rp = rep_by_row[r0 + tid];
        key[tid] = static_cast<uint16_t>(rp);
        isrep = rp == static_cast<uint32_t>(r0 + tid);
        if (isrep) {
            cs = static_cast<int>(csize[r0 + tid]);
            if (cs % V != 0) atomicOr(&flags[2], 1u);  // a failing class
        }
    }
    a[tid] = static_cast<uint16_t>(tid);
    {   // class segments start at the exclusive scan, in row order, of the
        // representatives' class sizes: this chunk's part
        int total;
        const int ex = block_scan_1024(cs, tmp, &total);
        if (isrep) seg_local[r0 + tid] = static_cast<uint16_t>(ex);
        if (tid == 0) chunk_seg[blockIdx.x] = total;
    }
    const uint16_t* srt = block_sort16(key, a, b, n, 32 - __clz(M - 1), wcnt, tmp);
    const int i = tid;
    int k = -1, head = -1;
    if (i < n) {
        k = key[srt[i]];
        if (i == 0 || key[srt[i - 1]] != k) head = i;
    }
    int start = head;  // inclusive max-scan: the run's first position
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, start, o);
        if (lane >= o) start = max(start, t);
    }
    if (lane == 31) tmp[warp] = start;
    __syncthreads();
    if (warp == 0) {
        int wv = tmp[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wv, o);
            if (lane >= o) wv = max(wv, t);
        }
        tmp[lane] = wv;
    }
    __syncthreads();
    if (warp > 0) start = max(start, tmp[warp - 1]);
    if (i < n) {
        local_rank[r0 + srt[i]] = static_cast<uint16_t>(i - start);
        if (i == n - 1 || key[srt[i + 1]] != k) crow[k] = static_cast<uint16_t>(i - start + 1);
    }
}

// K3b: exclusive prefix of each class's per-chunk counts over the chunks
// (in place), one thread per representative
__global__ void k_chunk_prefix(const uint32_t* __restrict__ rep_by_row, int M, int nchunks,
                               uint16_t* __restrict__ cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= M || rep_by_row[r] != static_cast<uint32_t>(r)) return;
    int run = 0;
    for (int c0 = 0; c0 < nchunks; c0 += 8) {
        uint16_t t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = c0 + u < nchunks ? cnt[static_cast<int64_t>(c0 + u) * M + r] : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c0 + u < nchunks) {
                cnt[static_cast<int64_t>(c0 + u) * M + r] = static_cast<uint16_t>(run);
                run += t[u];
            }
    }
}

// exclusive scan of v[0..n) (n <= 32) into out[0..n) by warp 0 (smem)
__device__ __forceinline__ void warp0_scan_small(const int* __restrict__ v, int n, int* out) {
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 32) {
        const int x = lane < n ? v[lane] : 0;
        int incl = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        out[lane] = incl - x;
    }
    __syncthreads();
}

// K3c (chunked planner): every row's rank in its class (earlier chunks +
// this chunk) and its position in the (representative, row) order -- the
// class's segment start + rank; leader flags (rank % V == 0) numbered within
// the chunk in row order.  Also clears this chunk's share of the outputs, so
// a non-conformant mask leaves every slot defined.
__global__ void __launch_bounds__(kPlanThreads, 1)
    k_chunk_place(const uint32_t* __restrict__ rep_by_row, const uint16_t* __restrict__ local_rank,
                  const uint16_t* __restrict__ cnt, const uint16_t* __restrict__ seg_local,
                  const int* __restrict__ chunk_seg, int M, int V, int nchunks, uint16_t* __restrict__ srt,
                  uint16_t* __restrict__ rank_pos, uint16_t* __restrict__ gid_local, int* __restrict__ chunk_lead,
                  int32_t* __restrict__ row_indices, int32_t* __restrict__ group_leader,
                  int32_t* __restrict__ group_ncols) {
    __shared__ int seg_off[32];
    __shared__ int tmp[33];
    const int tid = threadIdx.x;
    const int r0 = blockIdx.x * kPlanThreads;
    const int r = r0 + tid;
    const int G = M / V;
    warp0_scan_small(chunk_seg, nchunks, seg_off);
    bool lead = false;
    if (r < M) {
        const int rp = static_cast<int>(rep_by_row[r]);
        const int rank = cnt[static_cast<int64_t>(r >> 10) * M + rp] + local_rank[r];
        const int pos = seg_off[rp >> 10] + seg_local[rp] + rank;
        srt[pos] = static_cast<uint16_t>(r);
        rank_pos[pos] = static_cast<uint16_t>(rank);
        lead = rank % V == 0;
        row_indices[r] = 0;
    }
    const int GB = (G + nchunks - 1) / nchunks;
    for (int g = blockIdx.x * GB + tid; g < min(G, (blockIdx.x + 1) * GB); g += kPlanThreads)
        group_leader[g] = group_ncols[g] = 0;
    int total;
    const int ex = block_scan_1024(lead ? 1 : 0, tmp, &total);
    if (lead) gid_local[r] = static_cast<uint16_t>(ex);
    if (tid == 0) chunk_lead[blockIdx.x] = total;
}

// K3d (chunked planner): sorted positions i of this chunk -> row_indices[g *
// V + slot]; g = the leader's group number (chunks before it + its number in
// its chunk); leaders also write group_leader / n_g.
__global__ void __launch_bounds__(kPlanThreads, 1)
    k_chunk_assign(const uint16_t* __restrict__ srt, const uint16_t* __restrict__ rank_pos,
                   const uint16_t* __restrict__ gid_local, const int* __restrict__ chunk_lead,
                   const int* __restrict__ popc, int M, int V, int nchunks, int32_t* __restrict__ row_indices,
                   int32_t* __restrict__ group_leader, int32_t* __restrict__ group_ncols) {
    __shared__ int lead_off[32];
    warp0_scan_small(chunk_lead, nchunks, lead_off);
    const int i = blockIdx.x * kPlanThreads + threadIdx.x;
    if (i >= M) return;
    const int G = M / V;
    const int slot = rank_pos[i] % V;
    const int lead_row = srt[i - slot];
    const int g = lead_off[lead_row >> 10] + gid_local[lead_row];
    if (g < G) {
        row_indices[static_cast<int64_t>(g) * V + slot] = srt[i];
        if (slot == 0) {
            group_leader[g] = lead_row;
            group_ncols[g] = popc[lead_row];
        }
    }
}

// K3e (chunked planner, one CTA): group_ptr = exclusive scan of
// roundup(n_g, ktile), widest group, status; the lexicographically smallest
// failing class's smallest row when a chunk flagged one (flags[2]).
// row_indices == nullptr: validation only.
__global__ void __launch_bounds__(kPlanThreads, 1)
    k_plan_finish(const uint32_t* __restrict__ rep_by_row, const uint32_t* __restrict__ csize,
                  const uint64_t* __restrict__ words, int M, int W, int V, int ktile,
                  const uint32_t* __restrict__ flags, const int32_t* __restrict__ row_indices,
                  const int32_t* __restrict__ group_ncols, int32_t* __restrict__ group_ptr,
                  int32_t* __restrict__ status) {
    __shared__ int tmp[33];
    __shared__ int best_s[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool anyfail = flags[2] != 0;
    int best = -1;
    if (anyfail) {
        for (int r = tid; r < M; r += kPlanThreads)
            if (rep_by_row[r] == static_cast<uint32_t>(r) && csize[r] % static_cast<uint32_t>(V) != 0 &&
                row_less(words, W, r, best))
                best = r;
#pragma unroll 1
        for (int o = 16; o; o >>= 1) {
            const int other = __shfl_down_sync(0xffffffffu, best, o);
            if (lane < o && row_less(words, W, other, best)) best = other;
        }
        if (lane == 0) best_s[warp] = best;
        __syncthreads();
        if (warp == 0) {
            best = best_s[lane];
#pragma unroll 1
            for (int o = 16; o; o >>= 1) {
                const int other = __shfl_down_sync(0xffffffffu, best, o);
                if (lane < o && row_less(words, W, other, best)) best = other;
            }
            if (lane == 0) best_s[0] = best;
        }
        __syncthreads();
        best = best_s[0];
    }
    const int code = flags[0] ? SHFLBW_BAD_PARAMS
                              : (flags[1] ? SHFLBW_CUDA_ERROR : (anyfail ? SHFLBW_NONCONFORMANT_MASK : SHFLBW_OK));
    if (!row_indices) {
        if (tid == 0) {
            status[0] = code;
            status[1] = anyfail ? best : 0;
            status[2] = status[3] = 0;
        }
        return;
    }
    const int G = M / V;
    const int PG = (G + kPlanThreads - 1) / kPlanThreads;
    const int g0 = min(tid * PG, G), g1 = min(g0 + PG, G);
    int sum = 0, mx = 0;
    for (int g = g0; g < g1; ++g) {
        const int pd = (group_ncols[g] + ktile - 1) / ktile * ktile;
        sum += pd;
        mx = max(mx, pd);
    }
    int total;
    int run = block_scan_1024(sum, tmp, &total);
    for (int g = g0; g < g1; ++g) {
        group_ptr[g] = run;
        run += (group_ncols[g] + ktile - 1) / ktile * ktile;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) best_s[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        int m = 0;
        for (int w = 0; w < 32; ++w) m = max(m, best_s[w]);
        group_ptr[G] = total;
        status[0] = code;
        status[1] = anyfail ? best : 0;
        status[2] = total;
        status[3] = m;
    }
}

// K3, one CTA: (1) stable LSD sort of the rows by representative in shared
// memory (8-bit digits, per-warp digit counts, match_any ranks) -- classes
// become runs of ascending rows, like the reference's std::map buckets
// (src/formats.cpp:40-46); (2) rank = position - position of the run's
// representative; leaders = ranks that are multiples of V; (3) exclusive scan
// of the leader flags in row order = group number by first row (the
// reference's group order, src/formats.cpp:160-170); (4) failing classes
// (size % V != 0): lexicographically smallest one's smallest row
// (src/formats.cpp:113-125); (5) row_indices / leaders / n_g; (6) group_ptr
// = exclusive scan of roundup(n_g, ktile), widest group; status.
// row_indices == nullptr: validation only (status alone).
__global__ void __launch_bounds__(kPlanThreads, 1)
    k_plan(const uint32_t* __restrict__ rep_by_row, const uint32_t* __restrict__ csize, const int* __restrict__ popc,
           const uint64_t* __restrict__ words, int M, int W, int V, int ktile, const uint32_t* __restrict__ flags,
           int32_t* __restrict__ row_indices, int32_t* __restrict__ group_leader, int32_t* __restrict__ group_ncols,
           int32_t* __restrict__ group_ptr, int32_t* __restrict__ status) {
    extern __shared__ __align__(16) unsigned char sm_plan[];
    const int Mp = (M + 7) & ~7;
    uint16_t* rep = reinterpret_cast<uint16_t*>(sm_plan);  // rep by row, later rank by sorted position
    uint16_t* bufa = rep + Mp;
    uint16_t* bufb = bufa + Mp;
    uint16_t* wcnt = bufb + Mp;  // [32 warps][256 digits]
    __shared__ int tmp[33];
    __shared__ int best_s[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = M / V;
    load_u16(rep_by_row, M, rep);  // representatives
    for (int i = tid; i < M; i += kPlanThreads) bufa[i] = static_cast<uint16_t>(i);
    __syncthreads();
    // (1) rows by representative: sorted here (M <= kPlanSmall), else placed
    // from the per-chunk ranks of k_chunk_rank + k_chunk_prefix.
    // (2) rank of each sorted position within its class (dst).
    // Loops are not unrolled: a one-CTA kernel pays every instruction-cache
    // miss (fully unrolled, 45 % of the samples were no_instruction stalls).
    const int PT = (M + kPlanThreads - 1) / kPlanThreads;
    const int q0 = min(tid * PT, M), q1 = min(q0 + PT, M);
    int best = -1;
    bool anyfail = false;
    uint16_t* src;
    uint16_t* dst;
    {
        src = block_sort16(rep, bufa, bufb, M, M > 1 ? 32 - __clz(M - 1) : 0, wcnt, tmp);
        dst = src == bufa ? bufb : bufa;
        // a run (class) starts where the row is its own representative; rank
        // = position - run start (an exclusive max-scan carries the start
        // across the thread-contiguous ranges)
        int last = -1;
#pragma unroll 1
        for (int i = q0; i < q1; ++i) {
            const int row = src[i];
            if (rep[row] == row) {
                last = i;
                if (csize[row] % static_cast<uint32_t>(V) != 0) {
                    anyfail = true;
                    if (row_less(words, W, row, best)) best = row;
                }
            }
        }
        int carry = last;  // inclusive max over threads <= tid, then shifted
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, carry, o);
            if (lane >= o) carry = max(carry, t);
        }
        if (lane == 31) tmp[warp] = carry;
        __syncthreads();
        if (warp == 0) {
            int wv = tmp[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, wv, o);
                if (lane >= o) wv = max(wv, t);
            }
            tmp[lane] = wv;
        }
        __syncthreads();
        int excl = __shfl_up_sync(0xffffffffu, carry, 1);
        if (lane == 0) excl = -1;
        if (warp > 0) excl = max(excl, tmp[warp - 1]);
        int cur = excl;
#pragma unroll 1
        for (int i = q0; i < q1; ++i) {
            const int row = src[i];
            if (rep[row] == row) cur = i;
            dst[i] = static_cast<uint16_t>(i - cur);
        }
    }
    __syncthreads();
    const bool vpow2 = (V & (V - 1)) == 0;
    auto modV = [&](int x) { return vpow2 ? (x & (V - 1)) : x % V; };
    for (int i = tid; i < M; i += kPlanThreads) rep[src[i]] = modV(dst[i]) == 0 ? 1 : 0;  // leader flags by row
    anyfail = __syncthreads_or(anyfail);
    if (anyfail) {  // (4) lexicographic argmin over the failing classes' representatives
#pragma unroll 1
        for (int o = 16; o; o >>= 1) {
            const int other = __shfl_down_sync(0xffffffffu, best, o);
            if (lane < o && row_less(words, W, other, best)) best = other;
        }
        if (lane == 0) best_s[warp] = best;
        __syncthreads();
        if (warp == 0) {
            best = best_s[lane];
#pragma unroll 1
            for (int o = 16; o; o >>= 1) {
                const int other = __shfl_down_sync(0xffffffffu, best, o);
                if (lane < o && row_less(words, W, other, best)) best = other;
            }
            if (lane == 0) best_s[0] = best;
        }
        __syncthreads();
        best = best_s[0];
    }
    // (3) group number of each leader row: exclusive scan in row order
    const int nlead = block_scan_rows(
        M, [&](int r) { return static_cast<int>(rep[r]); },
        [&](int r, int x) { rep[r] = static_cast<uint16_t>(x); }, tmp);
    int code = flags[0] ? SHFLBW_BAD_PARAMS
                        : (flags[1] ? SHFLBW_CUDA_ERROR : (anyfail ? SHFLBW_NONCONFORMANT_MASK : SHFLBW_OK));
    if (!row_indices) {
        if (tid == 0) {
            status[0] = code;
            status[1] = anyfail ? best : 0;
            status[2] = status[3] = 0;
        }
        return;
    }
    // n_g is also kept in shared memory (free by now: the digit counters, or
    // the segment starts) when it fits, so (6) does not re-read it through L2
    int* ncs = reinterpret_cast<int*>(wcnt);
    const bool ncs_ok = G <= 32 * 256 / 2;
    if (nlead != G) {  // non-conformant: every output slot defined
        for (int i = tid; i < M; i += kPlanThreads) row_indices[i] = 0;
        for (int g = tid; g < G; g += kPlanThreads) {
            group_leader[g] = group_ncols[g] = 0;
            if (ncs_ok) ncs[g] = 0;
        }
        __syncthreads();
    }
    // (5) assignment
    for (int i = tid; i < M; i += kPlanThreads) {
        const int slot = modV(dst[i]);
        const int lead_row = src[i - slot];
        const int g = rep[lead_row];
        if (g < G) {
            row_indices[static_cast<int64_t>(g) * V + slot] = src[i];
            if (slot == 0) {
                const int n = popc[lead_row];
                group_leader[g] = lead_row;
                group_ncols[g] = n;
                if (ncs_ok) ncs[g] = n;
            }
        }
    }
    __syncthreads();
    // (6) group_ptr, widest group
    const int PG = (G + kPlanThreads - 1) / kPlanThreads;
    const int g0 = min(tid * PG, G), g1 = min(g0 + PG, G);
    int sum = 0, mx = 0;
    for (int g = g0; g < g1; ++g) {
        const int pd = ((ncs_ok ? ncs[g] : group_ncols[g]) + ktile - 1) / ktile * ktile;
        sum += pd;
        mx = max(mx, pd);
    }
    int total;
    int run = block_scan_1024(sum, tmp, &total);
    for (int g = g0; g < g1; ++g) {
        group_ptr[g] = run;
        run += ((ncs_ok ? ncs[g] : group_ncols[g]) + ktile - 1) / ktile * ktile;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) best_s[warp] = mx;
    __syncthreads();
    if (tid == 0) {
        int m = 0;
        for (int w = 0; w < 32; ++w) m = max(m, best_s[w]);
        group_ptr[G] = total;
        status[0] = code;
        status[1] = anyfail ? best : 0;
        status[2] = total;
        status[3] = m;
    }
}

// K4: one CTA per (group, 64-column K block): the block's column list from
// the leader row's words (prefix popcount, replaces k_pack_cols), the group's
// V rows gathered at those columns (independent loads, 16 per thread in
// flight), rounded to the value type and transposed through a bank-padded
// shared tile, written as one contiguous V x 64 slab.  Also flags block-wise
// K blocks (64 consecutive columns) in *contig.
template <int DT, int DIN>
__global__ void __launch_bounds__(256, 8) k_pack_group(const void* __restrict__ dense, int K, int V, int W,
                                                    const uint64_t* __restrict__ words,
                                                    const int32_t* __restrict__ group_leader,
                                                    const int32_t* __restrict__ group_ptr,
                                                    const int32_t* __restrict__ group_ncols,
                                                    const int32_t* __restrict__ row_indices,
                                                    int32_t* __restrict__ col_idx, void* __restrict__ values,
                                                    uint32_t* __restrict__ contig) {
    using T = typename Elem<DT>::T;
    using TI = typename Elem<DIN>::T;
    constexpr int JC = SHFLBW_K_TILE;
    constexpr int kWCap = 1024;  // leader words held as prefix counts (K <= 65536)
    extern __shared__ __align__(16) unsigned char sm_pack[];
    __shared__ int cols_s[JC];
    __shared__ int tmp[8];
    __shared__ int wpre[kWCap];
    const int SV = sizeof(T) == 2 ? V + 2 : V + 1;  // odd bank stride between columns
    T* stage = reinterpret_cast<T*>(sm_pack);       // [JC][SV]
    int* rows_s = reinterpret_cast<int*>(sm_pack + ((static_cast<size_t>(JC) * SV * sizeof(T) + 15) & ~size_t(15)));
    const int g = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gp = group_ptr[g];
    const int padded = group_ptr[g + 1] - gp;
    const int j0 = blockIdx.x * JC;
    if (j0 >= padded) return;
    const int ng = group_ncols[g];
    const int nvalid = max(0, min(JC, ng - j0));
    for (int v = tid; v < V; v += 256) rows_s[v] = row_indices[static_cast<int64_t>(g) * V + v];
    if (nvalid > 0) {
        // exclusive prefix popcount of the leader row's words, then thread t
        // < nvalid selects set bit j0 + t: binary search over the prefix, then
        // the bit inside the word (column 0 = MSB)
        const uint64_t* lw = words + static_cast<int64_t>(group_leader[g]) * W;
        const int wpt = (W + 255) / 256;
        const int w0 = min(tid * wpt, W), w1 = min(w0 + wpt, W);
        int cnt = 0;
        for (int w = w0; w < w1; ++w) cnt += __popcll(lw[w]);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) tmp[warp] = incl;
        __syncthreads();
        int r = incl - cnt;
        for (int w = 0; w < warp; ++w) r += tmp[w];
        if (W <= kWCap) {
            for (int w = w0; w < w1; ++w) {
                wpre[w] = r;
                r += __popcll(lw[w]);
            }
            __syncthreads();
            if (tid < nvalid) {
                const int target = j0 + tid;
                int lo = 0, hi = W - 1;  // last word whose prefix <= target
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (wpre[mid] <= target) lo = mid;
                    else hi = mid - 1;
                }
                const uint64_t x = lw[lo];
                int n = target - wpre[lo];
                const uint32_t xh = static_cast<uint32_t>(x >> 32), xl = static_cast<uint32_t>(x);
                const int ph = __popc(xh);
                const int b = n < ph ? static_cast<int>(__fns(__brev(xh), 0, n + 1))
                                     : 32 + static_cast<int>(__fns(__brev(xl), 0, n - ph + 1));
                cols_s[tid] = lo * 64 + b;
            }
        } else if (r < j0 + nvalid && r + cnt > j0) {
            for (int w = w0; w < w1 && r < j0 + nvalid; ++w) {
                uint64_t x = lw[w];
                const int pc = __popcll(x);
                if (r + pc <= j0) {
                    r += pc;
                    continue;
                }
                while (x && r < j0 + nvalid) {
                    const int b = __clzll(x);
                    if (r >= j0) cols_s[r - j0] = w * 64 + b;
                    ++r;
                    x &= ~(0x8000000000000000ULL >> b);
                }
            }
        }
    }
    __syncthreads();
    if (tid < JC) col_idx[gp + j0 + tid] = tid < nvalid ? cols_s[tid] : SHFLBW_PAD_COLUMN;
    if (contig && tid == 0 && nvalid == JC && cols_s[JC - 1] - cols_s[0] == JC - 1) atomicOr(contig, 1u);
    // gather: thread = (column jj = tid % 64, rows v = tid / 64 + 4u): a warp
    // reads 32 kept columns of one row; all of a thread's loads in flight
    const TI* src = static_cast<const TI*>(dense);
    const int jj = tid & (JC - 1), vq = tid >> 6;
    const bool live = jj < nvalid;
    const int col = live ? cols_s[jj] : 0;
    for (int v0 = 0; v0 < V; v0 += 32) {
        if constexpr (DT == DIN) {  // same type: the values move as raw bits (no convert pair)
            T x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + 4 * u + vq;
                x[u] = Elem<DT>::from_f(0.0f);
                if (live && v < V) x[u] = src[static_cast<int64_t>(rows_s[v]) * K + col];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + 4 * u + vq;
                if (v < V) stage[jj * SV + v] = x[u];
            }
        } else {
            float x[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + 4 * u + vq;
                x[u] = 0.0f;
                if (live && v < V) x[u] = Elem<DIN>::to_f(src[static_cast<int64_t>(rows_s[v]) * K + col]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int v = v0 + 4 * u + vq;
                if (v < V) stage[jj * SV + v] = Elem<DT>::from_f(x[u]);
            }
        }
    }
    __syncthreads();
    // contiguous V x 64 slab: values[(gp + j0 + jj) * V + v]
    const int total = V * JC;
    T* out = static_cast<T*>(values) + static_cast<int64_t>(gp + j0) * V;
    if (sizeof(T) == 2 && (V & 1) == 0) {
        uint32_t* out2 = reinterpret_cast<uint32_t*>(out);
        for (int e = tid; e < total / 2; e += 256) {
            const int jj = (2 * e) / V, v = (2 * e) % V;
            out2[e] = *reinterpret_cast<const uint32_t*>(stage + jj * SV + v);
        }
    } else {
        for (int e = tid; e < total; e += 256) out[e] = stage[(e / V) * SV + e % V];
    }
}

// ---- host helpers ------------------------------------------------------------

}  // namespace

// The converter's scratch and output matrices come from the device's default
// stream-ordered pool; with its default release threshold (0) every stream
// synchronisation handed the memory back to the driver and the next call paid
// for mapping it again (0.4 -> 2.4 ms swings per compress).  Keep it.
void retain_pool() {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    const uint64_t bit = dev < 64 ? (1ull << dev) : 0;
    if (bit && (done.load(std::memory_order_relaxed) & bit)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (bit) done.fetch_or(bit, std::memory_order_relaxed);
}

namespace {

struct DevBuf {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        s = st;
        retain_pool();
        return cudaMallocAsync(&p, bytes ? bytes : 16, st);
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

int grid_for(int64_t n, int per_block) {
    const int64_t b = (n + per_block - 1) / per_block;
    return static_cast<int>(b < 1 ? 1 : (b > 1048576 ? 1048576 : b));
}

}  // namespace

// exclusive scan, out may alias nothing; *total_dev (optional) = sum
int scan_exclusive(const int* in, int* out, int n, int* total_dev, cudaStream_t s) {
    if (n <= 0) {
        if (total_dev) SBW_CUDA(cudaMemsetAsync(total_dev, 0, sizeof(int), s));
        return SHFLBW_OK;
    }
    const int nb = (n + kScanTile - 1) / kScanTile;
    if (nb == 1) {
        k_scan_block<<<1, 256, 0, s>>>(in, out, n, nullptr);
        SBW_LAUNCHED("k_scan_block");
    } else {
        DevBuf sums, offs;
        SBW_CUDA(sums.alloc(sizeof(int) * nb, s));
        SBW_CUDA(offs.alloc(sizeof(int) * nb, s));
        k_scan_block<<<nb, 256, 0, s>>>(in, out, n, sums.as<int>());
        SBW_LAUNCHED("k_scan_block");
        const int st = scan_exclusive(sums.as<int>(), offs.as<int>(), nb, nullptr, s);
        if (st) return st;
        k_scan_add<<<nb, 256, 0, s>>>(out, n, offs.as<int>());
        SBW_LAUNCHED("k_scan_add");
    }
    if (total_dev) {
        k_total<<<1, 1, 0, s>>>(in, out, n, total_dev);
        SBW_LAUNCHED("k_total");
    }
    return SHFLBW_OK;
}

// stable LSD radix sort of (u64 key, u32 value) pairs, ascending by key;
// keys_tmp / vals_tmp are scratch of n elements (also used by prune.cu)
int radix_sort_pairs(uint64_t* keys, uint32_t* vals, uint64_t* keys_tmp, uint32_t* vals_tmp, int n,
                     cudaStream_t s) {
    if (n <= 1) return SHFLBW_OK;
    if (n <= kSmallSort) {
        int P = 2;
        while (P < n) P <<= 1;
        const size_t smem = static_cast<size_t>(P) * 16;
        if (smem > 48 * 1024)  // per call: the attribute is per device
            SBW_CUDA(cudaFuncSetAttribute(k_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
        k_sort_small<<<1, 1024, smem, s>>>(keys, vals, n, P);
        SBW_LAUNCHED("k_sort_small");
        return SHFLBW_OK;
    }
    const int nb = (n + kRadixTile - 1) / kRadixTile;
    DevBuf hist, offs;
    SBW_CUDA(hist.alloc(sizeof(int) * 256 * nb, s));
    SBW_CUDA(offs.alloc(sizeof(int) * 256 * nb, s));
    uint64_t *ki = keys, *ko = keys_tmp;
    uint32_t *vi = vals, *vo = vals_tmp;
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = pass * 8;
        k_radix_hist<<<nb, 256, 0, s>>>(ki, n, shift, hist.as<int>(), nb);
        SBW_LAUNCHED("k_radix_hist");
        int st = scan_exclusive(hist.as<int>(), offs.as<int>(), 256 * nb, nullptr, s);
        if (st) return st;
        k_radix_scatter<<<nb, 256, 0, s>>>(ki, vi, ko, vo, n, shift, offs.as<int>(), nb);
        SBW_LAUNCHED("k_radix_scatter");
        std::swap(ki, ko);
        std::swap(vi, vo);
    }
    // 8 passes: result is back in keys / vals
    return SHFLBW_OK;
}

namespace {

// run `f.template operator()<DT>()` for the matrix value dtype
template <class F>
void by_dtype(int dt, F&& f) {
    if (dt == SHFLBW_BF16) f.template operator()<SHFLBW_BF16>();
    else if (dt == SHFLBW_F16) f.template operator()<SHFLBW_F16>();
    else f.template operator()<SHFLBW_F32>();
}

int launch_pack_rows(const uint8_t* mask, int M, int K, int W, uint64_t seed, uint64_t* words, int* popc,
                     uint64_t* keys, uint32_t* vals, uint32_t* flags, cudaStream_t s,
                     const ClassTable& tab = ClassTable{}) {
    if (K > 0 && K % 16 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15) == 0) {
        k_pack_rows16<<<grid_for(M, 8), 256, 0, s>>>(mask, M, K, W, seed, words, popc, keys, vals, flags, tab);
        SBW_LAUNCHED("k_pack_rows16");
    } else {
        k_pack_rows<<<grid_for(M, 8), 256, 0, s>>>(mask, M, K, W, seed, words, popc, keys, vals, flags, tab);
        SBW_LAUNCHED("k_pack_rows");
    }
    return SHFLBW_OK;
}

// ---- hash planner host side (M <= kPlanMax) ---------------------------------
// K1 k_pack_rows(+table insert) -> K2 k_class_check -> [k_chunk_rank ->
// k_chunk_prefix, M > 4096] -> K3 k_plan (one CTA) -> K4 k_pack_group: four
// (six) launches and two memsets (the sort-based pipeline: 12-30 launches).  Option "converter_legacy"
// forces the sort-based pipeline (kept for M > kPlanMax).
bool use_planner(int M, int V) {
    return M >= 1 && M <= kPlanMax && V >= 1 && option("converter_legacy") == 0;
}

struct HashPlan {
    DevBuf words, popc, table, rep, csize, flags, leader, chunks;
    ClassTable tab;
    int W = 1;
    size_t table_bytes = 0;
};

int hash_plan_alloc(HashPlan& p, int M, int K, int V, cudaStream_t s) {
    p.W = K > 0 ? (K + 63) / 64 : 1;
    uint32_t P = 64;
    while (P < 2u * static_cast<uint32_t>(M)) P <<= 1;
    p.table_bytes = static_cast<size_t>(P) * 16;
    SBW_CUDA(p.words.alloc(sizeof(uint64_t) * static_cast<size_t>(M) * p.W, s));
    SBW_CUDA(p.popc.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.table.alloc(p.table_bytes + sizeof(uint32_t) * M, s));
    SBW_CUDA(p.rep.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.csize.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.flags.alloc(sizeof(uint32_t) * 4, s));
    SBW_CUDA(p.leader.alloc(sizeof(int32_t) * (M / V + 1), s));
    if (M > kPlanSmall) {  // five [M] u16 arrays + per-chunk class counts [chunks][M] + chunk sums
        const size_t nchunks = (M + kPlanThreads - 1) / kPlanThreads;
        const size_t Mp = (static_cast<size_t>(M) + 127) & ~size_t(127);
        SBW_CUDA(p.chunks.alloc(sizeof(uint16_t) * (5 * Mp + nchunks * M + 128) + 64 * sizeof(int), s));
    }
    p.tab.key = p.table.as<uint64_t>();
    p.tab.minrow = reinterpret_cast<uint32_t*>(p.tab.key + P);
    p.tab.cnt = p.tab.minrow + P;
    p.tab.slot = p.tab.cnt + P;
    p.tab.mask = P - 1;
    return SHFLBW_OK;
}

// K1-K3; status[4] (device) = {code, fail_row, total columns, widest group}.
// row_indices == nullptr: validation only.
int hash_plan_run(HashPlan& p, const uint8_t* mask, int M, int K, int V, uint64_t seed, int32_t* row_indices,
                  int32_t* group_ncols, int32_t* group_ptr, int32_t* status, cudaStream_t s) {
    SBW_CUDA(cudaMemsetAsync(p.table.p, 0xff, p.table_bytes, s));
    SBW_CUDA(cudaMemsetAsync(p.flags.p, 0, sizeof(uint32_t) * 4, s));
    if (int st = launch_pack_rows(mask, M, K, p.W, seed, p.words.as<uint64_t>(), p.popc.as<int>(), nullptr, nullptr,
                                  p.flags.as<uint32_t>(), s, p.tab))
        return st;
    k_class_check<<<grid_for(M, 8), 256, 0, s>>>(p.words.as<uint64_t>(), M, p.W, p.tab, p.rep.as<uint32_t>(),
                                                 p.csize.as<uint32_t>(), p.flags.as<uint32_t>());
    SBW_LAUNCHED("k_class_check");
    if (M > kPlanSmall) {
        // chunked planner: 1024-row chunks ranked in parallel, one small CTA
        // for the group offsets and the status
        const int nchunks = (M + kPlanThreads - 1) / kPlanThreads;
        const size_t Mp = (static_cast<size_t>(M) + 127) & ~size_t(127);
        uint16_t* lrank = p.chunks.as<uint16_t>();
        uint16_t* seg_local = lrank + Mp;
        uint16_t* srt = seg_local + Mp;
        uint16_t* rank_pos = srt + Mp;
        uint16_t* gid_local = rank_pos + Mp;
        uint16_t* cnt = gid_local + Mp;
        int* chunk_seg = reinterpret_cast<int*>(
            (reinterpret_cast<uintptr_t>(cnt + static_cast<size_t>(nchunks) * M) + 15) & ~static_cast<uintptr_t>(15));
        int* chunk_lead = chunk_seg + 32;
        k_chunk_rank<<<nchunks, kPlanThreads, 0, s>>>(p.rep.as<uint32_t>(), p.csize.as<uint32_t>(), M, V, lrank, cnt,
                                                      seg_local, chunk_seg, p.flags.as<uint32_t>());
        SBW_LAUNCHED("k_chunk_rank");
        if (row_indices) {
            k_chunk_prefix<<<grid_for(M, 256), 256, 0, s>>>(p.rep.as<uint32_t>(), M, nchunks, cnt);
            SBW_LAUNCHED("k_chunk_prefix");
            k_chunk_place<<<nchunks, kPlanThreads, 0, s>>>(p.rep.as<uint32_t>(), lrank, cnt, seg_local, chunk_seg, M, V,
                                                           nchunks, srt, rank_pos, gid_local, chunk_lead, row_indices,
                                                           p.leader.as<int32_t>(), group_ncols);
            SBW_LAUNCHED("k_chunk_place");
            k_chunk_assign<<<nchunks, kPlanThreads, 0, s>>>(srt, rank_pos, gid_local, chunk_lead, p.popc.as<int>(), M,
                                                            V, nchunks, row_indices, p.leader.as<int32_t>(),
                                                            group_ncols);
            SBW_LAUNCHED("k_chunk_assign");
        }
        k_plan_finish<<<1, kPlanThreads, 0, s>>>(p.rep.as<uint32_t>(), p.csize.as<uint32_t>(), p.words.as<uint64_t>(),
                                                 M, p.W, V, SHFLBW_K_TILE, p.flags.as<uint32_t>(), row_indices,
                                                 group_ncols, group_ptr, status);
        SBW_LAUNCHED("k_plan_finish");
        return SHFLBW_OK;
    }
    const size_t smem = static_cast<size_t>((M + 7) & ~7) * 6 + 32 * 256 * 2;
    if (smem > 48 * 1024)  // per call: the attribute is per device
        SBW_CUDA(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_plan<<<1, kPlanThreads, smem, s>>>(p.rep.as<uint32_t>(), p.csize.as<uint32_t>(), p.popc.as<int>(),
                                         p.words.as<uint64_t>(), M, p.W, V, SHFLBW_K_TILE, p.flags.as<uint32_t>(),
                                         row_indices, p.leader.as<int32_t>(), group_ncols, group_ptr, status);
    SBW_LAUNCHED("k_plan");
    return SHFLBW_OK;
}

// K4 (V <= 128; wider groups: k_pack_cols + k_pack_values + k_contig_blocks)
int launch_pack(const void* dense, int dense_dtype, int K, int V, int G, int64_t max_padded, int W,
                const uint64_t* words, const int32_t* leader, shflbw_cu_matrix* out, uint32_t* contig,
                cudaStream_t s) {
    if (G <= 0 || max_padded <= 0) return SHFLBW_OK;
    const dim3 grid(static_cast<unsigned>((max_padded + SHFLBW_K_TILE - 1) / SHFLBW_K_TILE), G);
    if (V <= 128) {
        const int esz = dtype_bytes(out->dtype);
        const int SV = esz == 2 ? V + 2 : V + 1;
        const size_t smem = ((static_cast<size_t>(SHFLBW_K_TILE) * SV * esz + 15) & ~size_t(15)) + 4 * V;
        by_dtype(out->dtype, [&]<int DT>() {
            auto go = [&](auto kern) {
                kern<<<grid, 256, smem, s>>>(dense, K, V, W, words, leader, out->group_ptr, out->group_ncols,
                                             out->row_indices, out->col_idx, out->values, contig);
            };
            if (dense_dtype == SHFLBW_BF16) go(k_pack_group<DT, SHFLBW_BF16>);
            else if (dense_dtype == SHFLBW_F16) go(k_pack_group<DT, SHFLBW_F16>);
            else go(k_pack_group<DT, SHFLBW_F32>);
        });
        SBW_LAUNCHED("k_pack_group");
        return SHFLBW_OK;
    }
    k_pack_cols<<<G, 128, 0, s>>>(words, W, leader, out->group_ptr, out->group_ncols, out->col_idx);
    SBW_LAUNCHED("k_pack_cols");
    const int jc = V <= 1024 ? 64 : 8;
    const size_t smem = static_cast<size_t>(jc) * V * dtype_bytes(out->dtype);
    const dim3 g2(static_cast<unsigned>((max_padded + jc - 1) / jc), G);
    cudaError_t ce = cudaSuccess;
    by_dtype(out->dtype, [&]<int DT>() {
        if (smem > 48 * 1024)
            ce = cudaFuncSetAttribute(k_pack_values<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem));
        k_pack_values<DT><<<g2, 256, smem, s>>>(dense, dense_dtype, K, V, jc, out->row_indices, out->group_ptr,
                                                 out->group_ncols, out->col_idx, out->values);
    });
    if (ce != cudaSuccess) return cuda_fail(ce, "cudaFuncSetAttribute");
    SBW_LAUNCHED("k_pack_values");
    if (contig) {
        k_contig_blocks<<<G, 32, 0, s>>>(out->group_ptr, out->col_idx, contig);
        SBW_LAUNCHED("k_contig_blocks");
    }
    return SHFLBW_OK;
}

// Steps 1-4 shared by validate and compress.
struct ClassPlan {
    DevBuf words, popc, keys, vals, keys2, vals2, rank, lead, fail_head, flags;
    int W = 1;
};

int plan_classes(const uint8_t* mask, int M, int K, int V, ClassPlan& p, uint32_t host_flags[4],
                 cudaStream_t s) {
    p.W = K > 0 ? (K + 63) / 64 : 1;
    const int64_t MW = static_cast<int64_t>(M) * p.W;
    SBW_CUDA(p.words.alloc(sizeof(uint64_t) * MW, s));
    SBW_CUDA(p.popc.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.keys.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(p.vals.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.keys2.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(p.vals2.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.rank.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.lead.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.fail_head.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.flags.alloc(sizeof(uint32_t) * 4, s));
    if (K == 0) SBW_CUDA(cudaMemsetAsync(p.words.p, 0, sizeof(uint64_t) * MW, s));
    for (int attempt = 0; attempt < 4; ++attempt) {
        const uint64_t seed = 0x5ca1ab1e00000000ULL + attempt;
        SBW_CUDA(cudaMemsetAsync(p.flags.p, 0, sizeof(uint32_t) * 4, s));
        if (attempt == 0) {
            if (int st = launch_pack_rows(mask, M, K, p.W, seed, p.words.as<uint64_t>(), p.popc.as<int>(),
                                          p.keys.as<uint64_t>(), p.vals.as<uint32_t>(), p.flags.as<uint32_t>(), s))
                return st;
            if (K == 0) {  // no columns: every row is the empty support
                SBW_CUDA(cudaMemsetAsync(p.popc.p, 0, sizeof(int) * M, s));
                k_hash_rows<<<grid_for(M, 8), 256, 0, s>>>(p.words.as<uint64_t>(), M, p.W, seed,
                                                           p.keys.as<uint64_t>(), p.vals.as<uint32_t>());
                SBW_LAUNCHED("k_hash_rows");
            }
        } else {
            k_hash_rows<<<grid_for(M, 8), 256, 0, s>>>(p.words.as<uint64_t>(), M, p.W, seed,
                                                       p.keys.as<uint64_t>(), p.vals.as<uint32_t>());
            SBW_LAUNCHED("k_hash_rows");
        }
        int st = radix_sort_pairs(p.keys.as<uint64_t>(), p.vals.as<uint32_t>(), p.keys2.as<uint64_t>(),
                                  p.vals2.as<uint32_t>(), M, s);
        if (st) return st;
        k_runs<<<grid_for(M, 256), 256, 0, s>>>(p.keys.as<uint64_t>(), p.vals.as<uint32_t>(),
                                                p.words.as<uint64_t>(), M, p.W, V, p.rank.as<int>(),
                                                p.lead.as<int>(), p.fail_head.as<int>(),
                                                p.flags.as<uint32_t>());
        SBW_LAUNCHED("k_runs");
        SBW_CUDA(cudaMemcpyAsync(host_flags, p.flags.p, sizeof(uint32_t) * 4, cudaMemcpyDeviceToHost, s));
        SBW_CUDA(cudaStreamSynchronize(s));
        if (host_flags[0]) return fail(SHFLBW_BAD_PARAMS, "SparsityMask: entries must be 0 or 1");
        if (!host_flags[1]) return SHFLBW_OK;
    }
    return fail(SHFLBW_CUDA_ERROR, "compress: unresolvable row-hash collisions");
}

int first_failing_row(ClassPlan& p, int M, uint32_t* fail_row, cudaStream_t s) {
    DevBuf fr;
    SBW_CUDA(fr.alloc(sizeof(uint32_t), s));
    k_fail_argmin<<<1, 1024, 0, s>>>(p.fail_head.as<int>(), p.vals.as<uint32_t>(),
                                     p.words.as<uint64_t>(), M, p.W, fr.as<uint32_t>());
    SBW_LAUNCHED("k_fail_argmin");
    SBW_CUDA(cudaMemcpyAsync(fail_row, fr.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int check_dtype16(int dt) {
    if (dt != SHFLBW_BF16 && dt != SHFLBW_F16 && dt != SHFLBW_F32)
        return fail(SHFLBW_BAD_PARAMS, "value dtype must be SHFLBW_BF16, SHFLBW_F16 or SHFLBW_F32");
    return SHFLBW_OK;
}

// allocate meta (row_indices, group_ptr, group_ncols) in one block
int alloc_meta(shflbw_cu_matrix* out, int M, int K, int V, int dtype, cudaStream_t s) {
    const int G = M / V;
    const size_t a = (static_cast<size_t>(M) * 4 + 255) / 256 * 256;
    const size_t b = (static_cast<size_t>(G + 1) * 4 + 255) / 256 * 256;
    const size_t c = (static_cast<size_t>(G) * 4 + 255) / 256 * 256;
    char* base = nullptr;
    // stream-ordered pool allocation (a plain cudaMalloc synchronises the
    // device and cost ~0.1-0.5 ms per matrix); freed with cudaFree
    retain_pool();
    SBW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), a + b + c + 256, s));
    *out = shflbw_cu_matrix{};
    out->rows = M;
    out->cols = K;
    out->v = V;
    out->groups = G;
    out->dtype = dtype;
    out->k_tile = SHFLBW_K_TILE;
    out->row_indices = reinterpret_cast<int32_t*>(base);
    out->group_ptr = reinterpret_cast<int32_t*>(base + a);
    out->group_ncols = reinterpret_cast<int32_t*>(base + a + b);
    int dev = 0;
    cudaGetDevice(&dev);
    out->device = dev;
    out->owns = 1;
    return SHFLBW_OK;
}

int alloc_data(shflbw_cu_matrix* out, int64_t total, cudaStream_t s) {
    const size_t a = (static_cast<size_t>(total) * 4 + 255) / 256 * 256;
    const size_t b = static_cast<size_t>(total) * out->v * dtype_bytes(out->dtype);
    char* base = nullptr;
    SBW_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), a + b + 256, s));
    out->col_idx = reinterpret_cast<int32_t*>(base);
    out->values = base + a;
    out->total_cols = total;
    return SHFLBW_OK;
}

}  // namespace

void free_matrix(shflbw_cu_matrix* m) {
    if (!m || !m->owns) return;
    if (m->row_indices) cudaFree(m->row_indices);
    if (m->col_idx) cudaFree(m->col_idx);
    m->row_indices = m->group_ptr = m->group_ncols = m->col_idx = nullptr;
    m->values = nullptr;
    m->owns = 0;
}

int validate_impl(const uint8_t* mask, int M, int K, int V, int32_t* pass, uint32_t* fail_row,
                  cudaStream_t s) {
    if (V <= 0 || M < 0 || K < 0 || M % V != 0) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    *pass = 1;
    *fail_row = 0;
    if (M == 0) return SHFLBW_OK;
    if (use_planner(M, V)) {
        HashPlan hp;
        DevBuf st;
        if (int e = hash_plan_alloc(hp, M, K, V, s)) return e;
        SBW_CUDA(st.alloc(sizeof(int32_t) * 4, s));
        int32_t h[4] = {0, 0, 0, 0};
        for (int attempt = 0; attempt < 4; ++attempt) {
            if (int e = hash_plan_run(hp, mask, M, K, V, 0x5ca1ab1e00000000ULL + attempt, nullptr, nullptr, nullptr,
                                      st.as<int32_t>(), s))
                return e;
            SBW_CUDA(cudaMemcpyAsync(h, st.p, sizeof(h), cudaMemcpyDeviceToHost, s));
            SBW_CUDA(cudaStreamSynchronize(s));
            if (h[0] != SHFLBW_CUDA_ERROR) break;
        }
        if (h[0] == SHFLBW_BAD_PARAMS) return fail(SHFLBW_BAD_PARAMS, "SparsityMask: entries must be 0 or 1");
        if (h[0] == SHFLBW_CUDA_ERROR) return fail(SHFLBW_CUDA_ERROR, "compress: unresolvable row-hash collisions");
        if (h[0] == SHFLBW_NONCONFORMANT_MASK) {
            *pass = 0;
            *fail_row = static_cast<uint32_t>(h[1]);
        }
        return SHFLBW_OK;
    }
    ClassPlan p;
    uint32_t hf[4];
    int st = plan_classes(mask, M, K, V, p, hf, s);
    if (st) return st;
    if (hf[2]) {
        *pass = 0;
        return first_failing_row(p, M, fail_row, s);
    }
    return SHFLBW_OK;
}

int compress_impl(const void* dense, int dense_dtype, const uint8_t* mask, int M, int K, int V,
                  int value_dtype, shflbw_cu_matrix* out, uint32_t* fail_row, cudaStream_t s) {
    if (int st = check_dtype16(value_dtype)) return st;
    if (dense_dtype < SHFLBW_F32 || dense_dtype > SHFLBW_F16) return fail(SHFLBW_BAD_PARAMS, "dense dtype");
    if (V <= 0 || M < 0 || K < 0 || M % V != 0) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    if (fail_row) *fail_row = 0;
    const int G = M / V;
    if (int st = alloc_meta(out, M, K, V, value_dtype, s)) return st;
    auto cleanup = [&](int st) {
        if (st) free_matrix(out);
        return st;
    };
    if (M == 0) {
        SBW_CUDA(cudaMemsetAsync(out->group_ptr, 0, sizeof(int32_t), s));
        return cleanup(alloc_data(out, 0, s));
    }
    if (use_planner(M, V)) {
        HashPlan hp;
        DevBuf stb, cf;
        if (int e = hash_plan_alloc(hp, M, K, V, s)) return cleanup(e);
        SBW_CUDA(stb.alloc(sizeof(int32_t) * 4, s));
        SBW_CUDA(cf.alloc(sizeof(uint32_t), s));
        int32_t h[4] = {0, 0, 0, 0};
        for (int attempt = 0; attempt < 4; ++attempt) {
            if (int e = hash_plan_run(hp, mask, M, K, V, 0x5ca1ab1e00000000ULL + attempt, out->row_indices,
                                      out->group_ncols, out->group_ptr, stb.as<int32_t>(), s))
                return cleanup(e);
            SBW_CUDA(cudaMemcpyAsync(h, stb.p, sizeof(h), cudaMemcpyDeviceToHost, s));
            SBW_CUDA(cudaStreamSynchronize(s));
            if (h[0] != SHFLBW_CUDA_ERROR) break;
        }
        if (h[0] == SHFLBW_BAD_PARAMS) return cleanup(fail(SHFLBW_BAD_PARAMS, "SparsityMask: entries must be 0 or 1"));
        if (h[0] == SHFLBW_CUDA_ERROR)
            return cleanup(fail(SHFLBW_CUDA_ERROR, "compress: unresolvable row-hash collisions"));
        if (h[0] == SHFLBW_NONCONFORMANT_MASK) {
            if (fail_row) *fail_row = static_cast<uint32_t>(h[1]);
            return cleanup(fail(SHFLBW_NONCONFORMANT_MASK,
                                "compress_shflbw: support class size is not a multiple of V (row " +
                                    std::to_string(h[1]) + ")"));
        }
        out->max_group_cols = h[3];
        if (int e = alloc_data(out, h[2], s)) return cleanup(e);
        SBW_CUDA(cudaMemsetAsync(cf.p, 0, sizeof(uint32_t), s));
        if (int e = launch_pack(dense, dense_dtype, K, V, G, h[3], hp.W, hp.words.as<uint64_t>(),
                                hp.leader.as<int32_t>(), out, cf.as<uint32_t>(), s))
            return cleanup(e);
        uint32_t contig = 0;
        SBW_CUDA(cudaMemcpyAsync(&contig, cf.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        // the matrix is complete on return (SpMM prologues read it before their
        // programmatic-launch wait, see the "pdl" option)
        SBW_CUDA(cudaStreamSynchronize(s));
        if (contig) out->reserved |= SHFLBW_CONTIG_BLOCKS;
        return SHFLBW_OK;
    }
    ClassPlan p;
    uint32_t hf[4];
    int st = plan_classes(mask, M, K, V, p, hf, s);
    if (st) return cleanup(st);
    if (hf[2]) {
        uint32_t fr = 0;
        st = first_failing_row(p, M, &fr, s);
        if (st) return cleanup(st);
        if (fail_row) *fail_row = fr;
        return cleanup(fail(SHFLBW_NONCONFORMANT_MASK,
                            "compress_shflbw: support class size is not a multiple of V (row " +
                                std::to_string(fr) + ")"));
    }
    DevBuf gid, leader, padded, total;
    SBW_CUDA(gid.alloc(sizeof(int) * M, s));
    SBW_CUDA(leader.alloc(sizeof(int) * G, s));
    SBW_CUDA(padded.alloc(sizeof(int) * G, s));
    SBW_CUDA(total.alloc(sizeof(int), s));
    if ((st = scan_exclusive(p.lead.as<int>(), gid.as<int>(), M, nullptr, s))) return cleanup(st);
    k_assign<<<grid_for(M, 256), 256, 0, s>>>(p.vals.as<uint32_t>(), p.rank.as<int>(), gid.as<int>(),
                                              p.popc.as<int>(), M, V, SHFLBW_K_TILE, out->row_indices,
                                              leader.as<int32_t>(), out->group_ncols, padded.as<int>());
    SBW_LAUNCHED("k_assign");
    if ((st = scan_exclusive(padded.as<int>(), out->group_ptr, G, out->group_ptr + G, s))) return cleanup(st);
    k_max<<<1, 256, 0, s>>>(padded.as<int>(), G, total.as<int>());
    SBW_LAUNCHED("k_max");
    int sizes[2] = {0, 0};
    SBW_CUDA(cudaMemcpyAsync(&sizes[0], out->group_ptr + G, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(&sizes[1], total.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    const int total_cols = sizes[0];
    out->max_group_cols = sizes[1];
    if ((st = alloc_data(out, total_cols, s))) return cleanup(st);
    if (G > 0) {
        k_pack_cols<<<G, 128, 0, s>>>(p.words.as<uint64_t>(), p.W, leader.as<int32_t>(), out->group_ptr,
                                      out->group_ncols, out->col_idx);
        SBW_LAUNCHED("k_pack_cols");
        const int jc = V <= 1024 ? 64 : 8;
        const size_t smem = static_cast<size_t>(jc) * V * dtype_bytes(value_dtype);
        int max_padded = K <= 0 ? 0 : (K + SHFLBW_K_TILE - 1) / SHFLBW_K_TILE * SHFLBW_K_TILE;
        dim3 grid((max_padded + jc - 1) / jc, G);
        if (grid.x > 0) {
            cudaError_t ce = cudaSuccess;
            by_dtype(value_dtype, [&]<int DT>() {
                if (smem > 48 * 1024)
                    ce = cudaFuncSetAttribute(k_pack_values<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem));
                k_pack_values<DT><<<grid, 256, smem, s>>>(dense, dense_dtype, K, V, jc, out->row_indices,
                                                          out->group_ptr, out->group_ncols, out->col_idx,
                                                          out->values);
            });
            if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "cudaFuncSetAttribute"));
            SBW_LAUNCHED("k_pack_values");
        }
    }
    // contiguous 64-column K blocks anywhere (block-wise masks)?
    uint32_t contig = 0;
    if (G > 0 && total_cols > 0) {
        DevBuf cf;
        SBW_CUDA(cf.alloc(sizeof(uint32_t), s));
        SBW_CUDA(cudaMemsetAsync(cf.p, 0, sizeof(uint32_t), s));
        k_contig_blocks<<<G, 32, 0, s>>>(out->group_ptr, out->col_idx, cf.as<uint32_t>());
        SBW_LAUNCHED("k_contig_blocks");
        SBW_CUDA(cudaMemcpyAsync(&contig, cf.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    }
    // the matrix is complete on return (SpMM prologues read it before their
    // programmatic-launch wait, see the "pdl" option)
    SBW_CUDA(cudaStreamSynchronize(s));
    if (contig) out->reserved |= SHFLBW_CONTIG_BLOCKS;
    return SHFLBW_OK;
}

// The converter without a host synchronisation (graph-capturable): the
// output is allocated from the bound G * roundup(K, 64) columns, hash
// collisions / bad mask bytes / non-conformance and the sizes are written to
// status[4] on the device, and the rest of the pipeline runs regardless (in
// bounds).  shflbw_cu_matrix_finalize reads the status back.
int compress_async_impl(const void* dense, int dense_dtype, const uint8_t* mask, int M, int K, int V,
                        int value_dtype, shflbw_cu_matrix* out, int32_t* status, cudaStream_t s) {
    if (int st = check_dtype16(value_dtype)) return st;
    if (dense_dtype < SHFLBW_F32 || dense_dtype > SHFLBW_F16) return fail(SHFLBW_BAD_PARAMS, "dense dtype");
    if (V <= 0 || M < 0 || K < 0 || M % V != 0) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    const int G = M / V;
    const int64_t kpad = (static_cast<int64_t>(K) + SHFLBW_K_TILE - 1) / SHFLBW_K_TILE * SHFLBW_K_TILE;
    const int64_t bound = static_cast<int64_t>(G) * kpad;
    if (bound > 0x7fffffffLL) return fail(SHFLBW_UNSUPPORTED, "compress_async: G * roundup(K, 64) exceeds 2^31");
    // reuse a bound-sized matrix of the same shape (e.g. converting into the
    // same buffers on every replay of a captured graph), else allocate one
    const bool reuse = out->owns && out->row_indices && (out->reserved & SHFLBW_BOUND_ALLOC) && out->rows == M &&
                       out->cols == K && out->v == V && out->dtype == value_dtype;
    auto cleanup = [&](int st) {
        if (st && !reuse) free_matrix(out);
        return st;
    };
    if (!reuse) {
        if (int st = alloc_meta(out, M, K, V, value_dtype, s)) return st;
        if (int st = alloc_data(out, bound, s)) return cleanup(st);
    }
    out->total_cols = bound;
    out->max_group_cols = static_cast<int32_t>(kpad);
    out->reserved = SHFLBW_SIZE_BOUND | SHFLBW_BOUND_ALLOC;
    if (M > 0 && use_planner(M, V)) {
        HashPlan hp;
        if (int e = hash_plan_alloc(hp, M, K, V, s)) return cleanup(e);
        if (int e = hash_plan_run(hp, mask, M, K, V, 0x5ca1ab1e00000000ULL, out->row_indices, out->group_ncols,
                                  out->group_ptr, status, s))
            return cleanup(e);
        if (int e = launch_pack(dense, dense_dtype, K, V, G, kpad, hp.W, hp.words.as<uint64_t>(),
                                hp.leader.as<int32_t>(), out, nullptr, s))
            return cleanup(e);
        return SHFLBW_OK;
    }
    DevBuf flags, fr, maxp;
    SBW_CUDA(flags.alloc(sizeof(uint32_t) * 4, s));
    SBW_CUDA(fr.alloc(sizeof(uint32_t), s));
    SBW_CUDA(maxp.alloc(sizeof(int), s));
    SBW_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(uint32_t) * 4, s));
    SBW_CUDA(cudaMemsetAsync(fr.p, 0, sizeof(uint32_t), s));
    SBW_CUDA(cudaMemsetAsync(maxp.p, 0, sizeof(int), s));
    if (M == 0) {
        SBW_CUDA(cudaMemsetAsync(out->group_ptr, 0, sizeof(int32_t), s));
        k_status<<<1, 1, 0, s>>>(flags.as<uint32_t>(), fr.as<uint32_t>(), out->group_ptr, maxp.as<int>(), status);
        SBW_LAUNCHED("k_status");
        return SHFLBW_OK;
    }
    ClassPlan p;
    p.W = K > 0 ? (K + 63) / 64 : 1;
    const int64_t MW = static_cast<int64_t>(M) * p.W;
    SBW_CUDA(p.words.alloc(sizeof(uint64_t) * MW, s));
    SBW_CUDA(p.popc.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.keys.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(p.vals.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.keys2.alloc(sizeof(uint64_t) * M, s));
    SBW_CUDA(p.vals2.alloc(sizeof(uint32_t) * M, s));
    SBW_CUDA(p.rank.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.lead.alloc(sizeof(int) * M, s));
    SBW_CUDA(p.fail_head.alloc(sizeof(int) * M, s));
    if (K == 0) SBW_CUDA(cudaMemsetAsync(p.words.p, 0, sizeof(uint64_t) * MW, s));
    const uint64_t seed = 0x5ca1ab1e00000000ULL;
    if (int st = launch_pack_rows(mask, M, K, p.W, seed, p.words.as<uint64_t>(), p.popc.as<int>(),
                                  p.keys.as<uint64_t>(), p.vals.as<uint32_t>(), flags.as<uint32_t>(), s))
        return cleanup(st);
    if (K == 0) {
        SBW_CUDA(cudaMemsetAsync(p.popc.p, 0, sizeof(int) * M, s));
        k_hash_rows<<<grid_for(M, 8), 256, 0, s>>>(p.words.as<uint64_t>(), M, p.W, seed, p.keys.as<uint64_t>(),
                                                   p.vals.as<uint32_t>());
        SBW_LAUNCHED("k_hash_rows");
    }
    int st = radix_sort_pairs(p.keys.as<uint64_t>(), p.vals.as<uint32_t>(), p.keys2.as<uint64_t>(),
                              p.vals2.as<uint32_t>(), M, s);
    if (st) return cleanup(st);
    k_runs<<<grid_for(M, 256), 256, 0, s>>>(p.keys.as<uint64_t>(), p.vals.as<uint32_t>(), p.words.as<uint64_t>(), M,
                                            p.W, V, p.rank.as<int>(), p.lead.as<int>(), p.fail_head.as<int>(),
                                            flags.as<uint32_t>());
    SBW_LAUNCHED("k_runs");
    k_fail_argmin<<<1, 1024, 0, s>>>(p.fail_head.as<int>(), p.vals.as<uint32_t>(), p.words.as<uint64_t>(), M, p.W,
                                     fr.as<uint32_t>());
    SBW_LAUNCHED("k_fail_argmin");
    DevBuf gid, leader, padded;
    SBW_CUDA(gid.alloc(sizeof(int) * M, s));
    SBW_CUDA(leader.alloc(sizeof(int) * G, s));
    SBW_CUDA(padded.alloc(sizeof(int) * G, s));
    // every slot defined even when a non-conformant mask leaves some unassigned
    SBW_CUDA(cudaMemsetAsync(out->row_indices, 0, sizeof(int32_t) * M, s));
    SBW_CUDA(cudaMemsetAsync(out->group_ncols, 0, sizeof(int32_t) * G, s));
    SBW_CUDA(cudaMemsetAsync(leader.p, 0, sizeof(int) * G, s));
    SBW_CUDA(cudaMemsetAsync(padded.p, 0, sizeof(int) * G, s));
    if ((st = scan_exclusive(p.lead.as<int>(), gid.as<int>(), M, nullptr, s))) return cleanup(st);
    k_assign<<<grid_for(M, 256), 256, 0, s>>>(p.vals.as<uint32_t>(), p.rank.as<int>(), gid.as<int>(), p.popc.as<int>(),
                                              M, V, SHFLBW_K_TILE, out->row_indices, leader.as<int32_t>(),
                                              out->group_ncols, padded.as<int>());
    SBW_LAUNCHED("k_assign");
    if ((st = scan_exclusive(padded.as<int>(), out->group_ptr, G, out->group_ptr + G, s))) return cleanup(st);
    k_max<<<1, 256, 0, s>>>(padded.as<int>(), G, maxp.as<int>());
    SBW_LAUNCHED("k_max");
    if (G > 0) {
        k_pack_cols<<<G, 128, 0, s>>>(p.words.as<uint64_t>(), p.W, leader.as<int32_t>(), out->group_ptr,
                                      out->group_ncols, out->col_idx);
        SBW_LAUNCHED("k_pack_cols");
        const int jc = V <= 1024 ? 64 : 8;
        const size_t smem = static_cast<size_t>(jc) * V * dtype_bytes(value_dtype);
        const dim3 grid(static_cast<unsigned>((kpad + jc - 1) / jc), G);
        if (grid.x > 0) {
            cudaError_t ce = cudaSuccess;
            by_dtype(value_dtype, [&]<int DT>() {
                if (smem > 48 * 1024)
                    ce = cudaFuncSetAttribute(k_pack_values<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              static_cast<int>(smem));
                k_pack_values<DT><<<grid, 256, smem, s>>>(dense, dense_dtype, K, V, jc, out->row_indices,
                                                          out->group_ptr, out->group_ncols, out->col_idx,
                                                          out->values);
            });
            if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "cudaFuncSetAttribute"));
            SBW_LAUNCHED("k_pack_values");
        }
    }
    k_status<<<1, 1, 0, s>>>(flags.as<uint32_t>(), fr.as<uint32_t>(), out->group_ptr + G, maxp.as<int>(), status);
    SBW_LAUNCHED("k_status");
    return SHFLBW_OK;
}

int finalize_impl(shflbw_cu_matrix* m, const int32_t* status, uint32_t* fail_row, cudaStream_t s) {
    int32_t h[4] = {0, 0, 0, 0};
    SBW_CUDA(cudaMemcpyAsync(h, status, sizeof(h), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    if (fail_row) *fail_row = static_cast<uint32_t>(h[1]);
    switch (h[0]) {
        case SHFLBW_OK: break;
        case SHFLBW_BAD_PARAMS: return fail(SHFLBW_BAD_PARAMS, "SparsityMask: entries must be 0 or 1");
        case SHFLBW_NONCONFORMANT_MASK:
            return fail(SHFLBW_NONCONFORMANT_MASK,
                        "compress_shflbw: support class size is not a multiple of V (row " + std::to_string(h[1]) + ")");
        default: return fail(SHFLBW_CUDA_ERROR, "compress_async: row-hash collision (retry with shflbw_cu_compress)");
    }
    m->total_cols = h[2];
    m->max_group_cols = h[3];
    m->reserved &= ~SHFLBW_SIZE_BOUND;
    return SHFLBW_OK;
}

int upload_impl(int M, int K, int V, const uint32_t* row_indices, const uint32_t* group_ncols,
                const uint32_t* cols, const float* values, int value_dtype, shflbw_cu_matrix* out,
                cudaStream_t s) {
    if (int st = check_dtype16(value_dtype)) return st;
    if (V <= 0 || M < 0 || K < 0 || M % V != 0) return fail(SHFLBW_BAD_PARAMS, "V must divide M");
    const int G = M / V;
    int64_t nnzc = 0;
    for (int g = 0; g < G; ++g) nnzc += group_ncols[g];
    if (int st = alloc_meta(out, M, K, V, value_dtype, s)) return st;
    auto cleanup = [&](int st) {
        if (st) free_matrix(out);
        return st;
    };
    DevBuf d_cols, d_vals, d_off, d_pad, flags;
    SBW_CUDA(d_cols.alloc(sizeof(uint32_t) * nnzc, s));
    SBW_CUDA(d_vals.alloc(sizeof(float) * nnzc * V, s));
    SBW_CUDA(d_off.alloc(sizeof(int) * (G + 1), s));
    SBW_CUDA(d_pad.alloc(sizeof(int) * (G + 1), s));
    SBW_CUDA(flags.alloc(sizeof(uint32_t) * 4, s));
    SBW_CUDA(cudaMemsetAsync(flags.p, 0, 16, s));
    SBW_CUDA(cudaMemcpyAsync(out->row_indices, row_indices, sizeof(int32_t) * M, cudaMemcpyHostToDevice, s));
    SBW_CUDA(cudaMemcpyAsync(out->group_ncols, group_ncols, sizeof(int32_t) * G, cudaMemcpyHostToDevice, s));
    if (nnzc) {
        SBW_CUDA(cudaMemcpyAsync(d_cols.p, cols, sizeof(uint32_t) * nnzc, cudaMemcpyHostToDevice, s));
        SBW_CUDA(cudaMemcpyAsync(d_vals.p, values, sizeof(float) * nnzc * V, cudaMemcpyHostToDevice, s));
    }
    int st;
    if (G > 0) {
        k_upload_groups<<<grid_for(G, 256), 256, 0, s>>>(out->group_ncols, G, V, K, SHFLBW_K_TILE,
                                                         d_pad.as<int>(), flags.as<uint32_t>());
        SBW_LAUNCHED("k_upload_groups");
    }
    if (M > 0) {
        k_check_rows<<<grid_for(M, 256), 256, 0, s>>>(out->row_indices, M, flags.as<uint32_t>());
        SBW_LAUNCHED("k_check_rows");
    }
    if ((st = scan_exclusive(out->group_ncols, d_off.as<int>(), G, nullptr, s))) return cleanup(st);
    if ((st = scan_exclusive(d_pad.as<int>(), out->group_ptr, G, out->group_ptr + G, s))) return cleanup(st);
    if (G > 0) {
        k_max<<<1, 256, 0, s>>>(d_pad.as<int>(), G, d_pad.as<int>() + G);
        SBW_LAUNCHED("k_max");
    } else {
        SBW_CUDA(cudaMemsetAsync(d_pad.as<int>(), 0, sizeof(int), s));
    }
    int total_cols = 0, max_cols = 0;
    uint32_t hf[4];
    SBW_CUDA(cudaMemcpyAsync(&max_cols, d_pad.as<int>() + G, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(&total_cols, out->group_ptr + G, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(hf, flags.p, 16, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    if (hf[0]) return cleanup(fail(SHFLBW_SHAPE_MISMATCH, "spmm: row index out of range"));
    if (hf[3]) return cleanup(fail(SHFLBW_BAD_PARAMS, "group column count exceeds K"));
    out->max_group_cols = max_cols;
    if ((st = alloc_data(out, total_cols, s))) return cleanup(st);
    if (G > 0 && total_cols > 0) {
        dim3 grid(grid_for(static_cast<int64_t>(K + SHFLBW_K_TILE) * V, 256 * 4), G);
        by_dtype(value_dtype, [&]<int DT>() {
            k_upload_values<DT><<<grid, 256, 0, s>>>(d_cols.as<uint32_t>(), d_vals.as<float>(), d_off.as<int>(),
                                                     out->group_ptr, out->group_ncols, V, K, out->col_idx,
                                                     out->values, flags.as<uint32_t>());
        });
        SBW_LAUNCHED("k_upload_values");
        SBW_CUDA(cudaMemcpyAsync(hf, flags.p, 16, cudaMemcpyDeviceToHost, s));
        SBW_CUDA(cudaStreamSynchronize(s));
        if (hf[1]) return cleanup(fail(SHFLBW_SHAPE_MISMATCH, "column index exceeds B rows or is not increasing"));
    }
    SBW_CUDA(cudaStreamSynchronize(s));
    {   // contiguous 64-column K blocks (the device layout's K blocks start at
        // each group's column 0)
        int64_t off = 0;
        for (int g = 0; g < G && !(out->reserved & SHFLBW_CONTIG_BLOCKS); ++g) {
            for (uint32_t j = 0; j + SHFLBW_K_TILE <= group_ncols[g]; j += SHFLBW_K_TILE)
                if (cols[off + j + SHFLBW_K_TILE - 1] - cols[off + j] == SHFLBW_K_TILE - 1) {
                    out->reserved |= SHFLBW_CONTIG_BLOCKS;
                    break;
                }
            off += group_ncols[g];
        }
    }
    return SHFLBW_OK;
}

int download_impl(const shflbw_cu_matrix* m, uint32_t* row_indices, uint32_t* group_ncols,
                  uint32_t* cols, float* values, cudaStream_t s) {
    const int G = m->groups, V = m->v, M = m->rows;
    SBW_CUDA(cudaMemcpyAsync(row_indices, m->row_indices, sizeof(int32_t) * M, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(group_ncols, m->group_ncols, sizeof(int32_t) * G, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    int64_t nnzc = 0;
    for (int g = 0; g < G; ++g) nnzc += group_ncols[g];
    if (nnzc == 0) return SHFLBW_OK;
    DevBuf d_off, d_cols, d_vals;
    SBW_CUDA(d_off.alloc(sizeof(int) * (G + 1), s));
    SBW_CUDA(d_cols.alloc(sizeof(uint32_t) * nnzc, s));
    SBW_CUDA(d_vals.alloc(sizeof(float) * nnzc * V, s));
    int st = scan_exclusive(m->group_ncols, d_off.as<int>(), G, nullptr, s);
    if (st) return st;
    dim3 grid(grid_for(static_cast<int64_t>(m->cols + 1) * V, 1024), G);
    by_dtype(m->dtype, [&]<int DT>() {
        k_download_values<DT><<<grid, 256, 0, s>>>(m->col_idx, m->values, d_off.as<int>(), m->group_ptr,
                                                   m->group_ncols, V, d_cols.as<uint32_t>(), d_vals.as<float>());
    });
    SBW_LAUNCHED("k_download_values");
    SBW_CUDA(cudaMemcpyAsync(cols, d_cols.p, sizeof(uint32_t) * nnzc, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(values, d_vals.p, sizeof(float) * nnzc * V, cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int conv_prepare_impl(const shflbw_cu_matrix* w, int S, shflbw_cu_matrix* out, cudaStream_t s) {
    if (S < 1 || S > 32) return fail(SHFLBW_UNSUPPORTED, "conv_prepare: filter width S must be 1..32");
    const int M = w->rows, K = w->cols, V = w->v, G = w->groups;
    if (int st = alloc_meta(out, M, K, V, w->dtype, s)) return st;
    auto cleanup = [&](int st) {
        if (st) free_matrix(out);
        return st;
    };
    DevBuf widths, slot;
    SBW_CUDA(widths.alloc(sizeof(int) * (G + 1), s));
    SBW_CUDA(slot.alloc(sizeof(int32_t) * std::max<int64_t>(w->total_cols, 1), s));
    SBW_CUDA(cudaMemcpyAsync(out->row_indices, w->row_indices, sizeof(int32_t) * M, cudaMemcpyDeviceToDevice, s));
    SBW_CUDA(cudaMemcpyAsync(out->group_ncols, w->group_ncols, sizeof(int32_t) * G, cudaMemcpyDeviceToDevice, s));
    int st;
    if (G > 0) {
        k_conv_widths<<<G, 256, 0, s>>>(w->group_ptr, w->col_idx, S, widths.as<int>());
        SBW_LAUNCHED("k_conv_widths");
    }
    if ((st = scan_exclusive(widths.as<int>(), out->group_ptr, G, out->group_ptr + G, s))) return cleanup(st);
    if (G > 0) {
        k_max<<<1, 256, 0, s>>>(widths.as<int>(), G, widths.as<int>() + G);
        SBW_LAUNCHED("k_max");
    } else {
        SBW_CUDA(cudaMemsetAsync(widths.as<int>(), 0, sizeof(int), s));
    }
    int total = 0, widest = 0;
    SBW_CUDA(cudaMemcpyAsync(&total, out->group_ptr + G, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaMemcpyAsync(&widest, widths.as<int>() + G, sizeof(int), cudaMemcpyDeviceToHost, s));
    SBW_CUDA(cudaStreamSynchronize(s));
    out->max_group_cols = widest;
    if ((st = alloc_data(out, total, s))) return cleanup(st);
    if (total > 0) {
        SBW_CUDA(cudaMemsetAsync(out->col_idx, 0xff, sizeof(int32_t) * static_cast<size_t>(total), s));
        SBW_CUDA(cudaMemsetAsync(out->values, 0, static_cast<size_t>(total) * V * dtype_bytes(w->dtype), s));
        by_dtype(w->dtype, [&]<int DT>() {
            k_conv_scatter<DT><<<G, 256, 0, s>>>(w->group_ptr, w->col_idx, w->values, out->group_ptr, S, V,
                                                 out->col_idx, out->values, slot.as<int32_t>());
        });
        SBW_LAUNCHED("k_conv_scatter");
    }
    out->reserved = (w->reserved & ~(SHFLBW_CONV_ORDER | SHFLBW_CONTIG_BLOCKS | (0xff << 8))) | SHFLBW_CONV_ORDER |
                    (S << 8);
    SBW_CUDA(cudaStreamSynchronize(s));
    return SHFLBW_OK;
}

int decompress_impl(const shflbw_cu_matrix* m, float* dense, cudaStream_t s) {
    SBW_CUDA(cudaMemsetAsync(dense, 0, sizeof(float) * static_cast<size_t>(m->rows) * m->cols, s));
    if (m->groups == 0) return SHFLBW_OK;
    const int64_t widest = m->max_group_cols > 0 ? m->max_group_cols : static_cast<int64_t>(m->cols) + SHFLBW_K_TILE;
    dim3 grid(grid_for(std::max<int64_t>(widest, m->cols + 1) * m->v, 1024), m->groups);
    by_dtype(m->dtype, [&]<int DT>() {
        k_decompress<DT><<<grid, 256, 0, s>>>(m->row_indices, m->group_ptr, m->group_ncols, m->col_idx, m->values,
                                              m->v, m->cols, dense);
    });
    SBW_LAUNCHED("k_decompress");
    return SHFLBW_OK;
}

int convert_impl(const void* src, int sdt, void* dst, int ddt, int64_t n, cudaStream_t s) {
    if (n <= 0) return SHFLBW_OK;
    k_convert<<<grid_for(n, 256 * 8), 256, 0, s>>>(src, sdt, dst, ddt, n);
    SBW_LAUNCHED("k_convert");
    return SHFLBW_OK;
}

int convert_2d_impl(const void* src, int sdt, int64_t ld_src, void* dst, int ddt, int64_t ld_dst, int64_t rows,
                    int64_t cols, cudaStream_t s) {
    if (rows <= 0 || cols <= 0) return SHFLBW_OK;
    const dim3 grid(static_cast<unsigned>(std::min<int64_t>((cols + 255) / 256, 64)),
                    static_cast<unsigned>(std::min<int64_t>(rows, 65535)));
    k_convert_2d<<<grid, 256, 0, s>>>(src, sdt, ld_src, dst, ddt, ld_dst, rows, cols);
    SBW_LAUNCHED("k_convert_2d");
    return SHFLBW_OK;
}

}  // namespace sbw
