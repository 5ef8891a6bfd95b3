// tc_kernels.cuh -- K2: Shfl-BW SpMM / implicit-GEMM conv on the 5th-generation
// tensor cores (kernels and launch templates; instantiated per input dtype and
// operand kind in tc_inst_*.cu so they compile in parallel, host planning in
// spmm_sm100.cu).
//
// Replaces spmm_execute (/root/reference/proj/src/spmm.cpp:76-146): the
// reference's per-group "in-buffer stitching" (stitch_into, src/spmm.cpp:24-34),
// tile_mma (src/spmm.cpp:60-74) and reordered write-back
// (src/spmm.cpp:115-123) become one warp-specialised sm_100a kernel:
//
//   * work unit: (group g, 128 output columns n0..n0+127, V-slice).  The MMA
//     runs transposed, D[n][v] = sum_j B[col_j][n] * W_g[v][j], so the
//     activation tile is the M=128 operand and the group's V rows are the
//     N operand (N = VS in {16, 32, 64, 128}): every V the paper uses maps
//     to one legal tcgen05.mma shape, and the fp32 accumulator lives in TMEM
//     (128 lanes x VS columns).
//   * producer warps (4 or 8): for each 64-column K block, 32 TMA
//     tile::gather4 instructions fetch the 64 activation rows named by the
//     group's column indices straight into the 128B-swizzled MN-major operand
//     layout; pad columns carry index -1, which TMA zero-fills.  One 2D TMA
//     tile load fetches the group's 64 x VS value block (V contiguous, the
//     reference's column-major group layout, include/shflbw/formats.hpp:14-18).
//     A full/empty mbarrier ring of `stages` slots keeps the loads ahead of
//     the MMAs (the explicit empty barrier is what the literal Alg. 1 lacks,
//     tests/test_pipeline.cpp:50-79).  No integer division on any per-K-block
//     path (ring counters are stepped; conv taps are decoded per staged
//     window): these loops are single-thread latency chains.
//   * MMA warp: one elected thread issues 4 x tcgen05.mma (K=16) per block and
//     releases the slot with tcgen05.commit.
//   * epilogue (4 warps, TMEM lane quarters): 16-bit outputs are read with
//     tcgen05.ld.16x256b, packed and transposed into a [VS][128] shared tile
//     with stmatrix; fp32 / K-split outputs with tcgen05.ld.32x32b; then every
//     output row row_indices[g*V+v] is written with coalesced 16-byte stores
//     -- the permuted write-back fused into the epilogue (optionally into
//     several GPUs' outputs: the fused all-gather).
//   * V split across a cluster of CS CTAs (CS*VS = V): each CTA owns VS of the
//     group's rows; the activation gathers are split between the CTAs and
//     multicast to all of them, so a group's activation tile is read from L2
//     once per cluster while CS SMs share the MMA work.  Used when the grid
//     would otherwise leave SMs idle (the north-star shape has 32 groups x 1
//     column tile).
//
// Accumulation order: tensor-core fp32 accumulation over K=16 slices in
// ascending k; products of 16-bit inputs are exact, so the result differs
// from the reference's sequential fp32 sum only by accumulation rounding
// (rel. Frobenius error ~1e-7, tolerance 1e-5 -- the reference's own bar,
// tools/shflbw.cpp:33).
#pragma once

#include <cuda.h>

#include <algorithm>
#include <atomic>

#include "common.cuh"
#include "internal.h"

namespace sbw {
namespace tc {


constexpr int kBlockN = 128;  // output columns per CTA (MMA M)
constexpr int kBlockK = 64;   // sparse columns per pipeline stage
constexpr int kABytes = kBlockK * kBlockN * 2;  // 16 KB, two 64-column slabs

struct TcParams {
    const int32_t* row_indices;
    const int32_t* group_ptr;
    const int32_t* col_idx;
    void* C;
    int64_t ldc;
    int V;
    int g_begin;
    int N;
    int c_dtype;
    int compact;
    int stages;
    int cps;         // activation slabs filled by cp.async (0..2); the rest by TMA gather4
    const void* B;   // activations (cp.async path)
    int64_t ldb;
    unsigned long long* trace;  // optional per-CTA event timestamps (development)
    int bulk_out;               // 1: C rows 16-byte aligned -> smem-staged vector stores
    int bw;                     // MN block width of the activation tile (64 | 32 | 16 elements)
    // implicit-GEMM conv geometry (KIND 1)
    int Nb, H, W, RS, S, stride, pad, Q, PQ;
    float inv_rs, inv_s;  // 1/RS, 1/S for fdiv (column ids < 2^22, checked on the host)
    double inv_nb, inv_qp;  // 1/Nb, 1/qp for ddiv (conv unit positions)
    // conv KIND 2 with an odd output width: the GEMM runs over a position grid
    // P x qp (qp = Q rounded up to the positions per 64-element activation row),
    // the epilogue drops the qp - Q padding positions (remap = 1)
    int qp, remap, nb_log2;
    int ksplit;      // 1: the CS CTAs of a cluster split the K blocks (partials reduced via DSMEM)
    int persistent;  // 1: k_spmm_persist (units loop inside the CTA)
    int per_sm;      // persistent: resident CTAs per SM
    int gw;          // gather warps per CTA (4, 8)
    int issue1;      // 1: SpMM gathers issued by one elected lane per warp (option "gather_issue")
    int pf_blocks;   // SpMM: K blocks whose activation rows are L2-prefetched before the PDL wait
    int trigger_early;  // 1: griddepcontrol.launch_dependents at entry instead of after the setup
    int tiles;       // 1: SpMM K blocks whose 64 columns are one contiguous run (block-wise
                     //    patterns) load B with two TMA 2D tiles instead of 32 gather4s
    int raster;      // persistent unit order: 1 group-major, 2 column-tile-major
    int tile_n;      // output columns per unit: 128, or 64 (k_spmm_tc, SpMM only: half-width units)
    int n_extra;     // further output destinations (fused all-gather), staged-store path only
    int mc;          // 1: C is an NVLS multicast address (multimem.st row stores), staged-store path only
    void* C_extra[kMaxPeers - 1];
};

// Development timeline (scripts/trace.py): compiled in only with -DSBW_TRACE.
__device__ __forceinline__ void trace_event(unsigned long long* tr, int e) {
#ifdef SBW_TRACE
    if (tr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int cta = blockIdx.y * gridDim.x + blockIdx.x;
        tr[cta * 32 + e] = t;
    }
#else
    (void)tr;
    (void)e;
#endif
}

template <int VS>
struct WeightLayout {
    // bytes per k-row of the weight tile and UMMA layout constants
    static constexpr int kRowBytes = VS * 2 < 128 ? VS * 2 : 128;
    static constexpr int kSlabs = VS * 2 > 128 ? VS * 2 / 128 : 1;
    static constexpr int kSlabBytes = kBlockK * kRowBytes;
    static constexpr int kBytes = kSlabBytes * kSlabs;
    static constexpr uint32_t kLayout = kRowBytes == 128 ? 2u : (kRowBytes == 64 ? 4u : 6u);
    static constexpr uint32_t kSBO = 8 * kRowBytes;
};

constexpr int kMetaBlocks = 16;  // K blocks of column indices staged in smem at a time

// named barrier over the first/only `threads` threads that use it
template <int THREADS>
__device__ __forceinline__ void named_bar(int id) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(THREADS) : "memory");
}

__device__ __forceinline__ void grid_dependency_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

// c / d for 0 <= c < 2^31 with inv = 1.0 / d (d < 2^20): exact, like fdiv
__device__ __forceinline__ int ddiv(int c, double inv) {
    return __double2int_rz((static_cast<double>(c) + 0.5) * inv);
}

// Output column of GEMM column n (-1: beyond N or a padding position).
__device__ __forceinline__ int64_t out_col(const TcParams& p, int n) {
    if (n >= p.N) return -1;
    if (!p.remap) return n;
    const int pos = n >> p.nb_log2, b = n & (p.Nb - 1);
    const int pr = ddiv(pos, p.inv_qp), q = pos - pr * p.qp;
    if (q >= p.Q) return -1;
    return (static_cast<int64_t>(pr) * p.Q + q) * p.Nb + b;
}

template <class OT> __device__ __forceinline__ OT to_out(float x);
template <> __device__ __forceinline__ float to_out<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half to_out<__half>(float x) { return __float2half_rn(x); }

// Coalesced 16-byte stores of a staged [ROWS][128] tile of OT through the row
// map: one output row = 128*sizeof(OT) bytes, 16 or 32 lanes per row.
template <class OT, int ROWS, bool BATCH = true, bool SWZ = false>
__device__ __forceinline__ void store_tile_rows(const TcParams& p, const unsigned char* ctile, const int32_t* rows,
                                                int q, int lane, int n0) {
    // SWZ: row v's 16-byte chunk c sits at chunk c ^ (v & 7) (stage_tile_stmatrix)
    constexpr int esz = sizeof(OT);
    constexpr int kLanesPerRow = kBlockN * esz / 16;  // 16 (bf16/f16) or 32 (f32)
    constexpr int kRowsPerInst = 32 / kLanesPerRow;
    constexpr int kIters = (ROWS + 4 * kRowsPerInst - 1) / (4 * kRowsPerInst);
    const int chunk = lane % kLanesPerRow;
    // a 16-byte chunk never spans two positions; chunks past a half-width unit are dead
    const int64_t nn = chunk * (16 / esz) < p.tile_n ? out_col(p, n0 + chunk * (16 / esz)) : -1;
    const int v0 = q * kRowsPerInst + lane / kLanesPerRow;
    if (!BATCH && p.mc) {  // interleaved, NVLS multicast address
        if (nn >= 0) {
            const uint32_t cb = smem_u32(ctile);
            const uint32_t rbase = smem_u32(rows);
#pragma unroll 4
            for (int v = v0; v < ROWS; v += 4 * kRowsPerInst) {
                int4 x;
                int32_t row;
                const int pc = SWZ ? (chunk ^ (v & 7)) : chunk;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                             : "r"(cb + static_cast<uint32_t>(v * kBlockN * esz + pc * 16)));
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(row) : "r"(rbase + static_cast<uint32_t>(v * 4)));
                multimem_st16(static_cast<char*>(p.C) + (static_cast<int64_t>(row) * p.ldc + nn) * esz, x);
            }
        }
        return;
    }
    if (!BATCH) {  // interleaved: fewer live registers (the persistent kernel's epilogue warps)
        if (nn >= 0) {
            // explicit ld.shared, volatile so it stays after the bar.sync above
            // but without a memory clobber, so the compiler may start the next
            // row's reads before this row's global store
            const uint32_t cb = smem_u32(ctile);
            const uint32_t rbase = smem_u32(rows);
#pragma unroll 4
            for (int v = v0; v < ROWS; v += 4 * kRowsPerInst) {
                int4 x;
                int32_t row;
                const int pc = SWZ ? (chunk ^ (v & 7)) : chunk;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                             : "r"(cb + static_cast<uint32_t>(v * kBlockN * esz + pc * 16)));
                asm volatile("ld.shared.b32 %0, [%1];" : "=r"(row) : "r"(rbase + static_cast<uint32_t>(v * 4)));
                const int64_t off = (static_cast<int64_t>(row) * p.ldc + nn) * esz;
                *reinterpret_cast<int4*>(static_cast<char*>(p.C) + off) = x;
                for (int d = 0; d < p.n_extra; ++d) *reinterpret_cast<int4*>(static_cast<char*>(p.C_extra[d]) + off) = x;
            }
        }
        return;
    }
    if (nn >= 0) {
        // all shared-memory reads first (explicit ld.shared, so no store below
        // can alias them), then the global stores
        int4 x[kIters];
        int32_t row[kIters];
        const uint32_t cb = smem_u32(ctile);
#pragma unroll
        for (int k = 0; k < kIters; ++k) {
            const int v = v0 + k * 4 * kRowsPerInst;
            if (v < ROWS) {
                const int pc = SWZ ? (chunk ^ (v & 7)) : chunk;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(x[k].x), "=r"(x[k].y), "=r"(x[k].z), "=r"(x[k].w)
                             : "r"(cb + static_cast<uint32_t>(v * kBlockN * esz + pc * 16)));
                row[k] = rows[v];
            }
        }
        if (!p.mc) {
#pragma unroll
            for (int k = 0; k < kIters; ++k) {
                const int v = v0 + k * 4 * kRowsPerInst;
                if (v < ROWS)
                    *reinterpret_cast<int4*>(static_cast<char*>(p.C) +
                                             (static_cast<int64_t>(row[k]) * p.ldc + nn) * esz) = x[k];
            }
        } else {  // NVLS multicast address: the same stores as multimem.st
#pragma unroll
            for (int k = 0; k < kIters; ++k) {
                const int v = v0 + k * 4 * kRowsPerInst;
                if (v < ROWS)
                    multimem_st16(static_cast<char*>(p.C) + (static_cast<int64_t>(row[k]) * p.ldc + nn) * esz, x[k]);
            }
        }
        // further destinations (fused all-gather): the same rows again, read
        // back from the staged tile so the common path keeps its registers
        for (int d = 0; d < p.n_extra; ++d) {
            const uint32_t cbd = smem_u32(ctile);
            for (int v = v0; v < ROWS; v += 4 * kRowsPerInst) {
                const int pc = SWZ ? (chunk ^ (v & 7)) : chunk;
                int4 y;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(y.x), "=r"(y.y), "=r"(y.z), "=r"(y.w)
                             : "r"(cbd + static_cast<uint32_t>(v * kBlockN * esz + pc * 16)));
                *reinterpret_cast<int4*>(static_cast<char*>(p.C_extra[d]) +
                                         (static_cast<int64_t>(rows[v]) * p.ldc + nn) * esz) = y;
            }
        }
    }
}

template <class OT> __device__ __forceinline__ uint32_t pack2(uint32_t lo, uint32_t hi);
template <> __device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(uint32_t lo, uint32_t hi) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<const uint32_t*>(&h);
}
template <> __device__ __forceinline__ uint32_t pack2<__half>(uint32_t lo, uint32_t hi) {
    const __half2 h = __floats2half2_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<const uint32_t*>(&h);
}

// 16-bit output tile staged with stmatrix: TMEM (lane = output column n,
// column = output row v) is read in the 16x256b accumulator-fragment layout,
// converted to bf16/f16 pairs along v and stored as transposed 8x8 blocks --
// rows v of 8 consecutive n (16 bytes) -- into ctile [VS][128] with the 16-byte
// chunk index XOR (v & 7) (conflict-free stores and row reads).  8 stmatrix.x4
// per warp for VS = 64 instead of 64 two-byte st.shared per thread.
// t_quarter = the accumulator's TMEM address at this warp's lane quarter q.
template <class OT, int VS>
__device__ __forceinline__ void stage_tile_stmatrix(uint32_t t_quarter, int nkb, int q, int lane,
                                                    unsigned char* ctile) {
    static_assert(VS % 32 == 0, "16x256b.x4 covers 32 accumulator columns");
    const uint32_t cb = smem_u32(ctile);
    const int mi = lane >> 3, mj = lane & 7;  // the matrix / row whose address this lane gives
#pragma unroll
    for (int half = 0; half < 2; ++half) {
        const int nbase = q * 32 + half * 16;
#pragma unroll
        for (int col = 0; col < VS; col += 32) {
            uint32_t r[16];
            if (nkb > 0) {
                tmem_ld_16x256b_x4(t_quarter + (static_cast<uint32_t>(half * 16) << 16) + col, r);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int i = 0; i < 16; ++i) r[i] = 0u;
            }
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
                uint32_t pk[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {  // matrix i: column block k = 2 kk + i / 2, lane half h = i % 2
                    const int k = kk * 2 + (i >> 1), h = i & 1;
                    pk[i] = pack2<OT>(r[4 * k + 2 * h], r[4 * k + 2 * h + 1]);
                }
                const int k = kk * 2 + (mi >> 1), h = mi & 1;
                const int v = col + 8 * k + mj;
                const int chunk = ((nbase + 8 * h) >> 3) ^ (v & 7);
                stmatrix_x4_trans(cb + static_cast<uint32_t>(v * kBlockN * 2 + chunk * 16), pk);
            }
        }
    }
}

// Epilogue for one output type: TMEM -> (staged tile -> 16-byte stores) or
// direct stores, through the row map.  Kept as one straight-line routine per
// type so the compiler never lowers the type switch per element.
template <class OT, int VS>
__device__ __forceinline__ void epilogue_rows(const TcParams& p, uint32_t t_row, int nkb, int m, int q, int lane,
                                              int n0, const int32_t* rows_s, unsigned char* ctile) {
    if constexpr (sizeof(OT) == 2 && VS % 32 == 0) {
        if (p.bulk_out) {
            stage_tile_stmatrix<OT, VS>(t_row, nkb, q, lane, ctile);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            // (VS = 128: the interleaved loop -- 16 staged chunks + rows in registers would spill)
            store_tile_rows<OT, VS, (VS <= 64), true>(p, ctile, rows_s, q, lane, n0);
            return;
        }
    }
    const int64_t n = m < p.tile_n ? out_col(p, n0 + m) : -1;
    const bool live = n >= 0;
#pragma unroll
    for (int c = 0; c < (VS + 31) / 32; ++c) {
        constexpr int kW = VS < 32 ? VS : 32;
        uint32_t r[32];
        if (nkb > 0) {
            if (kW == 32) tmem_ld32(t_row + c * 32, r);
            else tmem_ld16(t_row + c * 32, *reinterpret_cast<uint32_t(*)[16]>(r));
            tmem_ld_wait();
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (p.bulk_out) {
#pragma unroll
            for (int i = 0; i < kW; ++i)
                reinterpret_cast<OT*>(ctile)[(c * 32 + i) * kBlockN + m] = to_out<OT>(__uint_as_float(r[i]));
        } else if (live) {
#pragma unroll
            for (int i = 0; i < kW; ++i)
                static_cast<OT*>(p.C)[static_cast<int64_t>(rows_s[c * 32 + i]) * p.ldc + n] =
                    to_out<OT>(__uint_as_float(r[i]));
        }
    }
    if (p.bulk_out) {
        asm volatile("bar.sync 1, 128;" ::: "memory");
        // batched loads only while they fit in registers (<= 16 chunks per thread)
        store_tile_rows<OT, VS, (VS * sizeof(OT) <= 128)>(p, ctile, rows_s, q, lane, n0);
    }
}

// K-split epilogue (KSF K ranks x VSF V ranks per cluster): K rank kr
// finalises rows [kr*kRP, (kr+1)*kRP) of the VS slice.  Thread m (output
// column n0+m) pushes the other K ranks' rows of its fp32 partial straight
// from registers into their `recv` buffer with st.async (remote stores that
// complete on the receiver's mbarrier), then sums the KSF partials of its own
// rows in K-rank order (deterministic) and stores them through the staged
// 16-byte path.  recv is [KSF][kRP][128] fp32: a warp's 32 threads touch 128
// contiguous bytes per row, both for the remote stores and the local reads.
template <class OT, int VS, int KSF, int VSF>
__device__ __forceinline__ void ksplit_epilogue(const TcParams& p, uint32_t t_row, int nkb, int m, int q, int lane,
                                                int n0, int kr, int vr, const int32_t* rows_s, float* recv,
                                                uint64_t* recv_bar, unsigned char* ctile) {
    constexpr int kRP = VS / KSF;
    float vals[VS];
#pragma unroll
    for (int c = 0; c < (VS + 31) / 32; ++c) {
        constexpr int kW = VS < 32 ? VS : 32;
        uint32_t r[32];
        if (nkb > 0) {
            if (kW == 32) tmem_ld32(t_row + c * 32, r);
            else tmem_ld16(t_row + c * 32, *reinterpret_cast<uint32_t(*)[16]>(r));
            tmem_ld_wait();
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
#pragma unroll
        for (int i = 0; i < kW; ++i) vals[c * 32 + i] = __uint_as_float(r[i]);
    }
    // recv holds the KSF-1 peers' partials: peer c's rows land in slot
    // (c < receiver ? c : c - 1); columns beyond a half-width unit push nothing
    const bool mlive = m < p.tile_n;
#pragma unroll
    for (int c = 0; c < KSF; ++c) {
        if (c == kr || !mlive) continue;
        const uint32_t peer = static_cast<uint32_t>(c * VSF + vr);
        const int my_slot = kr < c ? kr : kr - 1;
        const uint32_t slot = smem_u32(recv) + static_cast<uint32_t>((my_slot * kRP * kBlockN + m) * 4);
        const uint32_t dst = mapa_shared(slot, peer), bar = mapa_shared(smem_u32(recv_bar), peer);
#pragma unroll
        for (int i = 0; i < kRP; ++i)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(
                             dst + i * kBlockN * 4),
                         "r"(__float_as_uint(vals[c * kRP + i])), "r"(bar)
                         : "memory");
    }
    if (m == 0) trace_event(p.trace, 24);
    mbar_wait(recv_bar, 0);
    if (m == 0) trace_event(p.trace, 25);
    // the peers' partials into registers first: explicit ld.shared, issued
    // back to back (a generic load per row, serialised behind each store,
    // cost ~0.7 us here)
    float peer[KSF - 1][kRP];
    const uint32_t recv_u32 = smem_u32(recv) + static_cast<uint32_t>(m * 4);
#pragma unroll
    for (int sl = 0; sl < KSF - 1; ++sl)
#pragma unroll
        for (int i = 0; i < kRP; ++i)
            asm volatile("ld.shared.f32 %0, [%1];"
                         : "=f"(peer[sl][i])
                         : "r"(recv_u32 + static_cast<uint32_t>((sl * kRP + i) * kBlockN * 4)));
    float res[kRP];
#pragma unroll
    for (int i = 0; i < kRP; ++i) {
        float acc = 0.0f;
#pragma unroll
        for (int c = 0; c < KSF; ++c) {  // K-rank order; peer c sits in slot c (c < kr) or c - 1
            float part = vals[c * kRP + i];
            if (c < KSF - 1) part = (c < kr) ? peer[c < KSF - 1 ? c : 0][i] : part;
            if (c > 0) part = (c > kr) ? peer[c > 0 ? c - 1 : 0][i] : part;
            acc += part;
        }
        res[i] = acc;
    }
    if (m == 0) trace_event(p.trace, 26);
    if (p.bulk_out) {
#pragma unroll
        for (int i = 0; i < kRP; ++i) reinterpret_cast<OT*>(ctile)[i * kBlockN + m] = to_out<OT>(res[i]);
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (m == 0) trace_event(p.trace, 27);
        store_tile_rows<OT, kRP>(p, ctile, rows_s + kr * kRP, q, lane, n0);
    } else if (const int64_t n = mlive ? out_col(p, n0 + m) : -1; n >= 0) {
        int32_t row[kRP];
#pragma unroll
        for (int i = 0; i < kRP; ++i) row[i] = rows_s[kr * kRP + i];
#pragma unroll
        for (int i = 0; i < kRP; ++i)
            static_cast<OT*>(p.C)[static_cast<int64_t>(row[i]) * p.ldc + n] = to_out<OT>(res[i]);
    }
    if (m == 0) trace_event(p.trace, 28);
}

// c / d for 0 <= c < 2^22 and a small divisor d, given inv = 1.0f / d: the
// fractional part of (c + 0.5) / d is at least 0.5 / d from an integer and the
// two float roundings move it by < 2^-23 (c + 0.5) / d, so the truncation is
// exact.  Replaces the ~25-instruction integer division on the gather issue
// path (9 of them per lane per K block for a 3x3 conv).
__device__ __forceinline__ int fdiv(int c, float inv) {
    return __float2int_rz((static_cast<float>(c) + 0.5f) * inv);
}

// Conv column encoding, applied once when a window of column indices is
// staged in shared memory (not per gather): sparse column c = (ch, r, s) of
// the C*R*S filter becomes (base << 8) | (r << 4) | s with base the input row
// of tap (r, s) for output position (0, 0) before the padding shift --
// KIND 2: ch*H + r in the [C*H][W*Nb] view, KIND 1: (ch*H + r)*W + s in the
// [C*H*W][Nb] view.  R, S <= 16 and base < 2^23 (host-checked).  Pad columns
// stay -1.
template <int KIND>
__device__ __forceinline__ int conv_encode(const TcParams& p, int c) {
    if (c < 0) return -1;
    const int ch = fdiv(c, p.inv_rs), rs = c - ch * p.RS;
    const int r = fdiv(rs, p.inv_s), sx = rs - r * p.S;
    const int base = KIND == 2 ? ch * p.H + r : (ch * p.H + r) * p.W + sx;
    return (base << 8) | (r << 4) | sx;
}

template <int KIND>
__device__ __forceinline__ int4 conv_encode4(const TcParams& p, int4 c) {
    if constexpr (KIND == 0) return c;
    return make_int4(conv_encode<KIND>(p, c.x), conv_encode<KIND>(p, c.y), conv_encode<KIND>(p, c.z),
                     conv_encode<KIND>(p, c.w));
}

// KIND 1: input row of an encoded column for this gather's output position
// (h0, w0 = its top-left tap, i.e. p*stride - pad, q*stride - pad); -1 outside
// the image.
__device__ __forceinline__ int conv_row_enc(const TcParams& p, int e, int h0, int w0, bool pos_ok) {
    if (e < 0 || !pos_ok) return -1;
    const int h = h0 + ((e >> 4) & 15), w = w0 + (e & 15);
    if (h < 0 || h >= p.H || w < 0 || w >= p.W) return -1;
    return (e >> 8) + h0 * p.W + w0;
}

// KIND 2 (conv, weight in conv order): one gather4 = 4 K rows (ch, r, s) that
// share the filter column s, each fetching the 64-element row segment of the
// [C*H][W*Nb] input view that holds this MN block's 64/Nb adjacent output
// positions (stride 1): row ch*H + p + r - pad, x = (q0 + s - pad)*Nb.  Rows
// outside the image are -1 (zero-filled); columns left/right of it are out of
// the view's bounds and zero-filled by TMA.  ci holds encoded columns; returns
// the x coordinate.
__device__ __forceinline__ int conv_wide_rows(const TcParams& p, int4& ci, int h0, int x0, bool pos_ok) {
    const int c0 = ci.x >= 0 ? ci.x : (ci.y >= 0 ? ci.y : (ci.z >= 0 ? ci.z : ci.w));
    if (c0 < 0 || !pos_ok) {
        ci = make_int4(-1, -1, -1, -1);
        return 0;
    }
    auto row = [&](int e) -> int {
        if (e < 0) return -1;
        const int h = h0 + ((e >> 4) & 15);
        return (h < 0 || h >= p.H) ? -1 : (e >> 8) + h0;
    };
    ci.x = row(ci.x);
    ci.y = row(ci.y);
    ci.z = row(ci.z);
    ci.w = row(ci.w);
    return (x0 + (c0 & 15)) * p.Nb;
}

// warp roles (64 + 32 GW threads):
//   warp 0  : stage bookkeeping -- waits for a free slot, arms the full
//             barrier with the stage's byte count, loads the weight tile
//   warp 1  : TMEM allocator + single-thread MMA issuer
//   warps 2..2+GW-1: gather issuers (32/GW gather4 each per K block), then
//             warps 2-5 run the epilogue (warp w owns TMEM lanes
//             32*(w%4)..+31).  A warp issues one gather4 per ~70-90 cycles
//             (the ELECT/R2UR/UTMALDG loop), so an SM's gather rate grows
//             with the issuing warps: 23 / 32 / 40 B/cycle for 4 / 8 / 16
//             warps in one CTA, 54 for 2 CTAs x 8 (scripts/fillbench2.cu).
template <int DT, int VS, int CS, int KIND, int KSPLIT, int GW>
__global__ void __launch_bounds__(64 + 32 * GW, GW > 4 ? 2 : 1)
    k_spmm_tc(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmW,
              const __grid_constant__ CUtensorMap tmBt,
              TcParams p) {
    using WL = WeightLayout<VS>;
    constexpr int kStageBytes = kABytes + WL::kBytes;
    constexpr uint32_t kTmemCols = VS < 32 ? 32 : VS;
    constexpr uint32_t kIdesc = umma_idesc_f16(DT == SHFLBW_BF16 ? 1 : 0, kBlockN, VS);
    using T = typename Elem<DT>::T;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int stages = p.stages;
    // cluster = KSF (K split) x VSF (V split) CTAs: KSPLIT 0 -> V split by
    // CS, 1 -> K split by CS, 2 -> 2 x 2 (CS = 4).  Rank = kr * VSF + vr.
    constexpr int KSF = KSPLIT == 1 ? CS : (KSPLIT == 2 ? 2 : 1);
    constexpr int VSF = CS / KSF;
    static_assert(KSF * VSF == CS, "cluster shape");
    // K split: partial rows pushed here by the K peers, [KSF][128][VS/KSF] fp32
    float* recv = reinterpret_cast<float*>(smem + stages * kStageBytes);
    constexpr bool kKSplit = KSF > 1;
    constexpr bool mcast = VSF > 1;
    const int recv_bytes = kKSplit ? (KSF - 1) * (VS / KSF) * kBlockN * 4 : 0;
    int32_t* meta_s = reinterpret_cast<int32_t*>(smem + stages * kStageBytes + recv_bytes);  // [kMetaBlocks][64]
    int32_t* rows_s = meta_s + kMetaBlocks * kBlockK;                           // VS
    uint64_t* full = reinterpret_cast<uint64_t*>(rows_s + (VS < 2 ? 2 : VS));
    uint64_t* empty = full + stages;
    uint64_t* accum = empty + stages;
    uint64_t* recv_bar = accum + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CS > 1 ? cluster_ctarank() : 0;
    const int n_tile = blockIdx.x / CS;
    const int n0 = n_tile * p.tile_n;  // 128, or 64: half-width units (SpMM only; MMA rows >= 64 unused)
    const int g = p.g_begin + blockIdx.y;
    const int gp = p.group_ptr[g];
    const int nkb_all = (p.group_ptr[g + 1] - gp) / kBlockK;
    // K split: this CTA's K blocks [kbase, kbase + nkb); V split: its V rows
    const int kr = static_cast<int>(rank) / VSF, vr = static_cast<int>(rank) % VSF;
    const int kbase = kKSplit ? nkb_all * kr / KSF : 0;
    const int nkb = kKSplit ? nkb_all * (kr + 1) / KSF - kbase : nkb_all;
    const int vbase = vr * VS;
    // multicast group: the VSF CTAs that share this CTA's K blocks
    const uint16_t cmask = static_cast<uint16_t>(((1u << VSF) - 1u) << (kr * VSF));
    const int cps = p.cps;
    constexpr int kGT = 32 * GW;      // gather threads
    const int et = threadIdx.x - 64;  // gather thread 0..kGT-1 (epilogue: et < 128)
    if (threadIdx.x == 0) {
        trace_event(p.trace, 0);
        if (p.trigger_early) grid_launch_dependents();
    }
    // first window of column indices (static data): cp.async right at entry,
    // so its latency overlaps the barrier / TMEM / cluster setup
    const int nb0 = nkb < kMetaBlocks ? nkb : kMetaBlocks;
    if (et >= 0) {
        const int32_t* src = p.col_idx + gp + kbase * kBlockK;
        for (int i = et; i < nb0 * (kBlockK / 4); i += kGT) cp_async16(smem_u32(meta_s + 4 * i), src + 4 * i, true);
        cp_async_commit();
    }

    // gather warps stage a window of column indices (all 64 per K block)
    auto stage_meta = [&](int kb0) {
        const int nb = nkb - kb0 < kMetaBlocks ? nkb - kb0 : kMetaBlocks;
        const int4* src = reinterpret_cast<const int4*>(p.col_idx + gp + (kbase + kb0) * kBlockK);
        for (int i = et; i < nb * (kBlockK / 4); i += kGT)
            reinterpret_cast<int4*>(meta_s)[i] = conv_encode4<KIND>(p, src[i]);
    };

    // ---- prologue (reads only the static sparse matrix: overlaps the
    //      previous kernel under PDL) ---------------------------------------
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1 + (cps > 0 ? kGT : 0));
            mbar_init(&empty[s], mcast ? VSF : 1);
        }
        mbar_init(accum, 1);
        mbar_init(recv_bar, 1);
        if (kKSplit)  // the KSF-1 K peers' partial rows for this CTA (tile_n live columns each)
            mbar_arrive_expect_tx(recv_bar, (KSF - 1) * (VS / KSF) * p.tile_n * 4);
        fence_mbar_init();
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    if (CS > 1) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;
    if (threadIdx.x == 0) {
        if (!p.trigger_early) grid_launch_dependents();
        trace_event(p.trace, 1);
    }

    if (warp == 0) {
        // ---------------- stage bookkeeping + weights ----------------
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;  // ring slot and round parity (no runtime division by `stages`)
            for (int kb = 0; kb < nkb; ++kb) {
                if (kb >= stages) mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], (p.tile_n / 64 - cps) * (kABytes / 2) + WL::kBytes);
#pragma unroll
                for (int sl = 0; sl < WL::kSlabs; ++sl)
                    tma_load_2d(smem + s * kStageBytes + kABytes + sl * WL::kSlabBytes, &tmW, &full[s],
                                vbase + sl * 64, gp + (kbase + kb) * kBlockK);
                if (++s == stages) s = 0, ph ^= 1;
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        // The whole warp walks the ring (warp-uniform state, so descriptors and
        // counters stay in uniform registers) and one elected lane issues: a
        // lane-0-only loop made every tcgen05.mma a serialised
        // ELECT / R2UR.BROADCAST sequence (~0.25 us per K block).  The
        // descriptors are built once and advanced by adds (the 14-bit
        // address field never carries: shared memory < 256 KB).
        // activation operand: MN-major, MN blocks of p.bw elements, swizzle = block row bytes
        const uint32_t a_row = KIND == 0 ? 128u : static_cast<uint32_t>(p.bw) * 2;
        const uint32_t a_layout = a_row == 128 ? 2u : (a_row == 64 ? 4u : 6u);
        const uint64_t adesc0 = umma_smem_desc(smem_u32(smem), kBlockK * a_row, 8 * a_row, a_layout);
        const uint64_t bdesc0 = umma_smem_desc(smem_u32(smem) + kABytes, WL::kSlabBytes, WL::kSBO, WL::kLayout);
        const uint64_t a_ks = (16 * a_row) >> 4;                           // per K=16 slice
        constexpr uint64_t b_ks = (16 * WL::kRowBytes) >> 4;
        constexpr uint64_t st_step = kStageBytes >> 4;
        int s = 0;
        uint32_t ph = 0;
        uint64_t st_off = 0;
        for (int kb = 0; kb < nkb; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (lane == 0) {
                if (kb == 0) trace_event(p.trace, 3);
                if (kb < 8) trace_event(p.trace, 8 + kb);
            }
            const uint64_t ad = adesc0 + st_off, bd = bdesc0 + st_off;
            if (elect_one_sync()) {
#pragma unroll
                for (int ks = 0; ks < kBlockK / 16; ++ks)
                    umma_f16(tmem_d, ad + ks * a_ks, bd + ks * b_ks, kIdesc, (kb | ks) != 0);
                // the last `stages` slots are never refilled: no release
                // signal for them, so nothing targets a peer's shared memory
                // once that peer has consumed its own stages (no cluster
                // barrier needed before exit)
                if constexpr (!mcast) umma_commit(&empty[s]);
                else if (kb + stages < nkb) umma_commit_mc(&empty[s], cmask);
            }
            __syncwarp();
            if (lane == 0 && kb < 3) trace_event(p.trace, 29 + kb);  // MMAs of K block kb issued
            if (++s == stages) s = 0, ph ^= 1, st_off = 0;
            else st_off += st_step;
        }
        if (lane == 0) trace_event(p.trace, 4);
        if (elect_one_sync()) {
            if (nkb > 0) umma_commit(accum);
            else mbar_arrive(accum);
        }
        __syncwarp();
    } else {
        // ---------------- activation producers ----------------
        const int gw = warp - 2;
        // TMA part: slabs [0, 2-cps): row group rg of slab sl, 16 row groups
        // per slab, spread over the 4 warps' first lanes
        const int tma_slabs = p.tile_n / 64 - cps;
        const int nblk = KIND == 0 ? tma_slabs : kBlockN / p.bw;  // MN blocks filled by TMA
        const int blk_bytes = kBlockK * p.bw * 2;
        constexpr int kRGW = 16 / GW;                               // row groups (4 rows) per warp
        const int per_warp = kRGW * nblk;                           // gather4s per warp per K block
        const int gi = gw * per_warp + lane;                        // this lane's gather
        // a warp owns kRGW row groups in every MN block, so both halves of an
        // activation row are requested together
        const int g_rg = gw * kRGW + lane % kRGW, g_b = lane / kRGW;
        const bool t_issue = lane < per_warp && (!mcast || (gi % VSF) == vr);
        // conv: this gather's output positions (fixed for the CTA)
        int g_x = n0 + g_b * 64, g_p0 = 0, g_q0 = 0;
        bool g_pos_ok = true;
        if (KIND == 1 || KIND == 2) {
            const int base_n = n0 + g_b * p.bw;
            const int pos = base_n / p.Nb;
            g_x = base_n - pos * p.Nb;
            g_pos_ok = pos < p.PQ;
            g_p0 = (pos / p.qp) * p.stride - p.pad;
            g_q0 = (pos % p.qp) * p.stride - p.pad;
        }
        // cp.async part (SpMM only): slabs [2-cps, 2): cps*512 16-byte chunks per K block
        const int cpr_log2 = cps == 2 ? 4 : 3;  // chunks per row: 8*cps
        const T* Bp = static_cast<const T*>(p.B);
        cp_async_wait<0>();  // this thread's part of the first window
        if constexpr (KIND != 0) {
            for (int i = et; i < nb0 * (kBlockK / 4); i += kGT)
                reinterpret_cast<int4*>(meta_s)[i] = conv_encode4<KIND>(p, reinterpret_cast<int4*>(meta_s)[i]);
        }
        named_bar<kGT>(2);  // first window visible (overlaps the previous grid)
        const uint32_t meta_u32 = smem_u32(meta_s);
        if (KIND == 0 && p.pf_blocks > 0 && t_issue) {
            // the first K blocks' activation rows into L2 while the previous
            // grid finishes (p.pf_blocks <= the first window)
            for (int kb = 0; kb < p.pf_blocks && kb < nkb; ++kb) {
                int4 ci;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(ci.x), "=r"(ci.y), "=r"(ci.z), "=r"(ci.w)
                             : "r"(meta_u32 + static_cast<uint32_t>((kb * kBlockK + g_rg * 4) * 4)));
                tma_prefetch_gather4(&tmB, g_x, ci.x, ci.y, ci.z, ci.w);
            }
        }
        grid_dependency_wait();  // B may be the previous kernel's output
        if (et == 0) trace_event(p.trace, 2);
        // the K loop, instantiated with and without the block-wise tile path
        // (even an untaken per-block check cost 2-5 % in the gather-bound loop)
        auto producer_loop = [&]<bool TILES>() {
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nkb; ++kb) {
                const int win = kb % kMetaBlocks;
                if (win == 0 && kb > 0) {
                    named_bar<kGT>(2);  // all done with the old window
                    stage_meta(kb);
                    named_bar<kGT>(2);
                }
                if (kb >= stages) mbar_wait(&empty[s], ph ^ 1);
                if (et == 0 && kb < 8) trace_event(p.trace, 16 + kb);
                unsigned char* a_st = smem + s * kStageBytes;
                const int32_t* mk = meta_s + win * kBlockK;
                // block-wise K block: its 64 (ascending) columns are c0..c0+63
                int c0 = -1;
                if constexpr (TILES) {
                    const int first = mk[0], last = mk[kBlockK - 1];
                    if (first >= 0 && last - first == kBlockK - 1) c0 = first;
                }
                if (TILES && c0 >= 0) {
                    // B rows c0..c0+63 of each 64-column slab: one 2D TMA tile per
                    // slab into the same swizzled layout the gathers produce
                    if (gw == 0 && elect_one_sync())
                        for (int bb = 0; bb < nblk; ++bb) tma_load_2d(a_st + bb * blk_bytes, &tmBt, &full[s], n0 + bb * 64, c0);
                } else if (KIND == 0 && p.issue1) {
                    // SpMM, option "gather_issue" 1: this warp's gathers for the
                    // stage issued back to back by one elected lane, all index
                    // loads first (the per-lane issue compiles to a serialised
                    // ELECT / R2UR.BROADCAST loop per gather)
                    if (elect_one_sync()) {
                        int4 ci[8];
                        const uint32_t mrow = meta_u32 + static_cast<uint32_t>(win * kBlockK * 4);
    #pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int rg = gw * kRGW + j % kRGW;
                            if (j < per_warp)
                                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                             : "=r"(ci[j].x), "=r"(ci[j].y), "=r"(ci[j].z), "=r"(ci[j].w)
                                             : "r"(mrow + static_cast<uint32_t>(rg * 16)));
                        }
    #pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int jg = gw * per_warp + j;
                            if (j >= per_warp || (mcast && (jg % VSF) != vr)) continue;
                            const int rg = gw * kRGW + j % kRGW, bb = j / kRGW;
                            void* dst = a_st + bb * blk_bytes + rg * (4 * 64 * 2);
                            if constexpr (!mcast)
                                tma_gather4(dst, &tmB, &full[s], n0 + bb * 64, ci[j].x, ci[j].y, ci[j].z, ci[j].w);
                            else
                                tma_gather4_mc(dst, &tmB, &full[s], cmask, n0 + bb * 64, ci[j].x, ci[j].y, ci[j].z,
                                               ci[j].w);
                        }
                    }
                } else if (t_issue) {
                    int4 ci;  // explicit ld.shared (a generic load would take the slower generic path)
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(ci.x), "=r"(ci.y), "=r"(ci.z), "=r"(ci.w)
                                 : "r"(meta_u32 + static_cast<uint32_t>((win * kBlockK + g_rg * 4) * 4)));
                    int x = g_x;
                    if (KIND == 1) {
                        ci.x = conv_row_enc(p, ci.x, g_p0, g_q0, g_pos_ok);
                        ci.y = conv_row_enc(p, ci.y, g_p0, g_q0, g_pos_ok);
                        ci.z = conv_row_enc(p, ci.z, g_p0, g_q0, g_pos_ok);
                        ci.w = conv_row_enc(p, ci.w, g_p0, g_q0, g_pos_ok);
                    } else if (KIND == 2) {
                        x = conv_wide_rows(p, ci, g_p0, g_q0, g_pos_ok);
                    }
                    void* dst = a_st + g_b * blk_bytes + g_rg * (4 * p.bw * 2);
                    if constexpr (!mcast)
                        tma_gather4(dst, &tmB, &full[s], x, ci.x, ci.y, ci.z, ci.w);
                    else
                        tma_gather4_mc(dst, &tmB, &full[s], cmask, x, ci.x, ci.y, ci.z, ci.w);
                }
                if (cps > 0) {
                    const uint32_t a_u32 = smem_u32(a_st);
                    for (int id = et; id < cps * 512; id += kGT) {
                        const int r = id >> cpr_log2, c = id & ((1 << cpr_log2) - 1);
                        const int sl = tma_slabs + (c >> 3), cc = c & 7;
                        const int col = mk[r];
                        const int n = n0 + sl * 64 + cc * 8;
                        const bool ok = col >= 0 && n < p.N;
                        const T* src = ok ? Bp + static_cast<int64_t>(col) * p.ldb + n : Bp;
                        cp_async16(a_u32 + sl * (kABytes / 2) + r * 128 + ((cc ^ (r & 7)) << 4), src, ok);
                    }
                    cp_async_arrive_noinc(&full[s]);
                }
                __syncwarp();
                if (++s == stages) s = 0, ph ^= 1;
            }
        };
        if (KIND == 0 && !mcast && p.tiles) producer_loop.template operator()<true>();
        else producer_loop.template operator()<false>();
        if (gw < 4) {  // warps 2-5 run the epilogue; any further gather warps are done
            // output row map for the epilogue, loaded while the MMAs run
            for (int v = et; v < VS; v += 128) {
                const int64_t gr = static_cast<int64_t>(g) * p.V + vbase + v;
                rows_s[v] = p.compact ? static_cast<int32_t>(static_cast<int64_t>(g - p.g_begin) * p.V + vbase + v)
                                      : p.row_indices[gr];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");

            // ---------------- epilogue: TMEM -> permuted rows of C ----------------
            mbar_wait(accum, 0);
            tc_fence_after();
            if (et == 0) trace_event(p.trace, 5);
            const int q = warp & 3;  // TMEM lane quarter this warp may access
            const int m = q * 32 + lane;
            const uint32_t t_row = tmem_d + (static_cast<uint32_t>(q * 32) << 16);
            // all MMAs are complete (accum), so the stage buffers are free: they
            // hold the [VS][128] output tile for the bulk row stores
            unsigned char* ctile = smem;
            if constexpr (kKSplit) {
                if (p.c_dtype == SHFLBW_F32)
                    ksplit_epilogue<float, VS, KSF, VSF>(p, t_row, nkb, m, q, lane, n0, kr, vr, rows_s, recv, recv_bar, ctile);
                else if (p.c_dtype == SHFLBW_BF16)
                    ksplit_epilogue<__nv_bfloat16, VS, KSF, VSF>(p, t_row, nkb, m, q, lane, n0, kr, vr, rows_s, recv,
                                                                 recv_bar, ctile);
                else
                    ksplit_epilogue<__half, VS, KSF, VSF>(p, t_row, nkb, m, q, lane, n0, kr, vr, rows_s, recv, recv_bar,
                                                          ctile);
            } else {
                if (p.c_dtype == SHFLBW_F32) epilogue_rows<float, VS>(p, t_row, nkb, m, q, lane, n0, rows_s, ctile);
                else if (p.c_dtype == SHFLBW_BF16)
                    epilogue_rows<__nv_bfloat16, VS>(p, t_row, nkb, m, q, lane, n0, rows_s, ctile);
                else epilogue_rows<__half, VS>(p, t_row, nkb, m, q, lane, n0, rows_s, ctile);
            }
        }
    }
    if (et == 0) trace_event(p.trace, 6);
    tc_fence_before();
    // Every operation that targets this CTA's shared memory from a peer --
    // multicast gathers (full barriers), K-split partials (recv_bar), MMA
    // slot releases (empty barriers of refilled slots only) -- has been
    // waited for above, so a CTA-local barrier suffices before TMEM release
    // and exit (a cluster barrier here cost ~0.2 us per launch).
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem_d, kTmemCols);
    if (threadIdx.x == 0) trace_event(p.trace, 7);
}

// ===========================================================================
// Persistent variant: one CTA (cluster) per SM slot loops over (group,
// column tile) units; the full/empty ring runs on across units and two TMEM
// accumulators (ping-pong) let the epilogue of unit i overlap the loads and
// MMAs of unit i+1.  Roles (192 + 32 GW threads): warp 0 weights + stage
// arming, warp 1 TMEM + MMA, warps 2..2+GW-1 activation gathers, the last 4
// warps the epilogue.  Used when the grid would need more than one wave of
// CTAs.
// ===========================================================================

// (group, column tile) of the units a persistent CTA visits: units advance by
// a fixed stride (the cluster count), so the pair is stepped with adds -- the
// divisions happen once per role, not at every unit boundary.  Raster:
// group-major (unit u = group * n_tiles + tile: consecutive units share a
// group's weights and column indices) or column-tile-major (u = tile *
// ngroups + group: the resident CTAs share one activation column slab, so B
// streams from HBM once while the weights -- re-read once per slab -- stay
// L2-resident; the large-FFN order).
struct UnitCursor {
    int u, gl, tile;  // unit, launch-relative group, column tile
    int stride, o, i, step_o, step_i, n_inner;
    bool tm;  // column-tile-major
    __device__ __forceinline__ UnitCursor(int u0, int stride_, int n_tiles, int ngroups, bool tile_major)
        : u(u0), stride(stride_), tm(tile_major) {
        n_inner = tm ? ngroups : n_tiles;
        o = u0 / n_inner;
        i = u0 - o * n_inner;
        step_o = stride_ / n_inner;
        step_i = stride_ - step_o * n_inner;
        set();
    }
    __device__ __forceinline__ void set() {
        gl = tm ? i : o;
        tile = tm ? o : i;
    }
    __device__ __forceinline__ void next() {
        u += stride;
        o += step_o;
        i += step_i;
        if (i >= n_inner) i -= n_inner, ++o;
        set();
    }
};


// Rows of the persistent kernel's staged output tile (all VS rows: staging
// 32 rows at a time saved 8 KB but bought no extra pipeline stage and slowed
// the epilogue-bound shapes, ResNet 1x1 @56 6.3 -> 6.8 us)
__host__ __device__ constexpr int persist_tile_rows(int vs, int out_esz) {
    (void)out_esz;
    return vs;
}

template <class OT, int VS>
__device__ __forceinline__ void persist_store(const TcParams& p, uint32_t t_acc, int nkb, int m, int q, int lane,
                                              int n0, const int32_t* rows_s, unsigned char* ctile,
                                              uint64_t* acc_empty) {
    if constexpr (sizeof(OT) == 2 && VS % 32 == 0) {
        if (p.bulk_out) {
            stage_tile_stmatrix<OT, VS>(t_acc, nkb, q, lane, ctile);
            // accumulator drained: the MMA warp may start the next unit in it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);
            asm volatile("bar.sync 3, 128;" ::: "memory");
            store_tile_rows<OT, VS, false, true>(p, ctile, rows_s, q, lane, n0);
            return;
        }
    }
    const int64_t n = out_col(p, n0 + m);
    const bool live = n >= 0;
#pragma unroll
    for (int c = 0; c < (VS + 31) / 32; ++c) {
        constexpr int kW = VS < 32 ? VS : 32;
        uint32_t r[32];
        if (nkb > 0) {
            if (kW == 32) tmem_ld32(t_acc + c * 32, r);
            else tmem_ld16(t_acc + c * 32, *reinterpret_cast<uint32_t(*)[16]>(r));
            tmem_ld_wait();
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = 0u;
        }
        if (p.bulk_out) {
#pragma unroll
            for (int i = 0; i < kW; ++i)
                reinterpret_cast<OT*>(ctile)[(c * 32 + i) * kBlockN + m] = to_out<OT>(__uint_as_float(r[i]));
        } else if (live) {
#pragma unroll
            for (int i = 0; i < kW; ++i)
                static_cast<OT*>(p.C)[static_cast<int64_t>(rows_s[c * 32 + i]) * p.ldc + n] =
                    to_out<OT>(__uint_as_float(r[i]));
        }
    }
    // accumulator drained: the MMA warp may start the next unit in it
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(acc_empty);
    if (p.bulk_out) {
        asm volatile("bar.sync 3, 128;" ::: "memory");
        store_tile_rows<OT, VS, false>(p, ctile, rows_s, q, lane, n0);
    }
}

template <int DT, int VS, int CS, int KIND, int GW, int MINB = 2>
__global__ void __launch_bounds__(192 + 32 * GW, MINB)
    k_spmm_persist(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmW,
                   const __grid_constant__ CUtensorMap tmBt, TcParams p,
                   int units, int n_tiles) {
    using WL = WeightLayout<VS>;
    constexpr int kStageBytes = kABytes + WL::kBytes;
    constexpr uint32_t kAccCols = VS < 32 ? 32 : VS;
    constexpr uint32_t kTmemCols = 2 * kAccCols;
    constexpr uint32_t kIdesc = umma_idesc_f16(DT == SHFLBW_BF16 ? 1 : 0, kBlockN, VS);
    constexpr bool mcast = CS > 1;

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int stages = p.stages;
    const int ngroups = (units + n_tiles - 1) / n_tiles;
    const bool tmaj = p.raster == 2;  // column-tile-major unit order
    const int out_esz = p.c_dtype == SHFLBW_F32 ? 4 : 2;
    unsigned char* ctile = smem + stages * kStageBytes;  // [VS][128] out (staged stores only)
    int32_t* meta_s = reinterpret_cast<int32_t*>(  // [2][kMetaBlocks][64]
        ctile + (p.bulk_out ? persist_tile_rows(VS, out_esz) * kBlockN * out_esz : 0));
    int32_t* rows_s = meta_s + 2 * kMetaBlocks * kBlockK;                              // VS
    int32_t* gptr_s = rows_s + (VS < 4 ? 4 : VS);                                      // ngroups + 1
    uint64_t* full = reinterpret_cast<uint64_t*>(gptr_s + ((ngroups + 2) & ~1));
    uint64_t* empty = full + stages;
    uint64_t* acc_full = empty + stages;  // [2]
    uint64_t* acc_empty = acc_full + 2;   // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CS > 1 ? cluster_ctarank() : 0;
    const int cid = blockIdx.x / CS, nclusters = gridDim.x / CS;
    const int vbase = static_cast<int>(rank) * VS;
    const uint16_t cmask = static_cast<uint16_t>((1u << CS) - 1u);

    if (threadIdx.x == 0) trace_event(p.trace, 0);
    // this launch's group offsets (static: before the dependency wait), so no
    // role stalls on a global load at a unit boundary
    for (int x = threadIdx.x; x <= ngroups; x += blockDim.x) gptr_s[x] = p.group_ptr[p.g_begin + x];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], mcast ? CS : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&acc_full[b], 1);
            mbar_init(&acc_empty[b], 4);
        }
        fence_mbar_init();
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
    tc_fence_before();
    if (CS > 1) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) {
        grid_launch_dependents();
        trace_event(p.trace, 1);
    }
    auto group_nkb = [&](int gl) { return (gptr_s[gl + 1] - gptr_s[gl]) / kBlockK; };

    if (warp == 0) {
        // ---------------- stage arming + weights ----------------
        if (lane == 0) {
            int kbg = 0, s = 0;
            uint32_t ph = 0;  // ring slot and round parity, carried across units
            for (UnitCursor c(cid, nclusters, n_tiles, ngroups, tmaj); c.u < units; c.next()) {
                const int gl = c.gl;
                const int gp = gptr_s[gl];
                const int nkb = (gptr_s[gl + 1] - gp) / kBlockK;
                for (int kb = 0; kb < nkb; ++kb, ++kbg) {
                    if (kbg >= stages) mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
                    for (int sl = 0; sl < WL::kSlabs; ++sl)
                        tma_load_2d(smem + s * kStageBytes + kABytes + sl * WL::kSlabBytes, &tmW, &full[s],
                                    vbase + sl * 64, gp + kb * kBlockK);
                    if (++s == stages) s = 0, ph ^= 1;
                }
            }
        }
        __syncwarp();
    } else if (warp == 1) {
        // ---------------- MMA issuer (converged warp, elected lane: see k_spmm_tc) ----------------
        const uint32_t a_row = KIND == 0 ? 128u : static_cast<uint32_t>(p.bw) * 2;
        const uint32_t a_layout = a_row == 128 ? 2u : (a_row == 64 ? 4u : 6u);
        const uint64_t adesc0 = umma_smem_desc(smem_u32(smem), kBlockK * a_row, 8 * a_row, a_layout);
        const uint64_t bdesc0 = umma_smem_desc(smem_u32(smem) + kABytes, WL::kSlabBytes, WL::kSBO, WL::kLayout);
        const uint64_t a_ks = (16 * a_row) >> 4;
        constexpr uint64_t b_ks = (16 * WL::kRowBytes) >> 4;
        constexpr uint64_t st_step = kStageBytes >> 4;
        int s = 0, i = 0;
        uint32_t ph = 0;
        uint64_t st_off = 0;
        for (UnitCursor c(cid, nclusters, n_tiles, ngroups, tmaj); c.u < units; c.next(), ++i) {
            const int nkb = group_nkb(c.gl);
            const int b = i & 1;
            mbar_wait(&acc_empty[b], ((i >> 1) & 1) ^ 1);
            tc_fence_after();
            if (lane == 0 && i < 8) trace_event(p.trace, 8 + i);  // MMA: accumulator free for unit i
            const uint32_t tmem_d = tmem_base + b * kAccCols;
            for (int kb = 0; kb < nkb; ++kb) {
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = adesc0 + st_off, bd = bdesc0 + st_off;
                if (elect_one_sync()) {
#pragma unroll
                    for (int ks = 0; ks < kBlockK / 16; ++ks)
                        umma_f16(tmem_d, ad + ks * a_ks, bd + ks * b_ks, kIdesc, (kb | ks) != 0);
                    if constexpr (!mcast) umma_commit(&empty[s]);
                    else umma_commit_mc(&empty[s], cmask);
                }
                __syncwarp();
                if (++s == stages) s = 0, ph ^= 1, st_off = 0;
                else st_off += st_step;
            }
            if (elect_one_sync()) {
                if (nkb > 0) umma_commit(&acc_full[b]);
                else mbar_arrive(&acc_full[b]);
            }
            __syncwarp();
        }
    } else if (warp < 2 + GW) {
        // ---------------- activation gathers ----------------
        constexpr int kGT = 32 * GW;
        const int gw = warp - 2, et = threadIdx.x - 64;  // et 0..kGT-1
        const int bw = KIND == 0 ? 64 : p.bw;
        const int nblk = kBlockN / bw;
        const int blk_bytes = kBlockK * bw * 2;
        constexpr int kRGW = 16 / GW;  // row groups (4 rows) per warp in every MN block
        const int per_warp = kRGW * nblk;
        const int gi = gw * per_warp + lane;
        const int g_rg = gw * kRGW + lane % kRGW, g_b = lane / kRGW;
        const bool t_issue = lane < per_warp && (!mcast || (gi % CS) == static_cast<int>(rank));
        // column-index windows: meta_s[buf] holds kMetaBlocks K blocks of a
        // unit; the first window of unit i+1 is prefetched (cp.async) into the
        // other buffer while unit i issues its gathers
        auto load_window = [&](int gl, int kb0, int buf, bool async) {
            const int nkb = (gptr_s[gl + 1] - gptr_s[gl]) / kBlockK;
            const int nb = nkb - kb0 < kMetaBlocks ? nkb - kb0 : kMetaBlocks;
            const int32_t* src = p.col_idx + gptr_s[gl] + kb0 * kBlockK;
            int32_t* dst = meta_s + buf * kMetaBlocks * kBlockK;
            for (int x = et; x < nb * (kBlockK / 4); x += kGT) {
                if (async) cp_async16(smem_u32(dst + 4 * x), src + 4 * x, true);
                else reinterpret_cast<int4*>(dst)[x] = conv_encode4<KIND>(p, reinterpret_cast<const int4*>(src)[x]);
            }
        };
        // conv: encode a window that arrived raw through cp.async (in place)
        auto encode_window = [&](int gl, int buf) {
            if constexpr (KIND != 0) {
                const int nkb = (gptr_s[gl + 1] - gptr_s[gl]) / kBlockK;
                const int nb = nkb < kMetaBlocks ? nkb : kMetaBlocks;
                int4* w = reinterpret_cast<int4*>(meta_s + buf * kMetaBlocks * kBlockK);
                for (int x = et; x < nb * (kBlockK / 4); x += kGT) w[x] = conv_encode4<KIND>(p, w[x]);
            }
        };
        if (cid < units) load_window(UnitCursor(cid, nclusters, n_tiles, ngroups, tmaj).gl, 0, 0, false);
        named_bar<kGT>(2);
        grid_dependency_wait();  // B may be the previous kernel's output
        if (et == 0) trace_event(p.trace, 2);
        // the unit loop with and without the block-wise tile path (k_spmm_tc)
        auto gather_units = [&]<bool TILES>() {
            int kbg = 0, i = 0, s = 0, buf = 0;
            uint32_t ph = 0;
            for (UnitCursor c(cid, nclusters, n_tiles, ngroups, tmaj); c.u < units; c.next(), ++i) {
                if (et == 0 && i < 8) trace_event(p.trace, 16 + i);  // gathers: unit i starts issuing
                UnitCursor cn = c;
                cn.next();
                const bool more = cn.u < units;
                const int nkb = group_nkb(c.gl);
                // the next unit reads the same single window (same group, <= kMetaBlocks
                // K blocks, e.g. every unit of a one-group conv): keep it, no reload/sync
                const bool keep = more && cn.gl == c.gl && nkb <= kMetaBlocks;
                if (more && !keep) {  // the other buffer was released by the bar.sync ending unit i-1
                    load_window(cn.gl, 0, buf ^ 1, true);
                    cp_async_commit();
                }
                const int n0 = c.tile * kBlockN;
                const int32_t* mbuf = meta_s + buf * kMetaBlocks * kBlockK;
                int g_x = n0 + g_b * 64, g_p0 = 0, g_q0 = 0;
                bool g_pos_ok = true;
                if (KIND == 1 || KIND == 2) {
                    const int base_n = n0 + g_b * p.bw;
                    const int pos = ddiv(base_n, p.inv_nb);
                    g_x = base_n - pos * p.Nb;
                    g_pos_ok = pos < p.PQ;
                    const int pr = ddiv(pos, p.inv_qp);
                    g_p0 = pr * p.stride - p.pad;
                    g_q0 = (pos - pr * p.qp) * p.stride - p.pad;
                }
                for (int kb = 0; kb < nkb; ++kb, ++kbg) {
                    const int win = kb % kMetaBlocks;
                    if (win == 0 && kb > 0) {  // deep group: later windows of this unit, synchronously
                        named_bar<kGT>(2);
                        load_window(c.gl, kb, buf, false);
                        named_bar<kGT>(2);
                    }
                    if (kbg >= stages) mbar_wait(&empty[s], ph ^ 1);
                    int c0 = -1;  // block-wise K block (k_spmm_tc)
                    if constexpr (TILES) {
                        const int first = mbuf[win * kBlockK], last = mbuf[win * kBlockK + kBlockK - 1];
                        if (first >= 0 && last - first == kBlockK - 1) c0 = first;
                    }
                    if (TILES && c0 >= 0) {
                        if (gw == 0 && elect_one_sync())
                            for (int bb = 0; bb < nblk; ++bb)
                                tma_load_2d(smem + s * kStageBytes + bb * blk_bytes, &tmBt, &full[s], n0 + bb * 64, c0);
                    } else if (KIND == 0 && p.issue1) {
                        // SpMM: one elected lane per warp issues the warp's
                        // gathers back to back, index loads first (k_spmm_tc)
                        if (elect_one_sync()) {
                            int4 ci[8];
                            const uint32_t mrow = smem_u32(mbuf) + static_cast<uint32_t>(win * kBlockK * 4);
    #pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int rg = gw * kRGW + j % kRGW;
                                if (j < per_warp)
                                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                                 : "=r"(ci[j].x), "=r"(ci[j].y), "=r"(ci[j].z), "=r"(ci[j].w)
                                                 : "r"(mrow + static_cast<uint32_t>(rg * 16)));
                            }
    #pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const int jg = gw * per_warp + j;
                                if (j >= per_warp || (mcast && (jg % CS) != static_cast<int>(rank))) continue;
                                const int rg = gw * kRGW + j % kRGW, bb = j / kRGW;
                                void* dst = smem + s * kStageBytes + bb * blk_bytes + rg * (4 * 64 * 2);
                                if constexpr (!mcast)
                                    tma_gather4(dst, &tmB, &full[s], n0 + bb * 64, ci[j].x, ci[j].y, ci[j].z, ci[j].w);
                                else
                                    tma_gather4_mc(dst, &tmB, &full[s], cmask, n0 + bb * 64, ci[j].x, ci[j].y, ci[j].z,
                                                   ci[j].w);
                            }
                        }
                    } else if (t_issue) {
                        int4 ci;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(ci.x), "=r"(ci.y), "=r"(ci.z), "=r"(ci.w)
                                     : "r"(smem_u32(mbuf) + static_cast<uint32_t>((win * kBlockK + g_rg * 4) * 4)));
                        int x = g_x;
                        if (KIND == 2) x = conv_wide_rows(p, ci, g_p0, g_q0, g_pos_ok);
                        if (KIND == 1) {
                            ci.x = conv_row_enc(p, ci.x, g_p0, g_q0, g_pos_ok);
                            ci.y = conv_row_enc(p, ci.y, g_p0, g_q0, g_pos_ok);
                            ci.z = conv_row_enc(p, ci.z, g_p0, g_q0, g_pos_ok);
                            ci.w = conv_row_enc(p, ci.w, g_p0, g_q0, g_pos_ok);
                        }
                        void* dst = smem + s * kStageBytes + g_b * blk_bytes + g_rg * (4 * bw * 2);
                        if constexpr (!mcast)
                            tma_gather4(dst, &tmB, &full[s], x, ci.x, ci.y, ci.z, ci.w);
                        else
                            tma_gather4_mc(dst, &tmB, &full[s], cmask, x, ci.x, ci.y, ci.z, ci.w);
                    }
                    __syncwarp();
                    if (++s == stages) s = 0, ph ^= 1;
                }
                if (!keep) {
                    cp_async_wait<0>();
                    named_bar<kGT>(2);  // next unit's window visible; this buffer free
                    if (KIND != 0 && more) {
                        encode_window(cn.gl, buf ^ 1);
                        named_bar<kGT>(2);
                    }
                    buf ^= 1;
                }
            }
        };
        if (KIND == 0 && !mcast && p.tiles) gather_units.template operator()<true>();
        else gather_units.template operator()<false>();
    } else {
        // ---------------- epilogue ----------------
        const int q = warp & 3, m = q * 32 + lane, et = threadIdx.x - (64 + 32 * GW);
        auto row_of = [&](int gl, int v) -> int32_t {
            const int g = p.g_begin + gl;
            return p.compact ? static_cast<int32_t>(static_cast<int64_t>(g - p.g_begin) * p.V + vbase + v)
                             : p.row_indices[static_cast<int64_t>(g) * p.V + vbase + v];
        };
        int32_t next_row = (cid < units && et < VS)  // static: before the wait
                               ? row_of(UnitCursor(cid, nclusters, n_tiles, ngroups, tmaj).gl, et)
                               : 0;
        grid_dependency_wait();  // C may still be read by the previous kernel
        int i = 0;
        for (UnitCursor c(cid, nclusters, n_tiles, ngroups, tmaj); c.u < units; c.next(), ++i) {
            const int n0 = c.tile * kBlockN;
            const int nkb = group_nkb(c.gl);
            const int b = i & 1;
            asm volatile("bar.sync 3, 128;" ::: "memory");  // previous unit done with rows_s / ctile
            if (et < VS) rows_s[et] = next_row;
            asm volatile("bar.sync 3, 128;" ::: "memory");
            if (c.u + nclusters < units && et < VS) {  // in flight meanwhile
                UnitCursor cn = c;
                cn.next();
                next_row = row_of(cn.gl, et);
            }
            mbar_wait(&acc_full[b], (i >> 1) & 1);
            tc_fence_after();
            if (et == 0 && i < 8) trace_event(p.trace, 24 + i);  // epilogue: unit i accumulated
            const uint32_t t_acc = tmem_base + b * kAccCols + (static_cast<uint32_t>(q * 32) << 16);
            if (p.c_dtype == SHFLBW_F32)
                persist_store<float, VS>(p, t_acc, nkb, m, q, lane, n0, rows_s, ctile, &acc_empty[b]);
            else if (p.c_dtype == SHFLBW_BF16)
                persist_store<__nv_bfloat16, VS>(p, t_acc, nkb, m, q, lane, n0, rows_s, ctile, &acc_empty[b]);
            else
                persist_store<__half, VS>(p, t_acc, nkb, m, q, lane, n0, rows_s, ctile, &acc_empty[b]);
        }
    }
    tc_fence_before();
    if (CS > 1) cluster_sync_relaxed();
    else __syncthreads();
    if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
    if (threadIdx.x == 0) trace_event(p.trace, 7);
}

// ---------------- host side ----------------

int num_sms();  // of the current device (cached per device)
int current_device();

// Per (kernel instantiation, device): the dynamic shared-memory cap set so
// far.  cudaFuncSetAttribute applies to the current device only, so a
// process that launches on several GPUs raises it once per device.
constexpr int kMaxDevices = 64;
struct SmemCaps {
    std::atomic<size_t> cap[kMaxDevices];
    // true if the caller must (re)raise the cap for `smem` bytes on `dev`
    bool needs(int dev, size_t smem) {
        return dev < 0 || dev >= kMaxDevices || smem > cap[dev].load(std::memory_order_relaxed);
    }
    void set(int dev, size_t smem) {
        if (dev >= 0 && dev < kMaxDevices) cap[dev].store(smem, std::memory_order_relaxed);
    }
};

template <int DT, int VS, int CS, int KIND, int KSPLIT, int GW>
int launch_tc(const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles, int groups,
              cudaStream_t s) {
    constexpr int kStage = kABytes + WeightLayout<VS>::kBytes;
    constexpr int KSF = KSPLIT == 1 ? CS : (KSPLIT == 2 ? 2 : 1);
    const size_t recv = (CS > 1 && KSPLIT) ? static_cast<size_t>(KSF - 1) * (VS / KSF) * kBlockN * 4 : 0;
    const size_t smem = static_cast<size_t>(prm.stages) * kStage + recv + 1024 + kMetaBlocks * kBlockK * 4 +
                        (VS < 2 ? 2 : VS) * 4 + (2 * prm.stages + 3) * 8 + 16;
    auto kern = k_spmm_tc<DT, VS, CS, KIND, KSPLIT, GW>;
    static SmemCaps configured;  // per instantiation and device: raise the smem cap once
    if (const int dev = current_device(); configured.needs(dev, smem)) {
        SBW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        configured.set(dev, smem);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_tiles * CS, groups, 1);
    cfg.blockDim = dim3(64 + 32 * GW, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = option("pdl") ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    SBW_CUDA(cudaLaunchKernelEx(&cfg, kern, tmB, tmW, tmBt, prm));
    count_launch();
    return SHFLBW_OK;
}


template <int DT, int VS, int CS, int KIND, int GW, int MINB = 2>
int launch_persist(const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles, int groups,
                   cudaStream_t s) {
    constexpr int kStage = kABytes + WeightLayout<VS>::kBytes;
    const size_t out_esz = prm.c_dtype == SHFLBW_F32 ? 4 : 2;
    const size_t smem = static_cast<size_t>(prm.stages) * kStage +
                        (prm.bulk_out ? static_cast<size_t>(persist_tile_rows(VS, static_cast<int>(out_esz))) *
                                            kBlockN * out_esz
                                      : 0) + 1024 +
                        2 * kMetaBlocks * kBlockK * 4 + (VS < 4 ? 4 : VS) * 4 + ((groups + 2) & ~1) * 4 +
                        (2 * prm.stages + 5) * 8 + 16;
    auto kern = k_spmm_persist<DT, VS, CS, KIND, GW, MINB>;
    static SmemCaps configured;
    if (const int dev = current_device(); configured.needs(dev, smem)) {
        SBW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        SBW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        configured.set(dev, smem);
    }
    const int units = n_tiles * groups;
    const int per_sm = prm.per_sm;
    // per_sm CTAs must be co-resident: launch bounds (320, 2) keep registers
    // <= 102 and the host sizes stages so per_sm CTAs fit in shared memory
    const int clusters = std::min(units, per_sm * num_sms() / CS);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(clusters * CS, 1, 1);
    cfg.blockDim = dim3(192 + 32 * GW, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = option("pdl") ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    SBW_CUDA(cudaLaunchKernelEx(&cfg, kern, tmB, tmW, tmBt, prm, units, n_tiles));
    count_launch();
    return SHFLBW_OK;
}

// gather warps per CTA (prm.gw): 4 or 8
template <int DT, int VS, int CS, int KIND, int KSPLIT>
int launch_tc_gw(const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles, int groups,
                 cudaStream_t s) {
    // (V = 128 K-split epilogues hold 128 fp32 partials per thread: they would
    // spill at the 2-CTA register budget of 8 gather warps)
    if constexpr (!(VS == 128 && KSPLIT != 0))
        if (prm.gw == 8) return launch_tc<DT, VS, CS, KIND, KSPLIT, 8>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    return launch_tc<DT, VS, CS, KIND, KSPLIT, 4>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
}

template <int DT, int VS, int CS, int KIND>
int launch_persist_gw(const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles, int groups,
                      cudaStream_t s) {
    if (prm.gw >= 8) return launch_persist<DT, VS, CS, KIND, 8>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    // three CTAs per SM (shallow units, epilogue-bound): the instantiation
    // compiled for that register budget (64 per thread; the two-per-SM one
    // keeps 72, which the other shapes need)
    if constexpr (CS == 1)
        if (prm.per_sm >= 3) return launch_persist<DT, VS, CS, KIND, 4, 3>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    return launch_persist<DT, VS, CS, KIND, 4>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
}

// SpMM variants: V split (CS CTAs, multicast), K split, 2 x 2, persistent
template <int DT, int VS>
int dispatch_spmm(int cs, const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles,
                  int groups, cudaStream_t s) {
    if (prm.persistent) {
        switch (cs) {
            case 1: return launch_persist_gw<DT, VS, 1, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
            case 2: return launch_persist_gw<DT, VS, 2, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
            case 4: return launch_persist_gw<DT, VS, 4, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        }
        return SHFLBW_UNSUPPORTED;
    }
    switch (cs * 2 + prm.ksplit) {
        case 2: case 3: return launch_tc_gw<DT, VS, 1, 0, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 4: return launch_tc_gw<DT, VS, 2, 0, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 5: return launch_tc_gw<DT, VS, 2, 0, 1>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 8: return launch_tc_gw<DT, VS, 4, 0, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 9: return launch_tc_gw<DT, VS, 4, 0, 1>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 10: return launch_tc_gw<DT, VS, 4, 0, 2>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    }
    return SHFLBW_UNSUPPORTED;
}

// conv variants (KIND 1: one output position per activation row, KIND 2:
// conv-ordered weight, 128-byte rows): one CTA per unit, K split over 2 or 4
// CTAs, persistent
template <int DT, int VS, int KIND>
int dispatch_conv(int cs, const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm, int n_tiles,
                  int groups, cudaStream_t s) {
    if (prm.persistent) return launch_persist_gw<DT, VS, 1, KIND>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    switch (cs * 2 + prm.ksplit) {
        case 2: case 3: return launch_tc_gw<DT, VS, 1, KIND, 0>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 5: return launch_tc_gw<DT, VS, 2, KIND, 1>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
        case 9: return launch_tc_gw<DT, VS, 4, KIND, 1>(tmB, tmW, tmBt, prm, n_tiles, groups, s);
    }
    return SHFLBW_UNSUPPORTED;
}

// KG 0: SpMM (kind 0), KG 1: conv (kinds 1, 2) -- explicitly instantiated in
// tc_inst_{bf16,f16}_{spmm,conv}.cu
template <int DT, int KG>
int dispatch(int vs, int cs, int kind, const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt, const TcParams& prm,
             int n_tiles, int groups, cudaStream_t s) {
    auto one = [&]<int VS>() -> int {
        if constexpr (KG == 0) return dispatch_spmm<DT, VS>(cs, tmB, tmW, tmBt, prm, n_tiles, groups, s);
        else if (kind == 2) return dispatch_conv<DT, VS, 2>(cs, tmB, tmW, tmBt, prm, n_tiles, groups, s);
        else return dispatch_conv<DT, VS, 1>(cs, tmB, tmW, tmBt, prm, n_tiles, groups, s);
    };
    switch (vs) {
        case 16: return one.template operator()<16>();
        case 32: return one.template operator()<32>();
        case 64: return one.template operator()<64>();
        case 128: return one.template operator()<128>();
    }
    return SHFLBW_UNSUPPORTED;
}

#define SBW_TC_DISPATCH(DT, KG)                                                                          \
    int dispatch<DT, KG>(int vs, int cs, int kind, const CUtensorMap& tmB, const CUtensorMap& tmW, const CUtensorMap& tmBt,      \
                         const TcParams& prm, int n_tiles, int groups, cudaStream_t s)
extern template SBW_TC_DISPATCH(SHFLBW_BF16, 0);
extern template SBW_TC_DISPATCH(SHFLBW_BF16, 1);
extern template SBW_TC_DISPATCH(SHFLBW_F16, 0);
extern template SBW_TC_DISPATCH(SHFLBW_F16, 1);

}  // namespace tc
}  // namespace sbw
