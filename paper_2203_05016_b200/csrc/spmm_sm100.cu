// spmm_sm100.cu -- K2: Shfl-BW SpMM on the 5th-generation tensor cores.
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
//   * producer warp: for each 64-column K block, 32 TMA tile::gather4
//     instructions (one per lane) fetch the 64 activation rows named by the
//     group's column indices straight into the 128B-swizzled MN-major operand
//     layout; pad columns carry index -1, which TMA zero-fills.  One 2D TMA
//     tile load fetches the group's 64 x VS value block (V contiguous, the
//     reference's column-major group layout, include/shflbw/formats.hpp:14-18).
//     A full/empty mbarrier ring of `stages` slots keeps the loads ahead of
//     the MMAs (the explicit empty barrier is what the literal Alg. 1 lacks,
//     tests/test_pipeline.cpp:50-79).
//   * MMA warp: one elected thread issues 4 x tcgen05.mma (K=16) per block and
//     releases the slot with tcgen05.commit.
//   * epilogue (all 4 warps): tcgen05.ld 32 columns at a time; thread t owns
//     output column n0+t, so for every group row v the warp writes 32
//     consecutive elements of output row row_indices[g*V+v] -- the permuted
//     write-back fused into the epilogue with fully coalesced stores.
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
#include <cuda.h>

#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace sbw {
namespace {

constexpr int kBlockN = 128;  // output columns per CTA (MMA M)
constexpr int kBlockK = 64;   // sparse columns per pipeline stage
constexpr int kABytes = kBlockK * kBlockN * 2;  // 16 KB, two 64-column slabs
constexpr int kThreads = 128;

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
};

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

__device__ __forceinline__ void grid_dependency_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" :::);
}

template <int DT, int VS, int CS>
__global__ void __launch_bounds__(kThreads, 1)
    k_spmm_tc(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmW,
              TcParams p) {
    using WL = WeightLayout<VS>;
    constexpr int kStageBytes = kABytes + WL::kBytes;
    constexpr uint32_t kTmemCols = VS < 32 ? 32 : VS;
    constexpr uint32_t kIdesc = umma_idesc_f16(DT == SHFLBW_BF16 ? 1 : 0, kBlockN, VS);

    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const int stages = p.stages;
    int32_t* meta_s = reinterpret_cast<int32_t*>(smem + stages * kStageBytes);  // kMetaBlocks*64
    int32_t* rows_s = meta_s + kMetaBlocks * kBlockK;                           // VS
    uint64_t* full = reinterpret_cast<uint64_t*>(rows_s + (VS < 2 ? 2 : VS));
    uint64_t* empty = full + stages;
    uint64_t* accum = empty + stages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accum + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CS > 1 ? cluster_ctarank() : 0;
    const int n_tile = blockIdx.x / CS;
    const int n0 = n_tile * kBlockN;
    const int g = p.g_begin + blockIdx.y;
    const int gp = p.group_ptr[g];
    const int nkb = (p.group_ptr[g + 1] - gp) / kBlockK;
    const int vbase = static_cast<int>(rank) * VS;

    // ---- prologue: everything here reads only the (static) sparse matrix,
    //      so with PDL it overlaps the tail of the previous kernel ----------
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CS);
        }
        mbar_init(accum, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmB);
        tma_prefetch_desc(&tmW);
    }
    if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
    for (int v = threadIdx.x; v < VS; v += kThreads) {
        const int64_t gr = static_cast<int64_t>(g) * p.V + vbase + v;
        rows_s[v] = p.compact ? static_cast<int32_t>(static_cast<int64_t>(g - p.g_begin) * p.V + vbase + v)
                              : p.row_indices[gr];
    }
    tc_fence_before();
    if (CS > 1) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;
    if (threadIdx.x == 0) grid_launch_dependents();

    if (warp == 0) {
        // ---------------- producer ----------------
        const int slab = lane >> 4, rg = lane & 15;
        const bool issue_gather = CS == 1 || (lane % CS) == static_cast<int>(rank);
        const int pre = nkb < stages ? nkb : stages;
        // weights of the first `pre` stages and the first index window: no
        // dependency on the previous grid
        if (lane == 0) {
            for (int kb = 0; kb < pre; ++kb) {
                mbar_arrive_expect_tx(&full[kb], kStageBytes);
#pragma unroll
                for (int sl = 0; sl < WL::kSlabs; ++sl)
                    tma_load_2d(smem + kb * kStageBytes + kABytes + sl * WL::kSlabBytes, &tmW, &full[kb],
                                vbase + sl * 64, gp + kb * kBlockK);
            }
        }
        auto stage_meta = [&](int kb) {  // next window of column indices, coalesced
            const int nb = nkb - kb < kMetaBlocks ? nkb - kb : kMetaBlocks;
            const int4* src = reinterpret_cast<const int4*>(p.col_idx + gp + kb * kBlockK);
            for (int i = lane; i < nb * (kBlockK / 4); i += 32) reinterpret_cast<int4*>(meta_s)[i] = src[i];
            __syncwarp();
        };
        if (nkb > 0) stage_meta(0);
        grid_dependency_wait();  // B may be the previous kernel's output
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % stages;
            const int win = kb % kMetaBlocks;
            if (win == 0 && kb > 0) stage_meta(kb);
            unsigned char* a_st = smem + s * kStageBytes;
            if (kb >= pre) {
                mbar_wait(&empty[s], ((kb / stages) & 1) ^ 1);
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], kStageBytes);
#pragma unroll
                    for (int sl = 0; sl < WL::kSlabs; ++sl)
                        tma_load_2d(a_st + kABytes + sl * WL::kSlabBytes, &tmW, &full[s], vbase + sl * 64,
                                    gp + kb * kBlockK);
                }
                __syncwarp();
            }
            if (issue_gather) {
                const int4 ci = reinterpret_cast<const int4*>(meta_s)[win * (kBlockK / 4) + rg];
                void* dst = a_st + slab * (kABytes / 2) + rg * 512;
                if (CS == 1)
                    tma_gather4(dst, &tmB, &full[s], n0 + slab * 64, ci.x, ci.y, ci.z, ci.w);
                else
                    tma_gather4_mc(dst, &tmB, &full[s], static_cast<uint16_t>((1u << CS) - 1u),
                                   n0 + slab * 64, ci.x, ci.y, ci.z, ci.w);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer ----------------
        if (lane == 0) {
            for (int kb = 0; kb < nkb; ++kb) {
                const int s = kb % stages;
                mbar_wait(&full[s], (kb / stages) & 1);
                tc_fence_after();
                const uint32_t a_addr = smem_u32(smem + s * kStageBytes);
                const uint32_t w_addr = a_addr + kABytes;
#pragma unroll
                for (int ks = 0; ks < kBlockK / 16; ++ks) {
                    const uint64_t adesc = umma_smem_desc(a_addr + ks * 16 * 128, kABytes / 2, 1024, 2);
                    const uint64_t bdesc = umma_smem_desc(w_addr + ks * 16 * WL::kRowBytes,
                                                          WL::kSlabBytes, WL::kSBO, WL::kLayout);
                    umma_f16(tmem_d, adesc, bdesc, kIdesc, (kb | ks) != 0);
                }
                if (CS == 1) umma_commit(&empty[s]);
                else umma_commit_mc(&empty[s], static_cast<uint16_t>((1u << CS) - 1u));
            }
            if (nkb > 0) umma_commit(accum);
            else mbar_arrive(accum);
        }
        __syncwarp();
    }

    // ---------------- epilogue: TMEM -> permuted rows of C ----------------
    mbar_wait(accum, 0);
    tc_fence_after();
    grid_dependency_wait();  // C may still be read by the previous kernel
    const int m = warp * 32 + lane;
    const int n = n0 + m;
    const bool live = n < p.N;
    const uint32_t t_row = tmem_d + (static_cast<uint32_t>(warp * 32) << 16);
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
        if (live) {
#pragma unroll
            for (int i = 0; i < kW; ++i) {
                const int64_t off = static_cast<int64_t>(rows_s[c * 32 + i]) * p.ldc + n;
                const float x = __uint_as_float(r[i]);
                if (p.c_dtype == SHFLBW_F32) static_cast<float*>(p.C)[off] = x;
                else if (p.c_dtype == SHFLBW_BF16) static_cast<__nv_bfloat16*>(p.C)[off] = __float2bfloat16_rn(x);
                else static_cast<__half*>(p.C)[off] = __float2half_rn(x);
            }
        }
    }
    tc_fence_before();
    if (CS > 1) cluster_sync();
    else __syncthreads();
    if (warp == 2) tmem_dealloc(tmem_d, kTmemCols);
}

// ---------------- host side ----------------

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

int make_map_2d(CUtensorMap* map, int dt, const void* ptr, uint64_t inner, uint64_t outer,
                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return fail(SHFLBW_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {row_stride_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    const CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult r = enc(map, dt == SHFLBW_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                           2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SHFLBW_CUDA_ERROR, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return SHFLBW_OK;
}

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

template <int DT, int VS, int CS>
int launch_tc(const CUtensorMap& tmB, const CUtensorMap& tmW, const TcParams& prm, int n_tiles, int groups,
              cudaStream_t s) {
    constexpr int kStage = kABytes + WeightLayout<VS>::kBytes;
    const size_t smem = static_cast<size_t>(prm.stages) * kStage + 1024 + kMetaBlocks * kBlockK * 4 +
                        (VS < 2 ? 2 : VS) * 4 + (2 * prm.stages + 2) * 8 + 16;
    auto kern = k_spmm_tc<DT, VS, CS>;
    SBW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(n_tiles * CS, groups, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
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
    SBW_CUDA(cudaLaunchKernelEx(&cfg, kern, tmB, tmW, prm));
    count_launch();
    return SHFLBW_OK;
}

template <int DT, int VS>
int dispatch_cs(int cs, const CUtensorMap& tmB, const CUtensorMap& tmW, const TcParams& prm, int n_tiles,
                int groups, cudaStream_t s) {
    switch (cs) {
        case 1: return launch_tc<DT, VS, 1>(tmB, tmW, prm, n_tiles, groups, s);
        case 2: return launch_tc<DT, VS, 2>(tmB, tmW, prm, n_tiles, groups, s);
        case 4: return launch_tc<DT, VS, 4>(tmB, tmW, prm, n_tiles, groups, s);
    }
    return SHFLBW_UNSUPPORTED;
}

template <int DT>
int dispatch_vs(int vs, int cs, const CUtensorMap& tmB, const CUtensorMap& tmW, const TcParams& prm,
                int n_tiles, int groups, cudaStream_t s) {
    switch (vs) {
        case 16: return dispatch_cs<DT, 16>(cs, tmB, tmW, prm, n_tiles, groups, s);
        case 32: return dispatch_cs<DT, 32>(cs, tmB, tmW, prm, n_tiles, groups, s);
        case 64: return dispatch_cs<DT, 64>(cs, tmB, tmW, prm, n_tiles, groups, s);
        case 128: return dispatch_cs<DT, 128>(cs, tmB, tmW, prm, n_tiles, groups, s);
    }
    return SHFLBW_UNSUPPORTED;
}

}  // namespace

int spmm_tc(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
            cudaStream_t s) {
    const int V = a->v;
    if (b.kind != 0) return SHFLBW_UNSUPPORTED;
    if (V != 16 && V != 32 && V != 64 && V != 128) return SHFLBW_UNSUPPORTED;
    if (b.ldb % 8 != 0 || (reinterpret_cast<uintptr_t>(b.ptr) & 15) != 0 || b.N <= 0 || b.K <= 0)
        return SHFLBW_UNSUPPORTED;
    const int groups = g_end - g_begin;
    if (groups <= 0) return SHFLBW_OK;
    if (groups > 65535) return SHFLBW_UNSUPPORTED;
    const int n_tiles = (b.N + kBlockN - 1) / kBlockN;

    // cluster split of V: smallest CS that gives ~one CTA per SM, VS >= 16
    int cs = static_cast<int>(option("split"));
    if (cs <= 0) {
        cs = 1;
        const int64_t units = static_cast<int64_t>(n_tiles) * groups;
        while (cs < 4 && V / (cs * 2) >= 16 && units * cs * 2 <= num_sms()) cs *= 2;
    }
    if (cs != 1 && cs != 2 && cs != 4) return fail(SHFLBW_BAD_PARAMS, "split must be 1, 2 or 4");
    if (V % cs != 0 || V / cs < 16) return SHFLBW_UNSUPPORTED;
    const int vs = V / cs;

    TcParams prm{};
    prm.row_indices = a->row_indices;
    prm.group_ptr = a->group_ptr;
    prm.col_idx = a->col_idx;
    prm.C = c.ptr;
    prm.ldc = c.ldc;
    prm.V = V;
    prm.g_begin = g_begin;
    prm.N = b.N;
    prm.c_dtype = c.dtype;
    prm.compact = c.compact;
    int stages = static_cast<int>(option("stages"));
    if (stages <= 0) stages = vs >= 128 ? 3 : 4;
    const int max_kb = (a->cols + kBlockK - 1) / kBlockK;
    if (stages > max_kb) stages = max_kb < 2 ? 2 : max_kb;
    prm.stages = stages;

    CUtensorMap tmB, tmW;
    int st = make_map_2d(&tmB, a->dtype, b.ptr, static_cast<uint64_t>(b.N), static_cast<uint64_t>(b.K),
                         static_cast<uint64_t>(b.ldb) * 2, 64, 1, 128);
    if (st) return st;
    const int wbox = vs < 64 ? vs : 64;
    const int64_t wrows = a->total_cols > 0 ? a->total_cols : 1;
    st = make_map_2d(&tmW, a->dtype, a->values, static_cast<uint64_t>(V), static_cast<uint64_t>(wrows),
                     static_cast<uint64_t>(V) * 2, wbox, kBlockK, wbox * 2);
    if (st) return st;
    return a->dtype == SHFLBW_BF16 ? dispatch_vs<SHFLBW_BF16>(vs, cs, tmB, tmW, prm, n_tiles, groups, s)
                                   : dispatch_vs<SHFLBW_F16>(vs, cs, tmB, tmW, prm, n_tiles, groups, s);
}

}  // namespace sbw
