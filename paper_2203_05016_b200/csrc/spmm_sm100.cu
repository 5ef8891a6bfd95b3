// spmm_sm100.cu -- host side of the tcgen05 SpMM / conv path: tensor maps,
// the launch plan (cluster split, pipeline depth, persistent kernel) and the
// dispatch into the kernels of tc_kernels.cuh (instantiated in tc_inst_*.cu).
// Replaces spmm_execute / conv2d (/root/reference/proj/src/spmm.cpp:76-146,
// :193-291); see tc_kernels.cuh for the kernel design.
#include <cuda.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>

#include "tc_kernels.cuh"

namespace sbw {
namespace tc {

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}

int num_sms() {
    static std::atomic<int> cache[kMaxDevices];  // per device (0 = not queried yet)
    const int dev = current_device();
    if (dev < 0 || dev >= kMaxDevices) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms > 0 ? sms : 148;
    }
    int sms = cache[dev].load(std::memory_order_relaxed);
    if (!sms) {
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
        cache[dev].store(sms, std::memory_order_relaxed);
    }
    return sms;
}

}  // namespace tc

namespace {
using tc::TcParams;
using tc::kBlockN;
using tc::kBlockK;
using tc::kABytes;
using tc::kMetaBlocks;
using tc::num_sms;

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

// Encoding a tensor map costs ~1-2 us of host time; repeated calls on the same
// buffers (weights every call, activations in steady state) hit this small
// per-thread direct-mapped cache instead.
struct MapKey {
    const void* ptr;
    uint64_t inner, outer, stride;
    uint32_t box_inner, box_outer;
    int dt, swz;
    bool operator==(const MapKey& o) const {
        return ptr == o.ptr && inner == o.inner && outer == o.outer && stride == o.stride &&
               box_inner == o.box_inner && box_outer == o.box_outer && dt == o.dt && swz == o.swz;
    }
};
struct MapEntry {
    MapKey key{};
    CUtensorMap map;
    bool valid = false;
};

int encode_map_2d(CUtensorMap* map, int dt, const void* ptr, uint64_t inner, uint64_t outer,
                  uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

int make_map_2d(CUtensorMap* map, int dt, const void* ptr, uint64_t inner, uint64_t outer,
                uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
    thread_local MapEntry cache[16];
    const MapKey key{ptr, inner, outer, row_stride_bytes, box_inner, box_outer, dt, swizzle_bytes};
    const size_t h = (reinterpret_cast<uintptr_t>(ptr) >> 8 ^ inner * 31 ^ outer * 17 ^ box_inner * 7 ^
                      static_cast<size_t>(swizzle_bytes)) & 15;
    MapEntry& e = cache[h];
    if (e.valid && e.key == key) {
        *map = e.map;
        return SHFLBW_OK;
    }
    const int st = encode_map_2d(map, dt, ptr, inner, outer, row_stride_bytes, box_inner, box_outer, swizzle_bytes);
    if (st == SHFLBW_OK) {
        e.key = key;
        e.map = *map;
        e.valid = true;
    }
    return st;
}

int encode_map_2d(CUtensorMap* map, int dt, const void* ptr, uint64_t inner, uint64_t outer,
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

}  // namespace

int spmm_tc(const shflbw_cu_matrix* a, int g_begin, int g_end, const Operand& b, const OutSpec& c,
            cudaStream_t s) {
    auto unsup = [](const char* why) { return fail(SHFLBW_UNSUPPORTED, std::string("tcgen05 path: ") + why); };
    const int V = a->v;
    if (V != 16 && V != 32 && V != 64 && V != 128) return unsup("V must be 16, 32, 64 or 128");
    if ((reinterpret_cast<uintptr_t>(b.ptr) & 15) != 0 || b.N <= 0 || b.K <= 0)
        return unsup("the activation operand must be 16-byte aligned and non-empty");
    int bw = 64;
    if (b.kind == 0) {
        if (b.ldb % 8 != 0) return unsup("ldb must be a multiple of 8 elements (16-byte rows)");
    } else if (b.kind == 2) {
        // conv order: 128-byte rows of the [C*H][W*Nb] view (capi.cu checked
        // stride 1, Nb in {16, 32}, 64/Nb | Q)
        bw = 64;
    } else {
        // conv: rows of the [C*H*W][Nb] view are Nb contiguous elements
        if (b.Nb == 16 || b.Nb == 32) bw = b.Nb;
        else if (b.Nb % 64 == 0) bw = 64;
        else return unsup("conv batch N must be 16, 32 or a multiple of 64");
        if (static_cast<int64_t>(b.C) * b.H * b.W >= (1LL << 31)) return unsup("conv input exceeds 2^31 rows");
    }
    // conv column encoding (tc_kernels.cuh conv_encode): fdiv's exact range,
    // R, S <= 16 and the tap's base row < 2^23
    if (b.kind != 0 && (b.K >= (1 << 22) || b.R > 16 || b.S > 16 ||
                        static_cast<int64_t>(b.C) * b.H * (b.kind == 1 ? b.W : 1) >= (1LL << 23)))
        return unsup("conv geometry outside the column encoding (R, S <= 16, C*R*S < 2^22)");
    const int groups = g_end - g_begin;
    if (groups <= 0) return SHFLBW_OK;
    if (groups > 65535) return unsup("more than 65535 groups");
    // conv KIND 2 with Q not a multiple of the positions per 64-element
    // activation row: GEMM over a P x qp position grid, padding dropped in the
    // epilogue (TcParams::remap)
    const int ppb = b.kind == 2 ? 64 / b.Nb : 1;
    const int qp = b.kind == 2 ? (b.Q + ppb - 1) / ppb * ppb : b.Q;
    const int64_t n_gemm = b.kind == 2 ? static_cast<int64_t>(b.P) * qp * b.Nb : b.N;
    if (n_gemm > 0x7fffff00LL) return unsup("GEMM N exceeds 2^31");
    // Cluster split for grids that would leave SMs idle: CS CTAs share one
    // (group, column tile).  Modes ("split_mode"):
    //   3  V split: each CTA owns V/CS rows; the activation tile is multicast
    //      to all CS CTAs (bit-identical to CS = 1);
    //   1  K split: each gathers 1/CS of the K blocks, fp32 partials reduced
    //      through DSMEM;
    //   2  2 x 2 (CS = 4): V split over a CTA pair (multicast) and K split
    //      over two pairs -- half the gathers per SM, VS/2 rows per CTA cross
    //      DSMEM;
    //   0  auto (default): an explicit "split" means V split; otherwise by
    //      the widest group's K blocks and how many CTAs per unit fit on the
    //      GPU (measured): >= 24 K blocks and 4 fit -> K split
    //      by 4; >= 8 and 4 fit (V >= 64) -> 2 x 2; >= 8 and 2 fit -> K split
    //      by 2; else V split.
    const int min_kb = 2;  // K blocks per CTA worth splitting for
    const int kb_all = (a->cols + kBlockK - 1) / kBlockK;
    const int kb_grp = a->max_group_cols > 0 ? a->max_group_cols / kBlockK : kb_all;  // widest group
    const int64_t mode_opt = option("split_mode");
    if (mode_opt < 0 || mode_opt > 3) return fail(SHFLBW_BAD_PARAMS, "split_mode must be 0..3");
    struct Split {
        int cs;
        int64_t mode;
        bool hybrid, vsplit;
    };
    auto choose_split = [&](int64_t units) {
        Split r{static_cast<int>(option("split")), mode_opt, false, false};
        if (r.mode == 0) {
            r.mode = 3;
            if (r.cs <= 0 && b.kind == 0 && kb_grp >= 4 && kb_grp < 8 && units * 4 <= num_sms() && V <= 64) {
                // shallow groups on a small grid: 2 x 2 (attention projection
                // N=128 50 %: V=32 2.75 -> 2.42 us, V=64 2.70 -> 2.49)
                r.mode = 2;
            } else if (r.cs <= 0 && b.kind == 0 && kb_grp >= 8) {
                const bool fit4 = units * 4 <= num_sms(), fit2 = units * 2 <= num_sms();
                const bool fit2x2 = units * 2 <= 2LL * num_sms();  // two CTAs per SM
                if (fit4 && kb_grp >= 24) {
                    r.mode = 1;
                    r.cs = 4;
                } else if (fit4 && V >= 64 && (V < 128 || kb_grp >= 16)) {
                    // (128-row groups of < 16 K blocks: the V split by 4, 32
                    // rows per CTA, is faster: FFN2 N=1024 75 % 5.04 -> 4.53
                    // us, north star V=128 4.08 -> 4.01; deeper ones keep the
                    // 2 x 2: FFN2 N=128 50 % 5.05 vs 5.77)
                    r.mode = 2;
                } else if (V <= 64 && ((fit2 && (V < 64 || kb_grp >= 16)) || (!fit2 && fit2x2 && kb_grp >= 16))) {
                    // a K split by 2 for 32-row groups and for deep groups
                    // (>= 16 K blocks, also at two CTAs per SM up to 64 rows:
                    // FFN2 N=1024 50 % V=32 8.07 -> 6.90 us, V=64 7.03 ->
                    // 6.69; at V = 128 the receive buffer costs the second
                    // CTA: FFN2 N=4096 50 % 9.06 -> 18.3, N=128 5.05 -> 7.16;
                    // 128-row groups take the V split); with 64 rows and
                    // shallower groups the multicast V split is faster
                    // (GNMT 50 %: 4.45 vs 4.57-5.24 us)
                    r.mode = 1;
                    r.cs = 2;
                }
            }
        }
        r.hybrid = r.mode == 2 && V >= 32 && (r.cs == 4 || (r.cs <= 0 && units * 4 <= num_sms()));
        r.vsplit = r.mode != 1 && !r.hybrid;
        if (r.hybrid) {
            r.cs = 4;
        } else if (r.cs <= 0) {
            r.cs = 1;
            if (r.vsplit) {
                while (r.cs < 4 && V / (r.cs * 2) >= 16 && units * r.cs * 2 <= num_sms()) r.cs *= 2;
            } else {
                while (r.cs < 4 && units * r.cs * 2 <= num_sms() && kb_all / (r.cs * 2) >= min_kb) r.cs *= 2;
            }
        }
        return r;
    };
    // Output columns per unit ("tile_n"): 128, or 64 -- half-width units
    // (SpMM only): twice the units, each gathering one 64-column activation
    // slab.  Auto: 64 when the 128-column plan (units x cluster split) would
    // still use at most half the SMs -- measured better there (V = 128 north
    // star 5.03 -> 4.54 us, attention projection 2.62 -> 2.56, FFN2 N=128
    // 3.99 -> 3.94) and worse where it only trades a K split for deeper
    // single-CTA units (north star V = 64: 4.2 -> 4.6 us).
    int tile_n = 128;
    {
        const int64_t tn = option("tile_n");
        if (tn != 0 && tn != 64 && tn != 128) return fail(SHFLBW_BAD_PARAMS, "tile_n must be 0, 64 or 128");
        const int64_t units128 = (n_gemm + kBlockN - 1) / kBlockN * groups;
        const Split sp128 = choose_split(units128);
        const int cs128 = sp128.cs;
        const int64_t popt = option("persistent");
        const bool ksplit128 = sp128.hybrid || (cs128 > 1 && !sp128.vsplit);  // K splits never run persistent
        const bool persist128 = !ksplit128 && (popt > 0 || (popt == 0 && units128 * cs128 > 2LL * num_sms()));
        // half-width units: SpMM on the one-CTA-per-unit kernel.  (In the
        // persistent kernel they would fill the last wave of CTA slots better
        // -- ResNet 3x3 @28: 392 units on 296 slots -- but measured slower:
        // @28 10.7 -> 14.9 us, FFN1 N=4096 8.9 -> 13.6 us.)
        const bool can = option("cp_async_slabs") == 0 && n_gemm > 64 && b.kind == 0 && !persist128;
        if (tn == 64 && can) tile_n = 64;
        else if (tn == 0 && can && units128 * cs128 * 2 <= num_sms()) tile_n = 64;
    }
    const int n_tiles = static_cast<int>((n_gemm + tile_n - 1) / tile_n);
    const int64_t units = static_cast<int64_t>(n_tiles) * groups;
    const Split sp = choose_split(units);
    int cs = sp.cs;
    bool hybrid = sp.hybrid;
    const bool vsplit = sp.vsplit;
    bool conv_ksplit = false;
    if (b.kind != 0) {
        // conv: K split only (the gathers' positions depend on the CTA's
        // column tile, not its V rows).  Auto: split deep groups over a CTA
        // pair when the units alone leave SMs idle (measured: ResNet 3x3 @7
        // 35.8 -> 21.4 us; with >= 1 unit per SM the split loses).
        hybrid = false;
        cs = static_cast<int>(option("split"));
        if (cs <= 0) cs = (units < num_sms() && kb_grp >= 6) ? 2 : 1;
        conv_ksplit = cs > 1;
    }
    if (cs != 1 && cs != 2 && cs != 4) return fail(SHFLBW_BAD_PARAMS, "split must be 1, 2 or 4");
    if (b.kind == 0 && vsplit && (V % cs != 0 || V / cs < 16)) return unsup("V split leaves fewer than 16 rows per CTA");
    const int vs = hybrid ? V / 2 : ((vsplit && b.kind == 0) ? V / cs : V);
    const int ksf = hybrid ? 2 : ((vsplit && !conv_ksplit) ? 1 : cs);  // K split factor

    TcParams prm{};
    prm.row_indices = a->row_indices;
    prm.group_ptr = a->group_ptr;
    prm.col_idx = a->col_idx;
    prm.C = c.ptr;
    prm.ldc = c.ldc;
    prm.V = V;
    prm.g_begin = g_begin;
    prm.N = static_cast<int>(n_gemm);
    prm.qp = qp;
    prm.remap = qp != b.Q ? 1 : 0;
    prm.nb_log2 = b.Nb == 16 ? 4 : 5;  // KIND 2: Nb in {16, 32}
    prm.c_dtype = c.dtype;
    prm.compact = c.compact;
    prm.B = b.ptr;
    prm.ldb = b.ldb;
    prm.bw = bw;
    prm.Nb = b.Nb;
    prm.H = b.H;
    prm.W = b.W;
    prm.RS = b.R * b.S;
    prm.S = b.S;
    prm.inv_rs = 1.0f / static_cast<float>(prm.RS > 0 ? prm.RS : 1);
    prm.inv_s = 1.0f / static_cast<float>(b.S > 0 ? b.S : 1);
    prm.inv_nb = 1.0 / static_cast<double>(b.Nb > 0 ? b.Nb : 1);
    prm.inv_qp = 1.0 / static_cast<double>(qp > 0 ? qp : 1);
    prm.stride = b.stride;
    prm.pad = b.pad;
    prm.Q = b.Q;
    prm.PQ = b.P * qp;
    prm.ksplit = hybrid ? 2 : ((cs > 1 && (!vsplit || conv_ksplit)) ? 1 : 0);
    prm.tile_n = tile_n;
    // TMA tile loads for contiguous K blocks: matrices that have them
    // (SHFLBW_CONTIG_BLOCKS); option "tile_loads" -1: gathers only, 1: check
    // every K block of any matrix
    {
        const int64_t tl = option("tile_loads");
        // (the per-block check "last - first == 63" relies on ascending
        // columns: not for folded or conv-ordered matrices)
        const bool ascending = !(a->reserved & (SHFLBW_FOLDED | SHFLBW_CONV_ORDER));
        prm.tiles = b.kind == 0 && ascending && (tl > 0 || (tl == 0 && (a->reserved & SHFLBW_CONTIG_BLOCKS))) ? 1 : 0;
    }
    {
        // SpMM gather issue ("gather_issue"): 1 = one elected lane per warp
        // issues the warp's gathers back to back, 2 = each issuing lane its
        // own (a hardware-serialised per-lane loop); auto = elected for
        // unicast gathers (measured: north star V = 32 4.03 -> 3.64 us, GNMT
        // 50 % 4.58 -> 4.47) and per-lane for multicast ones (north star
        // 3.55 vs 3.80 us, attention projection 2.19 vs 2.37)
        const int64_t gi = option("gather_issue");
        if (gi < 0 || gi > 2) return fail(SHFLBW_BAD_PARAMS, "gather_issue must be 0, 1 or 2");
        const bool multicast = (hybrid || (vsplit && b.kind == 0)) && cs > 1;
        // (the same for the conv KIND 2 producers measured 2x slower: ResNet
        // 3x3 @56 12.4 -> 25.9 us; convs keep the per-lane issue)
        prm.issue1 = b.kind == 0 && (gi == 1 || (gi == 0 && !multicast)) ? 1 : 0;
    }
    {
        // SpMM activation rows of the first K blocks prefetched into L2 (TMA
        // gather4 prefetches) before the programmatic-launch wait ("prefetch":
        // n = n K blocks, -1 = off, 0 = auto = the first column-index window
        // for half-width units only).  Measured: north star V = 128 (64-column
        // units) 4.39 -> 4.12-4.24 us, FFN2 N = 128 3.28 -> 3.25; with
        // 128-column units it costs 1-10 % (north star 3.66 -> 3.68, FFN2 N =
        // 4096 6.84 -> 7.5): the prefetches share the TMA unit with the
        // co-resident previous grid's gathers and delay its completion.  The
        // same through prefetch.global.L2 (no TMA) was no better.
        const int64_t pf = option("prefetch");
        const int64_t want = pf == 0 ? (tile_n == 64 ? kMetaBlocks : 0) : (pf < 0 ? 0 : pf);
        prm.pf_blocks = b.kind != 0 ? 0 : static_cast<int>(want > kMetaBlocks ? kMetaBlocks : want);
        // PDL trigger ("pdl_trigger": 1 = at kernel entry, -1 = after the
        // setup, 0 = auto): at entry only for one-K-block CTAs, whose whole
        // main loop is one gather -- there the successor's earlier prologue
        // pays (GNMT 95 % 2.97 -> 2.67 us); with longer main loops the early
        // successor CTAs slow this grid (north star 3.63 -> 3.88, GNMT 90 %
        // 2.86 -> 3.02, GNMT 50 % 4.57 -> 5.3)
        const int64_t trg = option("pdl_trigger");
        const int kb_cta = (kb_grp + ksf - 1) / ksf;
        prm.trigger_early = trg == 1 || (trg == 0 && kb_cta <= 1) ? 1 : 0;
    }
    {
        const int64_t r = option("raster");
        if (r < 0 || r > 2) return fail(SHFLBW_BAD_PARAMS, "raster must be 0, 1 or 2");
        // auto: column-tile-major (measured: large FFN 474-484 -> 436-454 us,
        // ResNet 3x3 @28 11.8 -> 11.1 us, FFN1 N=4096 9.37 -> 9.16 us; ncu
        // DRAM reads of the large FFN 552 -> 185 MB per launch)
        prm.raster = r ? static_cast<int>(r) : 2;
    }
    prm.cps = b.kind == 0 ? static_cast<int>(option("cp_async_slabs")) : 0;
    if (prm.cps < 0 || prm.cps > 2) return fail(SHFLBW_BAD_PARAMS, "cp_async_slabs must be 0, 1 or 2");
    prm.trace = option("trace") > 1 ? reinterpret_cast<unsigned long long*>(option("trace")) : nullptr;
    {
        const int esz = c.dtype == SHFLBW_F32 ? 4 : 2;
        const bool aligned = (reinterpret_cast<uintptr_t>(c.ptr) % 16 == 0) && ((c.ldc * esz) % 16 == 0) &&
                             ((static_cast<int64_t>(b.N) * esz) % 16 == 0);
        prm.bulk_out = aligned && !option("no_bulk_out") ? 1 : 0;
        if (c.n_extra > 0) {
            // extra destinations are written by the staged 16-byte stores only
            if (!prm.bulk_out) return unsup("peer destinations need 16-byte aligned output rows");
            for (int d = 0; d < c.n_extra; ++d)
                if (reinterpret_cast<uintptr_t>(c.extra[d]) % 16 != 0) return unsup("peer destination not 16-byte aligned");
        }
        prm.n_extra = c.n_extra;
        prm.mc = c.multicast;
        if (c.multicast && !prm.bulk_out) return unsup("multicast output needs 16-byte aligned output rows");
        for (int d = 0; d < c.n_extra; ++d) prm.C_extra[d] = c.extra[d];
    }
    // persistent when one wave of CTAs cannot cover the units (option
    // "persistent": -1 never, 1 always, 0 auto)
    {
        // "persistent": N > 0 -> persistent kernel with N CTAs per SM, -1 never,
        // 0 auto: 2 per SM once the units exceed one wave of 2 CTAs per SM
        // (a partial second wave of one-unit CTAs costs a whole CTA lifetime:
        // ResNet 3x3 @28, 392 units, 12.4 -> 11.8 us; below that the one-CTA-
        // per-unit kernel wins: FFN2 N=4096 256 units 7.4 vs 8.3 us)
        int64_t opt = option("persistent");
        // auto, many shallow SpMM units (<= 4 K blocks, <= 64 rows,
        // unclustered, >= 4 units per SM): 3 CTAs per SM (the 4-gather-warp
        // instantiation for 64 registers per thread) -- more epilogues in
        // flight for these epilogue-bound grids: ResNet 1x1 64->256 @56 18.4
        // -> 17.5 us, 128->512 @28 10.8 -> 10.0, FFN1 N=4096 75 % 8.72 ->
        // 8.33, 90 % 8.07 -> 7.52.  With fewer units (about one per slot:
        // 1x1 512->128 @28, +6 %) or the conv producers (3x3 @56, +4 %) the
        // two-per-SM kernel stays ahead.
        const bool three = cs == 1 && kb_grp <= 4 && vs <= 64 && b.kind == 0 && units >= 4LL * num_sms();
        if (opt == 0) opt = (units * cs > 2LL * num_sms()) ? (three ? 3 : 2) : -1;
        prm.persistent = !prm.ksplit && opt > 0 && groups <= 4096 && tile_n == kBlockN ? 1 : 0;
        prm.per_sm = static_cast<int>(std::min<int64_t>(3, std::max<int64_t>(1, opt)));  // launch bounds: 3 (GW = 4) / 2
    }
    int stages = static_cast<int>(option("stages"));
    if (prm.persistent) {
        // "persistent" = N resident CTAs per SM (1..4).  Gather throughput per
        // SM grows with the number of issuing CTAs; each gets
        // as many stages as its share of shared memory holds (>= 2), with the
        // staged output tile dropped when it would cost a stage.
        const int64_t budget = 232448 / prm.per_sm - 1024;
        const int out_esz = c.dtype == SHFLBW_F32 ? 4 : 2;
        const int64_t tile = static_cast<int64_t>(tc::persist_tile_rows(vs, out_esz)) * kBlockN * out_esz;
        const int64_t fixed = 1024 + 2 * kMetaBlocks * kBlockK * 4 + 4 * 128 + 4 * (groups + 2) + 512;
        const int64_t stage = kABytes + static_cast<int64_t>(kBlockK) * vs * 2;
        const int64_t with_tile = (budget - fixed - tile) / stage, without = (budget - fixed) / stage;
        if (prm.bulk_out && with_tile < 2) {  // the staged epilogue is worth a stage
            if (c.n_extra > 0 || c.multicast) prm.persistent = 0;  // ... unless it carries the extra / multicast stores
            else prm.bulk_out = 0;
        }
        const int64_t fit = prm.bulk_out ? with_tile : without;
        if (fit < 2) prm.persistent = 0;
        else if (stages <= 0 || stages > fit) stages = static_cast<int>(std::min<int64_t>(12, fit));
    }
    if (stages <= 0 && prm.persistent) {
        stages = 2;
    } else if (stages <= 0) {
        stages = vs >= 128 ? 3 : 4;
    }
    // Unclustered grids of at most one CTA per SM: no co-resident pair to
    // keep room for, so the ring goes as deep as the units are (<= 6 stages,
    // one CTA's shared memory): FFN2 N=4096 V=128 7.77 -> 6.60 us, FFN1
    // N=1024 50 % V=128 5.46 -> 4.98, FFN2 N=1024 75 % V=32 5.37 -> 4.95.
    // Cluster splits keep the two-per-SM footprint: measured both ways over
    // the transformer grid (`--grid transformer`), deeper rings there won on
    // some shapes and lost 10-14 % on others (GNMT 50 % 4.51 -> 5.13 us).
    const int kb_cta = (kb_grp + ksf - 1) / ksf;
    const bool deep_ring = !prm.persistent && option("stages") <= 0 && units * cs <= num_sms() && cs == 1 &&
                           !prm.ksplit;
    if (deep_ring) {
        const int64_t recv = prm.ksplit ? static_cast<int64_t>(vs / ksf) * (ksf - 1) * kBlockN * 4 : 0;
        const int64_t fixed = recv + 2048 + kMetaBlocks * kBlockK * 4 + 4 * vs + 256;
        const int64_t stage = kABytes + static_cast<int64_t>(kBlockK) * vs * 2;
        const int fit1 = static_cast<int>((232448 - fixed) / stage);
        const int deep = std::min(std::min(6, fit1), kb_cta);
        if (deep > stages) stages = deep;
    } else if (!prm.persistent && prm.ksplit && option("stages") <= 0) {
        // keep two CTAs per SM next to the DSMEM receive buffer
        const int64_t ksf_rows = vs / ksf * (ksf - 1);
        const int64_t fixed = ksf_rows * kBlockN * 4 + 1024 + kMetaBlocks * kBlockK * 4 + 4 * vs + 256;
        const int64_t stage = kABytes + static_cast<int64_t>(kBlockK) * vs * 2;
        const int fit = static_cast<int>((232448 / 2 - 1024 - fixed) / stage);
        if (fit >= 2 && stages > fit) stages = fit;
    }
    const int max_kb = (kb_grp + ksf - 1) / ksf;  // K blocks per CTA
    if (!prm.persistent && stages > max_kb) stages = max_kb < 2 ? 2 : max_kb;  // the ring spans units otherwise
    prm.stages = stages;
    {
        // gather warps per CTA ("gather_warps", 0 = auto): an SM's gather rate
        // grows with the warps issuing (scripts/fillbench2.cu)
        const int64_t gwo = option("gather_warps");
        // auto: 8 for units of >= 5 K blocks of >= 64 rows without a K split
        // (measured 2-7 % faster: large FFN, FFN2 N=4096, ResNet 3x3 @28/@14;
        // with 32 rows, FFN2 N=4096 V=32, 4 warps: 9.76 -> 9.50 us) and for
        // SpMM K splits of <= 32 V rows per CTA (north star 3.63 -> 3.60 us,
        // V = 32 3.74 -> 3.67; with 64 rows, GNMT 50 %, 4.57 -> 4.63: 4)
        const bool gw8 = (!prm.ksplit && kb_grp >= 5 && vs >= 64) || (prm.ksplit && vs <= 32 && b.kind == 0);
        prm.gw = gwo > 0 ? static_cast<int>(gwo) : (gw8 ? 8 : 4);
        if (prm.gw != 4 && prm.gw != 8) return fail(SHFLBW_BAD_PARAMS, "gather_warps must be 4 or 8");
    }

    CUtensorMap tmB, tmW, tmBt;
    int st;
    if (b.kind == 0)
        st = make_map_2d(&tmB, a->dtype, b.ptr, static_cast<uint64_t>(b.N), static_cast<uint64_t>(b.K),
                         static_cast<uint64_t>(b.ldb) * 2, 64, 1, 128);
    else if (b.kind == 2)
        st = make_map_2d(&tmB, a->dtype, b.ptr, static_cast<uint64_t>(b.W) * b.Nb, static_cast<uint64_t>(b.C) * b.H,
                         static_cast<uint64_t>(b.W) * b.Nb * 2, 64, 1, 128);
    else
        st = make_map_2d(&tmB, a->dtype, b.ptr, static_cast<uint64_t>(b.Nb),
                         static_cast<uint64_t>(b.C) * b.H * b.W, static_cast<uint64_t>(b.Nb) * 2, bw, 1, bw * 2);
    if (st) return st;
    // block-wise K blocks: B as 64-column x 64-row TMA tiles (SpMM only)
    if (b.kind == 0 && prm.tiles) {
        st = make_map_2d(&tmBt, a->dtype, b.ptr, static_cast<uint64_t>(b.N), static_cast<uint64_t>(b.K),
                         static_cast<uint64_t>(b.ldb) * 2, 64, 64, 128);
        if (st) return st;
    } else {
        tmBt = tmB;
    }
    const int wbox = vs < 64 ? vs : 64;
    const int64_t wrows = a->total_cols > 0 ? a->total_cols : 1;
    st = make_map_2d(&tmW, a->dtype, a->values, static_cast<uint64_t>(V), static_cast<uint64_t>(wrows),
                     static_cast<uint64_t>(V) * 2, wbox, kBlockK, wbox * 2);
    if (st) return st;
    {
        const char* split = prm.ksplit == 2 ? "2x2" : (prm.ksplit ? "k" : (cs > 1 ? "v" : "none"));
        std::string plan = std::string(prm.persistent ? "k_spmm_persist" : "k_spmm_tc") +
                           " kind=" + std::to_string(b.kind) + " v=" + std::to_string(V) + " vs=" + std::to_string(vs) +
                           " cs=" + std::to_string(cs) + " split=" + split + " gw=" + std::to_string(prm.gw) +
                           " stages=" + std::to_string(prm.stages) + " n_tiles=" + std::to_string(n_tiles) +
                           " groups=" + std::to_string(groups);
        if (prm.persistent) plan += " per_sm=" + std::to_string(prm.per_sm) + " raster=" + std::to_string(prm.raster);
        plan += " tile_n=" + std::to_string(tile_n);
        if (b.kind == 2 && prm.remap) plan += " remap=1";
        set_plan(plan);
    }
    if (a->dtype == SHFLBW_BF16)
        return b.kind == 0 ? tc::dispatch<SHFLBW_BF16, 0>(vs, cs, b.kind, tmB, tmW, tmBt, prm, n_tiles, groups, s)
                           : tc::dispatch<SHFLBW_BF16, 1>(vs, cs, b.kind, tmB, tmW, tmBt, prm, n_tiles, groups, s);
    return b.kind == 0 ? tc::dispatch<SHFLBW_F16, 0>(vs, cs, b.kind, tmB, tmW, tmBt, prm, n_tiles, groups, s)
                       : tc::dispatch<SHFLBW_F16, 1>(vs, cs, b.kind, tmB, tmW, tmBt, prm, n_tiles, groups, s);
}

}  // namespace sbw
