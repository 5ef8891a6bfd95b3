// fillbench2.cu -- development microbenchmark (second round): shared-memory
// fill rate of gathered 256-byte activation rows per SM as a function of the
// ring depth, the resident CTAs per SM and the load path, including a hybrid
// where TMA tile::gather4 fills one 128-byte slab of every row and cp.async
// the other.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I include -I paper_2203_05016_b200/csrc \
//        scripts/fillbench2.cu -o scripts/bin/fillbench2 && scripts/bin/fillbench2
//
// Each producer iteration fills one 16 KB stage (64 rows x 256 B, rows drawn
// from an index list over an L2-resident 8 MB source) and waits for the stage
// filled STAGES iterations earlier, i.e. STAGES stages are in flight.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "common.cuh"

using namespace sbw;

constexpr int kRows = 64, kTile = kRows * 256, kIters = 768;

// MODE 0: gather4 x 32 (4 warps x 8 lanes); 1: gather4 x 32 issued by one warp
// (32 lanes); 2: cp.async 16 B (128 threads x 8); 3: hybrid (slab 0 gather4 x 16,
// slab 1 cp.async, 128 threads x 4)
template <int MODE, int STAGES, int GW = 4>
__global__ void __launch_bounds__(64 + 32 * GW) fill(const __grid_constant__ CUtensorMap tm, const uint16_t* __restrict__ src,
                                            const int* __restrict__ idx, unsigned long long* out_cycles, int* sink) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES];
    __shared__ int ix_s[2048];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, et = threadIdx.x - 64;
    const int* my_idx = idx + (blockIdx.x * 131) % 4096;
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) ix_s[i] = my_idx[i];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], (MODE == 2 || MODE == 3) ? 1 + 128 : 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    if (warp == 1) return;  // idle (the real kernel's MMA warp)
    for (int it = 0; it < kIters; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) mbar_wait(&full[s], ((it / STAGES) - 1) & 1);
        unsigned char* dst = sm + s * kTile;
        const int* ix = ix_s + (it * 64) % 2048;
        if (warp == 0) {
            if (lane == 0) {
                const uint32_t tx = MODE == 2 ? 0u : (MODE == 3 ? kTile / 2 : kTile);
                mbar_arrive_expect_tx(&full[s], tx);
            }
            __syncwarp();
            continue;
        }
        if ((MODE == 0 || MODE == 4 || MODE == 5) && lane < 32 / GW) {  // 32 gathers over GW warps
            // MODE 4: every row segment 64 bytes off a 128-byte line; MODE 5: aligned, same map
            const int rgw = 16 / GW, rg = (warp - 2) * rgw + lane % rgw, sl = lane / rgw;
            tma_gather4(dst + sl * 8192 + rg * 512, &tm, &full[s], sl * 64 + (MODE == 4 ? 32 : 0), ix[4 * rg], ix[4 * rg + 1],
                        ix[4 * rg + 2], ix[4 * rg + 3]);
        } else if (MODE == 1 && warp == 2) {
            const int gi = lane, rg = gi & 15, sl = gi >> 4;
            tma_gather4(dst + sl * 8192 + rg * 512, &tm, &full[s], sl * 64, ix[4 * rg], ix[4 * rg + 1],
                        ix[4 * rg + 2], ix[4 * rg + 3]);
        } else if (MODE == 2) {
            const uint32_t d = smem_u32(dst);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int id = i * 128 + et, r = id >> 4, c = id & 15, sl = c >> 3, cc = c & 7;
                cp_async16(d + sl * 8192 + r * 128 + ((cc ^ (r & 7)) << 4), src + ix[r] * 128 + c * 8, true);
            }
            cp_async_arrive_noinc(&full[s]);
        } else if (MODE == 3) {
            if (lane < 4) {  // 16 gather4 for slab 0: 4 per warp
                const int rg = (warp - 2) * 4 + lane;
                tma_gather4(dst + rg * 512, &tm, &full[s], 0, ix[4 * rg], ix[4 * rg + 1], ix[4 * rg + 2],
                            ix[4 * rg + 3]);
            }
            const uint32_t d = smem_u32(dst) + 8192;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int id = i * 128 + et, r = id >> 3, cc = id & 7;
                cp_async16(d + r * 128 + ((cc ^ (r & 7)) << 4), src + ix[r] * 128 + 64 + cc * 8, true);
            }
            cp_async_arrive_noinc(&full[s]);
        }
        __syncwarp();
    }
    if (warp == 0 && lane == 0) {
        for (int it = kIters - STAGES; it < kIters; ++it) mbar_wait(&full[it % STAGES], (it / STAGES) & 1);
        out_cycles[blockIdx.x] = clock64() - t0;
        sink[blockIdx.x] = sm[64];
    }
}

CUtensorMap g_wide;  // 384-byte rows (MODE 4/5)

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int MODE, int STAGES, int GW = 4>
void run(const char* name, const CUtensorMap& tm_in, const uint16_t* src, const int* idx, int sms, int per_sm) {
    unsigned long long* cyc;
    int* sink;
    const int grid = sms * per_sm;
    cudaMalloc(&cyc, grid * 8);
    cudaMalloc(&sink, grid * 4);
    const size_t smem = STAGES * kTile + 1024;
    auto k = fill<MODE, STAGES, GW>;
    const CUtensorMap& tm = (MODE == 4 || MODE == 5) ? g_wide : tm_in;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<grid, 64 + 32 * GW, smem>>>(tm, src, idx, cyc, sink);
        cudaEventRecord(e1);
        cudaError_t err = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = double(kIters) * kTile * grid;
        if (rep == 1)
            printf("%-20s GW %2d stages %2d  ctas/SM %d  %s  %.1f B/cycle/SM (at 1965 MHz)  %.2f TB/s  %.3f ms\n", name, GW,
                   STAGES, per_sm, err == cudaSuccess ? "ok " : cudaGetErrorString(err),
                   bytes / sms / (ms * 1e-3 * 1.965e9), bytes / (ms * 1e-3) / 1e12, ms);
        fflush(stdout);
    }
    cudaFree(cyc);
    cudaFree(sink);
}

int main(int argc, char** argv) {
    const int which = argc > 1 ? atoi(argv[1]) : -1;
    const int nrows = argc > 2 ? atoi(argv[2]) : 32768;  // default 8 MB of 256-byte rows: L2 resident
    uint16_t* src;
    cudaMalloc(&src, size_t(nrows) * 256);
    cudaMemset(src, 1, size_t(nrows) * 256);
    std::vector<int> h(8192);
    srand(1);
    for (auto& x : h) x = static_cast<int>((static_cast<long long>(rand()) * 32768 + rand()) % (nrows / 2));
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    CUtensorMap tm;
    cuuint64_t dims[2] = {128, (cuuint64_t)nrows}, strides[1] = {256};
    cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    {
        cuuint64_t dw[2] = {192, (cuuint64_t)nrows * 2 / 3}, sw[1] = {384};
        enc(&g_wide, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dw, sw, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (which < 0 || which == 0) run<5, 4, 4>("gather4 aligned", tm, src, idx, sms, 1);
    if (which < 0 || which == 1) run<4, 4, 4>("gather4 64B-off", tm, src, idx, sms, 1);
    if (which < 0 || which == 2) run<5, 4, 4>("gather4 aligned", tm, src, idx, sms, 2);
    if (which < 0 || which == 3) run<4, 4, 4>("gather4 64B-off", tm, src, idx, sms, 2);
    if (which < 0 || which == 4) run<5, 4, 8>("gather4 aligned", tm, src, idx, sms, 2);
    if (which < 0 || which == 5) run<4, 4, 8>("gather4 64B-off", tm, src, idx, sms, 2);
    return 0;
}
