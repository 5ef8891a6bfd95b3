// fillbench.cu -- development microbenchmark: how fast can one SM fill shared
// memory with gathered 256-byte rows (the Shfl-BW activation operand)?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -I include -I paper_2203_05016_b200/csrc \
//        scripts/fillbench.cu -o build/fillbench -lcuda && build/fillbench
//
// Every CTA (one per SM) repeatedly fills a 16 KB tile (64 rows x 256 B,
// rows picked by a pseudo-random index list over an L2-resident source) in a
// 4-deep ring, using one of: TMA tile::gather4 (32 instr/tile), TMA 2D tile
// loads of contiguous rows (2 instr/tile, the upper bound), cp.async 16 B,
// or LDG.128 + STS.128.  Reports bytes/cycle/SM and aggregate TB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

#include <vector>

#include "common.cuh"

using namespace sbw;

constexpr int kRows = 64, kRowBytes = 256, kTile = kRows * kRowBytes, kStages = 4, kIters = 512;

template <int MODE>
__global__ void __launch_bounds__(192, 1) fill(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_tile,
                                               const uint16_t* __restrict__ src, const int* __restrict__ idx, int nrows,
                                               unsigned long long* out_cycles, int* sink) {
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kStages];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, et = threadIdx.x - 64;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&full[s], MODE >= 2 ? 128 : 1);
        fence_mbar_init();
    }
    __syncthreads();
    const long long t0 = clock64();
    const int* my_idx = idx + (blockIdx.x * 131) % 4096;
    for (int it = 0; it < kIters; ++it) {
        const int s = it % kStages;
        if (it >= kStages) {  // consumer side: wait for the stage from kStages iterations ago
            mbar_wait(&full[s], ((it / kStages) - 1) & 1);
        }
        unsigned char* dst = sm + s * kTile;
        const int* ix = my_idx + (it * 64) % 2048;
        if (MODE == 0) {  // TMA gather4: 32 instructions (2 slabs x 16 row groups), 4 warps
            if (warp == 0 && lane == 0) mbar_arrive_expect_tx(&full[s], kTile);
            __syncthreads();
            if (warp >= 2 && lane < 8) {
                const int gi = (warp - 2) * 8 + lane, rg = gi & 15, sl = gi >> 4;
                tma_gather4(dst + sl * 8192 + rg * 512, &tm, &full[s], sl * 64, ix[4 * rg], ix[4 * rg + 1],
                            ix[4 * rg + 2], ix[4 * rg + 3]);
            }
        } else if (MODE == 1) {  // TMA 2D tile of 64 contiguous rows, 2 slabs
            if (threadIdx.x == 0) {
                mbar_arrive_expect_tx(&full[s], kTile);
                tma_load_2d(dst, &tm_tile, &full[s], 0, ix[0] & ~63);
                tma_load_2d(dst + 8192, &tm_tile, &full[s], 64, ix[0] & ~63);
            }
        } else if (MODE == 2) {  // cp.async 16 B, 128 threads x 8 chunks
            if (et >= 0) {
                const uint32_t d = smem_u32(dst);
                for (int i = 0; i < 8; ++i) {
                    const int id = i * 128 + et, r = id >> 4, c = id & 15, sl = c >> 3, cc = c & 7;
                    cp_async16(d + sl * 8192 + r * 128 + ((cc ^ (r & 7)) << 4), src + ix[r] * 128 + c * 8, true);
                }
                cp_async_arrive_noinc(&full[s]);
            }
        } else {  // LDG.128 + STS.128
            if (et >= 0) {
                int4 v[8];
                for (int i = 0; i < 8; ++i) {
                    const int id = i * 128 + et, r = id >> 4, c = id & 15;
                    v[i] = *reinterpret_cast<const int4*>(src + ix[r] * 128 + c * 8);
                }
                for (int i = 0; i < 8; ++i) {
                    const int id = i * 128 + et, r = id >> 4, c = id & 15, sl = c >> 3, cc = c & 7;
                    *reinterpret_cast<int4*>(dst + sl * 8192 + r * 128 + ((cc ^ (r & 7)) << 4)) = v[i];
                }
                fence_proxy_async();
                mbar_arrive(&full[s]);
            }
        }
        if (MODE == 1 || MODE == 0) __syncwarp();
    }
    for (int it = kIters - kStages; it < kIters; ++it) mbar_wait(&full[it % kStages], (it / kStages) & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out_cycles[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 64) sink[blockIdx.x] = sm[threadIdx.x];
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int nrows = 32768;  // 8 MB of 256-byte rows: L2 resident
    uint16_t* src;
    cudaMalloc(&src, size_t(nrows) * kRowBytes);
    cudaMemset(src, 1, size_t(nrows) * kRowBytes);
    std::vector<int> h(8192);
    srand(1);
    for (auto& x : h) x = rand() % nrows;
    int* idx;
    cudaMalloc(&idx, h.size() * 4);
    cudaMemcpy(idx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    CUtensorMap tm, tmt;
    cuuint64_t dims[2] = {128, (cuuint64_t)nrows}, strides[1] = {256};
    cuuint32_t box[2] = {64, 1}, boxt[2] = {64, 64}, es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&tmt, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, boxt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cyc;
    int* sink;
    cudaMalloc(&cyc, sms * 8);
    cudaMalloc(&sink, sms * 4);
    const size_t smem = kStages * kTile + 1024;
    const char* names[] = {"TMA gather4 (32/tile)", "TMA 2D tile (2/tile)", "cp.async 16B", "LDG.128+STS.128"};
    void (*kers[])(const CUtensorMap, const CUtensorMap, const uint16_t*, const int*, int, unsigned long long*, int*) = {
        fill<0>, fill<1>, fill<2>, fill<3>};
    for (int m = 0; m < 4; ++m) {
        cudaFuncSetAttribute(kers[m], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            kers[m]<<<sms, 192, smem>>>(tm, tmt, src, idx, nrows, cyc, sink);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            std::vector<unsigned long long> hc(sms);
            cudaMemcpy(hc.data(), cyc, sms * 8, cudaMemcpyDeviceToHost);
            double avg = 0;
            for (auto c : hc) avg += c;
            avg /= sms;
            const double bytes = double(kIters) * kTile;
            if (rep == 1)
                printf("%-24s %s  %.1f B/cycle/SM  %.2f TB/s aggregate (%.3f ms)\n", names[m],
                       err == cudaSuccess ? "ok " : cudaGetErrorString(err), bytes / avg,
                       bytes * sms / (ms * 1e-3) / 1e12, ms);
        }
    }
    return 0;
}
