// tma_bench.cu — standalone TMA throughput probe (not part of libsemipd).
// Each CTA streams NBOX boxes of a 4-D page map (64 cols x R rows x 2 halves x 1 page,
// 128-B swizzle, like the decode / prefill page boxes) through a 4-deep smem ring and
// reports bytes / cycle per SM.  Patterns: 0 = every CTA reads distinct pages (HBM-sized
// buffer), 1 = every CTA reads the same pages (L2-shared), 2 = distinct pages inside a
// small L2-resident buffer, 3 = fully out-of-bounds boxes (TMA zero fill).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_2504_19867_b200/csrc tma_bench.cu -o tma_bench -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace spd;

#ifndef STAGES
#define STAGES 4
#endif

__global__ void __launch_bounds__(64, 1)
    bench(const __grid_constant__ CUtensorMap map, int nbox, int pages, int pattern, int R,
          long long* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES];
    const int box_bytes = R * 256;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long t0 = clock64();
    for (int i = 0; i < nbox + STAGES; ++i) {
        if (i >= STAGES) {  // consume box i - STAGES
            const int s = (i - STAGES) % STAGES;
            mbar_wait(&full[s], ((i - STAGES) / STAGES) & 1);
        }
        if (i < nbox) {
            const int s = i % STAGES;
            int page;
            if (pattern == 3) page = pages + 7;                                 // out of bounds
            else if (pattern == 1) page = i % pages;                            // shared
            else page = (int)(((long long)blockIdx.x * nbox + i) % pages);      // distinct
            mbar_arrive_expect_tx(&full[s], box_bytes);
            tma_load_4d(smem + s * box_bytes, &map, &full[s], 0, 0, 0, page);
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                        CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                        CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    const int R = argc > 1 ? atoi(argv[1]) : 64;
    const int grid = argc > 2 ? atoi(argv[2]) : 74;
    const int nbox = 2000;
    void* encp;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &encp, cudaEnableDefault, &q);
    Enc enc = (Enc)encp;
    long long* dout;
    cudaMalloc(&dout, sizeof(long long) * 1024);
    for (int pattern = 0; pattern < 4; ++pattern) {
        const size_t bytes = pattern == 0 ? (size_t)4 << 30 : (size_t)8 << 20;
        const int pages = (int)(bytes / (R * 256));
        void* buf;
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 1, bytes);
        CUtensorMap map;
        cuuint64_t dims[4] = {64, (cuuint64_t)R, 2, (cuuint64_t)pages};
        cuuint64_t str[3] = {256, 128, (cuuint64_t)R * 256};
        cuuint32_t box[4] = {64, (cuuint32_t)R, 2, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
        const int smem = STAGES * R * 256 + 1024;
        cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0);
            bench<<<grid, 64, smem>>>(map, nbox, pages, pattern, R, dout);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            std::vector<long long> cyc(grid);
            cudaMemcpy(cyc.data(), dout, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
            double avg = 0; for (auto c : cyc) avg += c; avg /= grid;
            const double tot = (double)nbox * R * 256 * grid;
            if (rep) printf("R=%d grid=%d pattern=%d: %.1f B/cycle/SM, %.0f GB/s total, %.3f ms, err=%s\n", R, grid,
                   pattern, (double)nbox * R * 256 / avg, tot / (ms * 1e6), ms,
                   cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(buf);
    }
    return 0;
}
