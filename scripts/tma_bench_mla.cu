// tma_bench_mla.cu — TMA throughput probe for the MLA latent page geometry (dev tool).
// A page is 64 keys x 576 bf16 (72 KiB).  Layout 0 = the pool's row-major page
// ([64 rows][1152 B]); layout 1 = column-block-major page ([9][64 rows][128 B], contiguous
// in box order).  Each CTA streams pages through a ring of STAGES boxes of NB column blocks
// (box = 64 cols x 64 rows x NB blocks) and reports bytes / cycle / SM and total GB/s.
// usage: tma_bench_mla <NB> <grid> <stages> <layout>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

using namespace spd;

__global__ void __launch_bounds__(64, 1)
    bench(const __grid_constant__ CUtensorMap map, int nbox, int pages, int NB, int stages,
          long long* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t full[16];
    const int box_bytes = NB * 64 * 128;
    const int ncb = (8 % NB == 0) ? 8 : 9;
    const int per_page = (ncb + NB - 1) / NB;
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i) mbar_init(&full[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const long long t0 = clock64();
    for (int i = 0; i < nbox + stages; ++i) {
        if (i >= stages) {
            const int s = (i - stages) % stages;
            mbar_wait(&full[s], ((i - stages) / stages) & 1);
        }
        if (i < nbox) {
            const int s = i % stages;
            const int pg = (int)(((long long)blockIdx.x * (nbox / per_page) + i / per_page) % pages);
            const int cb = (i % per_page) * NB;
            mbar_arrive_expect_tx(&full[s], box_bytes);
            tma_load_4d(smem + s * box_bytes, &map, &full[s], 0, 0, cb, pg);
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
    const int NB = argc > 1 ? atoi(argv[1]) : 4;
    const int grid = argc > 2 ? atoi(argv[2]) : 148;
    const int stages = argc > 3 ? atoi(argv[3]) : 4;
    const int layout = argc > 4 ? atoi(argv[4]) : 0;
    const int ncb = (8 % NB == 0) ? 8 : 9;  // NB | 8: boxes never leave the page (no OOB fill)
    const int per_page = (ncb + NB - 1) / NB;
    const int nbox = 600 * per_page;
    void* encp;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &encp, cudaEnableDefault, &q);
    Enc enc = (Enc)encp;
    long long* dout;
    cudaMalloc(&dout, sizeof(long long) * 1024);
    const size_t bytes = (size_t)6 << 30;
    const int pages = (int)(bytes / (64 * 1152));
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    CUtensorMap map;
    cuuint64_t dims[4] = {64, 64, (cuuint64_t)ncb, (cuuint64_t)pages};
    cuuint64_t str0[3] = {1152, 128, 64 * 1152};
    cuuint64_t str1[3] = {128, 64 * 128, 64 * 1152};
    cuuint32_t box[4] = {64, 64, (cuuint32_t)NB, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, layout ? str1 : str0, box,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
    const int smem = stages * NB * 64 * 128 + 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        bench<<<grid, 64, smem>>>(map, nbox, pages, NB, stages, dout);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> cyc(grid);
        cudaMemcpy(cyc.data(), dout, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
        double avg = 0; for (auto c : cyc) avg += c; avg /= grid;
        const double per_cta = (double)nbox * NB * 64 * 128;
        if (rep) printf("NB=%d grid=%d stages=%d layout=%d: %.1f B/cycle/SM, %.0f GB/s, err=%s\n", NB, grid,
                        stages, layout, per_cta / avg, per_cta * grid / (ms * 1e6),
                        cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
