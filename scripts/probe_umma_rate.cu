// Probe (dev tool): issue rate / execution time of small swap-AB tcgen05.mma shapes used by
// the MLA decode kernel.  One CTA, one issuing thread, REPS x 36 MMAs, clock64 around
// issue and around commit-completion.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include "common.cuh"
using namespace spd;

__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
           ((M >> 4) << 24);
}

__device__ __forceinline__ void umma_ss_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                              uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}

__global__ void rate(int M, int N, int reps, long long* out, int mode) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) { mbar_init(&bar, mode == 3 ? 2 : 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc(&tbase, 256);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (mode == 1 && threadIdx.x < 32) {
        const uint32_t id = idesc(M, N, 0, 0);
        const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 96 * 1024);
        const uint64_t da = umma_desc_sw128(a0, 16, 1024), db = umma_desc_sw128(b0, 16, 1024);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int k = 0; k < 36; ++k) {
                umma_ss_elect(tbase, da + (uint64_t)((k >> 2) * 512 + (k & 3) * 2),
                              db + (uint64_t)((k >> 2) * 128 + (k & 3) * 2), id, k > 0);
            }
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    if (mode == 2) {
        // TMEM load latency while the tensor pipe is busy: warp 0 issues 36*reps MMAs into
        // cols [0,16); warp 1 then loads cols [128,144) and times load -> wait::ld
        const uint32_t id = idesc(M, N, 0, 0);
        const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 96 * 1024);
        const uint64_t da = umma_desc_sw128(a0, 16, 1024), db = umma_desc_sw128(b0, 16, 1024);
        if (threadIdx.x < 32) {
            for (int r = 0; r < reps; ++r)
#pragma unroll
                for (int k = 0; k < 36; ++k)
                    umma_ss_elect(tbase, da + (uint64_t)((k >> 2) * 512 + (k & 3) * 2),
                                  db + (uint64_t)((k >> 2) * 128 + (k & 3) * 2), id, k > 0);
        }
        __syncthreads();
        if (threadIdx.x >= 32 && threadIdx.x < 64) {
            uint32_t r16[16];
            long long t0 = clock64();
            tmem_ld16(tbase + 128, r16);
            tmem_wait_ld();
            long long t1 = clock64();
            if (threadIdx.x == 32) { out[0] = t1 - t0; out[1] = r16[0]; }
        }
        if (threadIdx.x == 0) umma_commit(&bar);
        mbar_wait(&bar, 0);
    }
    if (mode == 3 && threadIdx.x < 64) {
        // two issuing warps, each 36 x reps MMAs into its own accumulator columns: does the
        // aggregate MMA rate grow with a second issuer?
        const uint32_t id = idesc(M, N, 0, 0);
        const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 96 * 1024);
        const uint64_t da = umma_desc_sw128(a0, 16, 1024), db = umma_desc_sw128(b0, 16, 1024);
        const uint32_t dt = tbase + (threadIdx.x >> 5) * 64;
        __syncwarp();
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int k = 0; k < 36; ++k) {
                umma_ss_elect(dt, da + (uint64_t)((k >> 2) * 512 + (k & 3) * 2),
                              db + (uint64_t)((k >> 2) * 128 + (k & 3) * 2), id, k > 0);
            }
        }
        long long t1 = clock64();
        if ((threadIdx.x & 31) == 0) umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    if (mode == 0 && threadIdx.x == 0) {
        const uint32_t id = idesc(M, N, 0, 0);
        const uint32_t a0 = smem_u32(base), b0 = smem_u32(base + 96 * 1024);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
#pragma unroll
            for (int k = 0; k < 36; ++k) {
                const uint32_t a = a0 + (k >> 2) * 8192 + (k & 3) * 32;
                const uint32_t b = b0 + (k >> 2) * 2048 + (k & 3) * 32;
                umma_ss(tbase, umma_desc_sw128(a, 16, 1024), umma_desc_sw128(b, 16, 1024), id, k > 0);
            }
        }
        long long t1 = clock64();
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tbase, 256);
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 170 * 1024);
    const int shapes[][2] = {{64, 16}, {128, 16}, {64, 32}, {128, 32}, {128, 64}, {64, 64}, {128, 128}};
    for (int reps : {0, 1, 4, 16}) {
        rate<<<1, 128, 170 * 1024>>>(64, 16, reps, d, 2);
        long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("tmem ld latency with %d queued M64N16 MMAs: %lld cycles (%s)\n", 36 * reps, h[0],
               cudaGetErrorString(cudaGetLastError()));
    }
    for (auto& s : shapes) {
        for (int mode : {0, 1, 3}) for (int reps : {1, 20}) {
            rate<<<1, 128, 170 * 1024>>>(s[0], s[1], reps, d, mode);
            long long h[2];
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            const int nmma = 36 * reps * (mode == 3 ? 2 : 1);  // mode 3: per-MMA over both warps
            printf("mode=%d M=%d N=%d reps=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", mode, s[0], s[1], reps,
                   (double)h[0] / nmma, (double)h[1] / nmma,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
