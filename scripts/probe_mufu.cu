// Probe (dev tool): per-SM throughput of the exp2 variants the prefill softmax can use on
// sm_100a — ex2.approx.ftz.f32, ex2.approx.ftz.bf16x2, ex2.approx.f16x2 — and of the packed
// f32x2 FMA.  Every thread runs 8 independent chains; clock64 around the loop, results as
// operations (elements) per clock per SM with 4 warps per SMSP resident.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, float seed, unsigned* sink, long long* cyc) {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) {
        float f = -seed * (float)(threadIdx.x + i) * 1e-3f;
        if (MODE == 0 || MODE == 3) r[i] = __float_as_uint(f);
        else r[i] = 0xbc00bc00u ^ (threadIdx.x + i);
    }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(r[i]));
            if (MODE == 1) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(r[i]));
            if (MODE == 2) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(r[i]));
            if (MODE == 4) {  // cvt.rn.bf16x2.f32 (F2FP.BF16.F32.PACK_AB) feeding back
                asm volatile("cvt.rn.bf16x2.f32 %0, %0, %1;" : "+r"(r[i]) : "f"(__uint_as_float(r[(i + 1) & 7])));
            }
            if (MODE == 5) {  // add.rn.f32.bf16 on both halves (FHADD.BF16 x2)
                float a = __uint_as_float(r[i]);
                asm volatile("{ .reg .b16 lo, hi;\n\t mov.b32 {lo, hi}, %1;\n\t add.rn.f32.bf16 %0, lo, %0;\n\t add.rn.f32.bf16 %0, hi, %0;\n\t}" : "+f"(a) : "r"(r[(i + 3) & 7]));
                r[i] = __float_as_uint(a);
            }
            if (MODE == 6) {  // prmt (truncating bf16x2 pack)
                asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(r[i]) : "r"(r[(i + 1) & 7]));
            }
            if (MODE == 7) {  // max.f32 with immediate (FMNMX)
                asm volatile("max.f32 %0, %0, 0fC2FA0000;" : "+r"(r[i]));
            }
            if (MODE == 3) {
                uint64_t a = ((uint64_t)r[i] << 32) | r[i];
                asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a));
                r[i] = (uint32_t)a ^ (uint32_t)(a >> 32);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    unsigned x = 0;
    for (int i = 0; i < 8; ++i) x ^= r[i];
    if (x == 0x12345678u) sink[0] = x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int per_inst) {
    unsigned* sink;
    long long* cyc;
    cudaMalloc(&sink, 4);
    cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096, threads = 512;
    k<MODE><<<148, threads>>>(iters, 1.f, sink, cyc);
    k<MODE><<<148, threads>>>(iters, 1.f, sink, cyc);
    cudaDeviceSynchronize();
    long long c[148];
    cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    double ops = (double)iters * 8 * threads;  // instructions per SM (per-thread ops)
    printf("{\"op\": \"%s\", \"cycles\": %lld, \"inst_lanes_per_clk_sm\": %.2f, \"elems_per_clk_sm\": %.2f}\n",
           name, c[0], ops / c[0], ops * per_inst / c[0]);
    cudaFree(sink);
    cudaFree(cyc);
}

int main() {
    run<0>("ex2.approx.ftz.f32", 1);
    run<1>("ex2.approx.ftz.bf16x2", 2);
    run<2>("ex2.approx.f16x2", 2);
    run<3>("fma.rn.f32x2 (+xor)", 2);
    run<4>("cvt.rn.bf16x2.f32 (F2FP)", 2);
    run<5>("add.rn.f32.bf16 x2 (FHADD.BF16)", 2);
    run<6>("prmt.b32", 2);
    run<7>("max.f32 imm (FMNMX)", 1);
    return 0;
}
