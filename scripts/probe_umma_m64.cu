// Probe (dev tool, not part of the library): where does tcgen05.mma M=64 (cta_group::1)
// put its D rows in TMEM, and are the swap-AB MLA decode operand descriptors right?
//   QK: S^T[64 keys x 16 heads] = C[64 x 576] (K-major SW128, [9 cb][64][128 B]) . Q^T
//       (Q K-major SW128 [9 cb][16][128 B]); 36 K16 steps.
//   PV: O^T[128 dv x 16] = V^T (A MN-major: cb 0,1 of C, LBO 8 KiB, SBO 1 KiB) . P^T
//       (B K-major SW128 [16 heads][64 keys]); 4 K16 steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2504_19867_b200/csrc -o /tmp/probe scripts/probe_umma_m64.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include "common.cuh"

using namespace spd;

constexpr int DK = 576, NH = 16, KEYS = 64, NCB = 9;

__host__ __device__ constexpr uint32_t idesc(uint32_t M, uint32_t N, uint32_t a_mn, uint32_t b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((N >> 3) << 17) |
           ((M >> 4) << 24);
}

// swizzled byte offset of (row, col) in a [rows][64 bf16] SW128 block
__host__ __device__ inline uint32_t swz(int row, int col) {
    return row * 128 + ((((col >> 3) ^ (row & 7)) << 4) | ((col & 7) << 1));
}

__global__ void probe(const uint16_t* cimg, const uint16_t* qimg, const uint16_t* pimg,
                      float* s_out, float* o_out, uint32_t lbo, uint32_t sbo) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* cs = base;                       // 9 * 8 KiB
    unsigned char* qs = cs + NCB * KEYS * 128;      // 9 * 2 KiB
    unsigned char* ps = qs + NCB * NH * 128;        // 2 KiB
    __shared__ uint32_t tbase;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x;
    for (int i = tid; i < NCB * KEYS * 64; i += blockDim.x) reinterpret_cast<uint16_t*>(cs)[i] = cimg[i];
    for (int i = tid; i < NCB * NH * 64; i += blockDim.x) reinterpret_cast<uint16_t*>(qs)[i] = qimg[i];
    for (int i = tid; i < NH * 64; i += blockDim.x) reinterpret_cast<uint16_t*>(ps)[i] = pimg[i];
    if (tid == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
    if (tid < 32) tmem_alloc(&tbase, 128);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t t0 = tbase;
    if (tid == 0) {
        const uint32_t id_qk = idesc(64, 16, 0, 0);
        for (int k = 0; k < DK / 16; ++k) {
            const int cb = k >> 2, sub = k & 3;
            uint64_t a = umma_desc_sw128(smem_u32(cs + cb * KEYS * 128) + sub * 32, 16, 1024);
            uint64_t b = umma_desc_sw128(smem_u32(qs + cb * NH * 128) + sub * 32, 16, 1024);
            umma_ss(t0, a, b, id_qk, k > 0);
        }
        const uint32_t id_pv = idesc(128, 16, 1, 0);
        for (int k = 0; k < KEYS / 16; ++k) {
            uint64_t a = umma_desc_sw128(smem_u32(cs) + k * 2048, lbo, sbo);
            uint64_t b = umma_desc_sw128(smem_u32(ps) + k * 32, 16, 1024);
            umma_ss(t0 + 16, a, b, id_pv, k > 0);
        }
        // same QK into TMEM lane offset 16, column 64 (is a lane-16 base legal for M=64?)
        for (int k = 0; k < DK / 16; ++k) {
            const int cb = k >> 2, sub = k & 3;
            uint64_t a = umma_desc_sw128(smem_u32(cs + cb * KEYS * 128) + sub * 32, 16, 1024);
            uint64_t b = umma_desc_sw128(smem_u32(qs + cb * NH * 128) + sub * 32, 16, 1024);
            umma_ss(t0 + (16u << 16) + 64, a, b, id_qk, k > 0);
        }
        umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int w = tid >> 5, l = tid & 31;
    uint32_t r[32];
    tmem_ld32(t0 + ((uint32_t)(w * 32) << 16), r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) s_out[(w * 32 + l) * 16 + j] = __uint_as_float(r[j]);
    for (int j = 0; j < 16; ++j) o_out[(w * 32 + l) * 16 + j] = __uint_as_float(r[16 + j]);
    tmem_ld32(t0 + ((uint32_t)(w * 32) << 16) + 64, r);
    tmem_wait_ld();
    for (int j = 0; j < 16; ++j) s_out[128 * 16 + (w * 32 + l) * 16 + j] = __uint_as_float(r[j]);
    tc_fence_before();
    __syncthreads();
    if (tid < 32) tmem_dealloc(t0, 128);
}

static uint16_t f2bf(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return (uint16_t)((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf2f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

int main() {
    srand(1);
    auto rnd = [] { return (float)((rand() % 17) - 8) / 8.0f; };  // exact in bf16
    std::vector<float> C(KEYS * DK), Q(NH * DK), P(NH * KEYS);
    for (auto& x : C) x = rnd();
    for (auto& x : Q) x = rnd();
    for (auto& x : P) x = rnd();
    std::vector<uint16_t> cimg(NCB * KEYS * 64), qimg(NCB * NH * 64), pimg(NH * 64);
    for (int r = 0; r < KEYS; ++r)
        for (int c = 0; c < DK; ++c) cimg[(c / 64) * KEYS * 64 + swz(r, c % 64) / 2] = f2bf(C[r * DK + c]);
    for (int h = 0; h < NH; ++h)
        for (int c = 0; c < DK; ++c) qimg[(c / 64) * NH * 64 + swz(h, c % 64) / 2] = f2bf(Q[h * DK + c]);
    for (int h = 0; h < NH; ++h)
        for (int k = 0; k < KEYS; ++k) pimg[swz(h, k) / 2] = f2bf(P[h * KEYS + k]);
    uint16_t *dc, *dq, *dp;
    float *ds, *dout;
    cudaMalloc(&dc, cimg.size() * 2);
    cudaMalloc(&dq, qimg.size() * 2);
    cudaMalloc(&dp, pimg.size() * 2);
    cudaMalloc(&ds, 2 * 128 * 16 * 4);
    cudaMalloc(&dout, 128 * 16 * 4);
    cudaMemcpy(dc, cimg.data(), cimg.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, qimg.data(), qimg.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dp, pimg.data(), pimg.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(ds, 0xFF, 2 * 128 * 16 * 4);
    const int smem = 1024 + NCB * KEYS * 128 + NCB * NH * 128 + NH * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int variant = 0; variant < 2; ++variant) {
    uint32_t lbo = variant == 0 ? KEYS * 128 : 1024, sbo = variant == 0 ? 1024 : KEYS * 128;
    cudaMemset(dout, 0, 128 * 16 * 4);
    probe<<<1, 128, smem>>>(dc, dq, dp, ds, dout, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant lbo=%u sbo=%u kernel: %s\n", lbo, sbo, cudaGetErrorString(e));
    std::vector<float> s(2 * 128 * 16), o(128 * 16);
    cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
    std::vector<float> ref(KEYS * NH);
    for (int k = 0; k < KEYS; ++k)
        for (int h = 0; h < NH; ++h) {
            double a = 0;
            for (int c = 0; c < DK; ++c) a += (double)C[k * DK + c] * Q[h * DK + c];
            ref[k * NH + h] = (float)a;
        }
    if (variant == 0) for (int half = 0; half < 2; ++half) {
    printf("QK M=64 (D lane base %d) lane -> key map:\n", half * 16);
    for (int lane = 0; lane < 128; ++lane) {
        int match = -1;
        for (int k = 0; k < KEYS; ++k) {
            bool ok = true;
            for (int h = 0; h < NH; ++h) ok &= fabsf(s[half * 2048 + lane * 16 + h] - ref[k * NH + h]) < 1e-3f;
            if (ok) { match = k; break; }
        }
        printf("%d:%d ", lane, match);
        if (lane % 16 == 15) printf("\n");
    }
    }
    std::vector<double> oref(128 * NH);
    double maxerr = 0;
    for (int d = 0; d < 128; ++d)
        for (int h = 0; h < NH; ++h) {
            double a = 0;
            for (int k = 0; k < KEYS; ++k) a += (double)C[k * DK + d] * P[h * KEYS + k];
            oref[d * NH + h] = a;
            maxerr = fmax(maxerr, fabs(a - o[d * 16 + h]));
        }
    printf("PV M=128 MN-major A: max err %g\nlane -> dv map:\n", maxerr);
    for (int lane = 0; lane < 128; ++lane) {
        int match = -1;
        for (int d = 0; d < 128; ++d) {
            bool ok = true;
            for (int h = 0; h < NH; ++h) ok &= fabs(o[lane * 16 + h] - oref[d * NH + h]) < 1e-3;
            if (ok) { match = d; break; }
        }
        printf("%d:%d ", lane, match);
        if (lane % 16 == 15) printf("\n");
    }
    printf("lane0 got: "); for (int h = 0; h < 4; ++h) printf("%g ", o[h]); printf(" ref: ");
    for (int h = 0; h < 4; ++h) printf("%g ", oref[h]); printf("\n");
    }
    return 0;
}
