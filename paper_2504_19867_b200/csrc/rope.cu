// rope.cu — rotary position embedding of q and k in place (§6:
// "To support the Llama3.1 series model, we also modify the RoPE kernel").  It is applied to
// the step's new q / k rows before the attention call that writes k into the pool (a3 / a5),
// so the pool holds rotated keys, as in Llama.
//
// Definition (reading R27) over the rotated columns [off, off + rd) of each row (the
// whole head for Llama; the 64 decoupled-rope columns of a 576-d MLA row): half-split pairs
// (i, i + rd/2), i < rd/2 (Llama), or interleaved pairs (2i, 2i + 1) (GPT-J / DeepSeek layout),
//   f_i   = theta^(-2i/rd), rescaled by the Llama-3.1 rule when factor > 1:
//           wavelength w_i = 2 pi / f_i; w_i < L0/hf: f_i;  w_i > L0/lf: f_i / factor;
//           else (1 - a) f_i / factor + a f_i with a = (L0 / w_i - lf) / (hf - lf)
//   phi   = pos * f_i
//   x'_i        = x_i cos phi - x_{i+d/2} sin phi
//   x'_{i+d/2}  = x_{i+d/2} cos phi + x_i sin phi
// HBM-bound elementwise pass: one CTA per token; the token's d/2 (cos, sin) pairs are formed
// once in fp64 (the angle reaches 1e5 rad at 128k positions, where fp32 would lose ~1e-2 rad)
// from the host's f_i table while the CTA's first loads are in flight, and shared by all of
// its q and k heads;
// every thread rotates one 16-byte vector of x_i and
// the matching vector of x_{i+d/2} (coalesced 128-bit loads and stores).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"

namespace {

constexpr int MAX_HALF = 128;  // head_dim <= 256 (Llama 128, MLA rope part 64)

struct RopeParams {
    unsigned char* q;
    unsigned char* k;
    const int* pos;
    int Hq, Hkv, d, off, rd;  // row length, rotated columns [off, off + rd)
    double inv_freq[MAX_HALF];  // f_i in fp64, formed once per call on the host
};

// f_i with the Llama-3.1 rescaling (host).  Measured alternatives: fp64 pow or exp2 per CTA
// on the device cost 20-25 % of the large-T bandwidth (3.8-4.0 vs 5.1 TB/s)
double rope_inv_freq(int i, int d, double theta, double factor, double lf, double hf, double L0) {
    const double f = std::pow(theta, -2.0 * i / d);
    if (!(factor > 1.0)) return f;
    const double w = 2.0 * 3.14159265358979323846 / f;
    if (w < L0 / hf) return f;
    if (w > L0 / lf) return f / factor;
    const double a = (L0 / w - lf) / (hf - lf);
    return (1.0 - a) * f / factor + a * f;
}

template <typename T, bool INTER>
__global__ void __launch_bounds__(512) rope_kernel(const __grid_constant__ RopeParams p) {
    constexpr int VEC = 16 / sizeof(T);  // elements per 16-byte vector
    extern __shared__ float cs[];         // [rd/2] cos, [rd/2] sin
    const int t = blockIdx.x;
    const int half = p.rd >> 1;
    // half-split: a vector of x_i and the matching vector of x_{i+rd/2};
    // interleaved: one vector of VEC/2 adjacent pairs (x_2i, x_2i+1)
    const int vph = (INTER ? p.rd : half) / VEC;  // vectors per head
    const int nvec = (p.Hq + p.Hkv) * vph;
    auto row_of = [&](int v, int& i0) {
        const int h = v / vph;
        i0 = (v % vph) * VEC;
        T* row = h < p.Hq ? reinterpret_cast<T*>(p.q) + ((size_t)t * p.Hq + h) * p.d
                          : reinterpret_cast<T*>(p.k) + ((size_t)t * p.Hkv + (h - p.Hq)) * p.d;
        return row + p.off;
    };
    // this thread's first vectors are loaded before the angles are formed, so the HBM
    // latency overlaps the fp64 sincos
    const int v0 = threadIdx.x;
    T* row0 = nullptr;
    uint4 a0 = make_uint4(0, 0, 0, 0), b0 = a0;
    int i00 = 0;
    if (v0 < nvec) {
        row0 = row_of(v0, i00);
        a0 = __ldcs(reinterpret_cast<const uint4*>(row0 + i00));
        if (!INTER) b0 = __ldcs(reinterpret_cast<const uint4*>(row0 + half + i00));
    }
    const double pos = (double)__ldg(p.pos + t);
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
        double s, c;
        sincos(pos * p.inv_freq[i], &s, &c);
        cs[i] = (float)c;
        cs[half + i] = (float)s;
    }
    __syncthreads();
    auto rot = [](T& e0, T& e1, float c, float s) {
        if constexpr (sizeof(T) == 2) {
            const float x0 = __bfloat162float(e0), x1 = __bfloat162float(e1);
            e0 = __float2bfloat16_rn(fmaf(x0, c, -x1 * s));
            e1 = __float2bfloat16_rn(fmaf(x1, c, x0 * s));
        } else {
            const float x0 = e0, x1 = e1;
            e0 = fmaf(x0, c, -x1 * s);
            e1 = fmaf(x1, c, x0 * s);
        }
    };
    for (int v = v0; v < nvec; v += blockDim.x) {
        T* row;
        int i0;
        uint4 a, b;
        if (v == v0) {
            row = row0, i0 = i00, a = a0, b = b0;
        } else {
            row = row_of(v, i0);
            a = __ldcs(reinterpret_cast<const uint4*>(row + i0));
            if (!INTER) b = __ldcs(reinterpret_cast<const uint4*>(row + half + i0));
        }
        T* xa = reinterpret_cast<T*>(&a);
        if constexpr (INTER) {
#pragma unroll
            for (int j = 0; j < VEC / 2; ++j) {
                const int fi = (i0 >> 1) + j;
                rot(xa[2 * j], xa[2 * j + 1], cs[fi], cs[half + fi]);
            }
            __stcs(reinterpret_cast<uint4*>(row + i0), a);
        } else {
            T* xb = reinterpret_cast<T*>(&b);
#pragma unroll
            for (int j = 0; j < VEC; ++j) rot(xa[j], xb[j], cs[i0 + j], cs[half + i0 + j]);
            __stcs(reinterpret_cast<uint4*>(row + i0), a);
            __stcs(reinterpret_cast<uint4*>(row + half + i0), b);
        }
    }
}

}  // namespace

extern "C" semipd_status semipd_rope(void* q, void* k, const int32_t* positions,
                                     int32_t num_tokens, int32_t num_q_heads, int32_t num_kv_heads,
                                     int32_t head_dim, int32_t rot_offset, int32_t rot_dim,
                                     int32_t interleaved, int32_t dtype, double theta, double factor,
                                     double low_freq_factor, double high_freq_factor,
                                     int32_t original_max_pos, semipd_stream_t s) {
    if (num_tokens < 0 || num_q_heads < 0 || num_kv_heads < 0 || head_dim <= 0 || rot_offset < 0 ||
        rot_dim <= 0 || rot_dim % 2 || rot_offset + rot_dim > head_dim || !(theta > 1.0) ||
        (dtype != SEMIPD_BF16 && dtype != SEMIPD_FP32))
        return SEMIPD_ERR_INVALID;
    if (factor > 1.0 && (!(high_freq_factor > low_freq_factor) || !(low_freq_factor > 0.0) ||
                         original_max_pos <= 0))
        return SEMIPD_ERR_INVALID;
    if (num_tokens == 0 || num_q_heads + num_kv_heads == 0) return SEMIPD_OK;
    if ((num_q_heads > 0 && !q) || (num_kv_heads > 0 && !k) || !positions) return SEMIPD_ERR_INVALID;
    const int vec = dtype == SEMIPD_BF16 ? 8 : 4;
    const int half = rot_dim / 2;
    if ((interleaved ? rot_dim : half) % vec || rot_offset % vec || head_dim % vec || half > MAX_HALF)
        return SEMIPD_ERR_UNSUPPORTED;
    if ((q && reinterpret_cast<uintptr_t>(q) % 16) || (k && reinterpret_cast<uintptr_t>(k) % 16))
        return SEMIPD_ERR_UNSUPPORTED;
    RopeParams p;
    p.q = static_cast<unsigned char*>(q);
    p.k = static_cast<unsigned char*>(k);
    p.pos = positions;
    p.Hq = num_q_heads;
    p.Hkv = num_kv_heads;
    p.d = head_dim;
    p.off = rot_offset;
    p.rd = rot_dim;
    for (int i = 0; i < half; ++i)
        p.inv_freq[i] = rope_inv_freq(i, rot_dim, theta, factor, low_freq_factor, high_freq_factor,
                                      (double)original_max_pos);
    const int nvec = (num_q_heads + num_kv_heads) * ((interleaved ? rot_dim : half) / vec);
    int threads = ((nvec + 31) / 32) * 32;
    if (threads > 512) threads = 512;
    if (threads < 64) threads = 64;
    const size_t smem = (size_t)rot_dim * sizeof(float);
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (dtype == SEMIPD_BF16)
        interleaved ? rope_kernel<__nv_bfloat16, true><<<num_tokens, threads, smem, st>>>(p)
                    : rope_kernel<__nv_bfloat16, false><<<num_tokens, threads, smem, st>>>(p);
    else
        interleaved ? rope_kernel<float, true><<<num_tokens, threads, smem, st>>>(p)
                    : rope_kernel<float, false><<<num_tokens, threads, smem, st>>>(p);
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
