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

#include "common.cuh"
#include "internal.h"

namespace {

using spd::quant8;

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

// the rotation of one pair in fp32 (shared by rope_kernel and rope_write_kernel, so both
// produce bit-identical rows)
template <typename T>
__device__ __forceinline__ void rot_pair(T& e0, T& e1, float c, float s) {
    if constexpr (sizeof(T) == 2) {
        const float x0 = __bfloat162float(e0), x1 = __bfloat162float(e1);
        e0 = __float2bfloat16_rn(fmaf(x0, c, -x1 * s));
        e1 = __float2bfloat16_rn(fmaf(x1, c, x0 * s));
    } else {
        const float x0 = e0, x1 = e1;
        e0 = fmaf(x0, c, -x1 * s);
        e1 = fmaf(x1, c, x0 * s);
    }
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
    auto rot = [](T& e0, T& e1, float c, float s) { rot_pair<T>(e0, e1, c, s); };
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

// ---------------------------------------------------------------------------------------
// RoPE fused with the K/V write (semipd_set_rope; R28).  One CTA per new row t:
//   position  prefill: prefix[r] + (t - cu[r]) for the request r holding t (R4);
//             decode (cu == NULL): ctx[t] (R5)
//   q rows    rotated in place (the attention reads them next)
//   k rows    rotated in place (the prefill attention reads the chunk's keys from k_new) and
//             stored, with the unrotated columns, into the pool slot of that position
//   v rows    copied into the pool slot (absent for the MLA latent: V aliases K)
// The angles and the rotation are rope_kernel's (fp64 sincos, rot_pair), so a fused call and
// semipd_rope followed by an unfused call leave bit-identical rows and pool pages.
struct RopeWriteParams {
    unsigned char* q;
    unsigned char* k;
    const unsigned char* v;
    unsigned char* kpool;  // this layer's pages [N_B][Hkv][bs][dk]
    unsigned char* vpool;  // [N_B][Hkv][bs][dv] or null (kv_shared)
    const int* cu;         // prefill [n + 1]; null = decode
    const int* req_ids;
    const int* base;       // prefix_lens (prefill) / ctx_lens (decode)
    const int* bt;
    int* status;
    int n, Hq, Hkv, dk, dv, off, rd, lg_bs, MBR, N_B;
    float ks, vs;  // E4M3 pools (F8): the layer's scales of the quantised write (R31)
    int qdk, qoff;  // q row length and the first rotated q column (the pool's dk / off unless
                    // q is narrower, as the expanded MLA prefill's [q_nope | q_pe] rows)
    int write_pool; // 0: rotate q / k in place only (the caller's next pass writes the pool)
    double inv_freq[MAX_HALF];
};

// F8: E4M3 pages — the rotated k rows, the unrotated k columns and the v rows are written as
// codes with fp8.cu's rule (quant8), exactly the bytes its own quantised append / chunk write
// would store from the rotated k_new (so fused and composed paths leave identical pages)
template <typename T, bool INTER, bool F8>
__global__ void __launch_bounds__(256) rope_write_kernel(const __grid_constant__ RopeWriteParams p) {
    static_assert(!F8 || sizeof(T) == 2, "E4M3 pools take bf16 activations");
    constexpr int VEC = 16 / sizeof(T);
    extern __shared__ float cs[];  // [rd/2] cos, [rd/2] sin
    const int t = blockIdx.x;
    int r = t, pos;
    if (p.cu) {
        int hi = p.n - 1;  // the last request r with cu[r] <= t
        r = 0;
        while (r < hi) {
            const int mid = (r + hi + 1) >> 1;
            if (__ldg(p.cu + mid) <= t) r = mid; else hi = mid - 1;
        }
        pos = __ldg(p.base + r) + t - __ldg(p.cu + r);
    } else {
        pos = __ldg(p.base + t);
    }
    const int page = pos >> p.lg_bs;
    const int blk = p.write_pool && page < p.MBR ? __ldg(p.bt + (size_t)__ldg(p.req_ids + r) * p.MBR + page) : -1;
    const bool ok = blk >= 0 && blk < p.N_B;
    if (p.write_pool && !ok && threadIdx.x == 0 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
    const int half = p.rd >> 1;
    for (int i = threadIdx.x; i < half; i += blockDim.x) {
        double s, c;
        sincos((double)pos * p.inv_freq[i], &s, &c);
        cs[i] = (float)c;
        cs[half + i] = (float)s;
    }
    __syncthreads();
    const int nrot = (INTER ? p.rd : half) / VEC;  // rotation items per head row
    const int nkp = p.write_pool ? (p.dk - p.rd) / VEC : 0;  // unrotated k vectors per head row
    const int nv = p.write_pool && p.vpool ? p.dv / VEC : 0;
    const int n_q = p.Hq * nrot, n_kr = p.Hkv * nrot, n_kp = p.Hkv * nkp, n_v = p.Hkv * nv;
    const int total = n_q + n_kr + n_kp + n_v;
    const size_t bs_mask = ((size_t)1 << p.lg_bs) - 1;
    auto slot = [&](int h) { return (((size_t)blk * p.Hkv + h) << p.lg_bs) + ((size_t)pos & bs_mask); };
    for (int it = threadIdx.x; it < total; it += blockDim.x) {
        if (it < n_q + n_kr) {
            const bool is_q = it < n_q;
            const int j = is_q ? it : it - n_q;
            const int h = j / nrot, i0 = (j % nrot) * VEC;
            T* row = is_q ? reinterpret_cast<T*>(p.q) + ((size_t)t * p.Hq + h) * p.qdk + p.qoff
                          : reinterpret_cast<T*>(p.k) + ((size_t)t * p.Hkv + h) * p.dk + p.off;
            uint4 a = *reinterpret_cast<const uint4*>(row + i0);
            T* xa = reinterpret_cast<T*>(&a);
            uint4 b = a;
            if constexpr (INTER) {
#pragma unroll
                for (int e = 0; e < VEC / 2; ++e) {
                    const int fi = (i0 >> 1) + e;
                    rot_pair<T>(xa[2 * e], xa[2 * e + 1], cs[fi], cs[half + fi]);
                }
            } else {
                b = *reinterpret_cast<const uint4*>(row + half + i0);
                T* xb = reinterpret_cast<T*>(&b);
#pragma unroll
                for (int e = 0; e < VEC; ++e) rot_pair<T>(xa[e], xb[e], cs[i0 + e], cs[half + i0 + e]);
            }
            *reinterpret_cast<uint4*>(row + i0) = a;
            if (!INTER) *reinterpret_cast<uint4*>(row + half + i0) = b;
            if (!is_q && ok) {
                if constexpr (F8) {
                    unsigned char* dst = p.kpool + slot(h) * p.dk + p.off;
                    *reinterpret_cast<uint2*>(dst + i0) = quant8(a, p.ks);
                    if (!INTER) *reinterpret_cast<uint2*>(dst + half + i0) = quant8(b, p.ks);
                } else {
                    T* dst = reinterpret_cast<T*>(p.kpool) + slot(h) * p.dk + p.off;
                    *reinterpret_cast<uint4*>(dst + i0) = a;
                    if (!INTER) *reinterpret_cast<uint4*>(dst + half + i0) = b;
                }
            }
        } else if (it < n_q + n_kr + n_kp) {
            if (!ok) continue;
            const int j = it - n_q - n_kr;
            const int h = j / nkp, c0 = (j % nkp) * VEC;
            const int c = c0 < p.off ? c0 : c0 + p.rd;  // columns outside [off, off + rd)
            const T* src = reinterpret_cast<const T*>(p.k) + ((size_t)t * p.Hkv + h) * p.dk + c;
            if constexpr (F8)
                *reinterpret_cast<uint2*>(p.kpool + slot(h) * p.dk + c) =
                    quant8(*reinterpret_cast<const uint4*>(src), p.ks);
            else
                *reinterpret_cast<uint4*>(reinterpret_cast<T*>(p.kpool) + slot(h) * p.dk + c) =
                    *reinterpret_cast<const uint4*>(src);
        } else {
            if (!ok) continue;
            const int j = it - n_q - n_kr - n_kp;
            const int h = j / nv, c = (j % nv) * VEC;
            const T* src = reinterpret_cast<const T*>(p.v) + ((size_t)t * p.Hkv + h) * p.dv + c;
            if constexpr (F8)
                *reinterpret_cast<uint2*>(p.vpool + slot(h) * p.dv + c) =
                    quant8(__ldg(reinterpret_cast<const uint4*>(src)), p.vs);
            else
                *reinterpret_cast<uint4*>(reinterpret_cast<T*>(p.vpool) + slot(h) * p.dv + c) =
                    __ldg(reinterpret_cast<const uint4*>(src));
        }
    }
}

// the semipd_rope argument checks (shared with semipd_set_rope)
semipd_status rope_check(int head_dim, int rot_offset, int rot_dim, int dtype, double theta,
                         double factor, double lf, double hf, int L0) {
    if (head_dim <= 0 || rot_offset < 0 || rot_dim <= 0 || rot_dim % 2 ||
        rot_offset + rot_dim > head_dim || !(theta > 1.0) ||
        (dtype != SEMIPD_BF16 && dtype != SEMIPD_FP32))
        return SEMIPD_ERR_INVALID;
    if (factor > 1.0 && (!(hf > lf) || !(lf > 0.0) || L0 <= 0)) return SEMIPD_ERR_INVALID;
    return SEMIPD_OK;
}

}  // namespace

semipd_status spd_launch_rope_write(semipd_pool_t pool, int layer, void* q, void* k_new,
                                    const void* v_new, const int* cu_seqlens, const int* req_ids,
                                    const int* base_pos, int n, int T, int Hq, int* status_dev,
                                    cudaStream_t st) {
    return spd_launch_rope_write_ex(pool, layer, q, pool->cfg.head_dim_k, pool->rope.rot_offset,
                                    k_new, v_new, cu_seqlens, req_ids, base_pos, n, T, Hq, 1,
                                    status_dev, st);
}

semipd_status spd_launch_rope_write_ex(semipd_pool_t pool, int layer, void* q, int q_dk, int q_off,
                                       void* k_new, const void* v_new, const int* cu_seqlens,
                                       const int* req_ids, const int* base_pos, int n, int T, int Hq,
                                       int write_pool, int* status_dev, cudaStream_t st) {
    const auto& c = pool->cfg;
    const auto& rc = pool->rope;
    if (T <= 0) return SEMIPD_OK;
    const uintptr_t mis = reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k_new) |
                          reinterpret_cast<uintptr_t>(v_new);
    if (mis % 16) return SEMIPD_ERR_UNSUPPORTED;
    RopeWriteParams p;
    p.q = static_cast<unsigned char*>(q);
    p.k = static_cast<unsigned char*>(k_new);
    p.v = static_cast<const unsigned char*>(v_new);
    p.kpool = static_cast<unsigned char*>(pool->k_layer(layer));
    p.vpool = c.kv_shared ? nullptr : static_cast<unsigned char*>(pool->v_layer(layer));
    p.cu = cu_seqlens;
    p.req_ids = req_ids;
    p.base = base_pos;
    p.bt = pool->bt;
    p.status = status_dev;
    p.n = n;
    p.Hq = Hq;
    p.Hkv = c.num_kv_heads;
    p.dk = c.head_dim_k;
    p.dv = c.head_dim_v;
    p.off = rc.rot_offset;
    p.rd = rc.rot_dim;
    p.qdk = q_dk;
    p.qoff = q_off;
    p.write_pool = write_pool;
    p.lg_bs = __builtin_ctz((unsigned)c.block_size);
    p.MBR = c.max_blocks_per_req;
    p.N_B = c.num_blocks;
    for (int i = 0; i < MAX_HALF; ++i) p.inv_freq[i] = pool->rope_inv_freq[i];
    const bool f8 = c.dtype == SEMIPD_FP8_E4M3;
    p.ks = f8 ? pool->k_scale[layer] : 1.f;
    p.vs = f8 ? pool->v_scale[layer] : 1.f;
    const size_t smem = (size_t)rc.rot_dim * sizeof(float);
    if (f8)
        rc.interleaved ? rope_write_kernel<__nv_bfloat16, true, true><<<T, 256, smem, st>>>(p)
                       : rope_write_kernel<__nv_bfloat16, false, true><<<T, 256, smem, st>>>(p);
    else if (c.dtype == SEMIPD_BF16)
        rc.interleaved ? rope_write_kernel<__nv_bfloat16, true, false><<<T, 256, smem, st>>>(p)
                       : rope_write_kernel<__nv_bfloat16, false, false><<<T, 256, smem, st>>>(p);
    else
        rc.interleaved ? rope_write_kernel<float, true, false><<<T, 256, smem, st>>>(p)
                       : rope_write_kernel<float, false, false><<<T, 256, smem, st>>>(p);
    pool->launches += 1;
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

extern "C" semipd_status semipd_set_rope(semipd_pool_t pool, const semipd_rope_config* cfg) {
    if (!pool) return SEMIPD_ERR_INVALID;
    if (!cfg) {
        pool->rope_on = false;
        return SEMIPD_OK;
    }
    const auto& c = pool->cfg;
    // E4M3 pools carry bf16 activations (q / k_new); the fused write quantises (R31)
    const int act = c.dtype == SEMIPD_FP8_E4M3 ? SEMIPD_BF16 : c.dtype;
    const semipd_status e = rope_check(c.head_dim_k, cfg->rot_offset, cfg->rot_dim, act,
                                       cfg->theta, cfg->factor, cfg->low_freq_factor,
                                       cfg->high_freq_factor, cfg->original_max_pos);
    if (e != SEMIPD_OK) return e;
    const int vec = act == SEMIPD_BF16 ? 8 : 4;
    const int half = cfg->rot_dim / 2;
    if ((cfg->interleaved ? cfg->rot_dim : half) % vec || cfg->rot_offset % vec ||
        c.head_dim_k % vec || c.head_dim_v % vec || half > MAX_HALF)
        return SEMIPD_ERR_UNSUPPORTED;
    pool->rope = *cfg;
    for (int i = 0; i < MAX_HALF; ++i)
        pool->rope_inv_freq[i] = i < half ? rope_inv_freq(i, cfg->rot_dim, cfg->theta, cfg->factor,
                                                           cfg->low_freq_factor, cfg->high_freq_factor,
                                                           (double)cfg->original_max_pos)
                                          : 0.0;
    pool->rope_on = true;
    return SEMIPD_OK;
}

extern "C" semipd_status semipd_rope(void* q, void* k, const int32_t* positions,
                                     int32_t num_tokens, int32_t num_q_heads, int32_t num_kv_heads,
                                     int32_t head_dim, int32_t rot_offset, int32_t rot_dim,
                                     int32_t interleaved, int32_t dtype, double theta, double factor,
                                     double low_freq_factor, double high_freq_factor,
                                     int32_t original_max_pos, semipd_stream_t s) {
    if (num_tokens < 0 || num_q_heads < 0 || num_kv_heads < 0) return SEMIPD_ERR_INVALID;
    const semipd_status e = rope_check(head_dim, rot_offset, rot_dim, dtype, theta, factor,
                                       low_freq_factor, high_freq_factor, original_max_pos);
    if (e != SEMIPD_OK) return e;
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
