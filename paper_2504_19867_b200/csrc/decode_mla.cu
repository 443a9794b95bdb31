// decode_mla.cu — absorbed-MLA decode attention over the unified paged latent pool
// (cfg 5, DeepSeek-V2-Lite style: 16 q heads share ONE latent KV head, dk = 576 (512
// latent + 64 rope), dv = 512, V = K[..., :512]; R19).  Same hot-path contract
// as decode.cu (P:184 fused append, P:229 paged access, split-K merge in split order),
// tensor cores via mma.sync: AI ~ 30 FLOP/B, so the math must stay below HBM time.
//
// Per CTA: warp 4 = producer (unit fetch, K append of the latent row, one 4-D TMA box of
// 32 keys x 576 columns = 36 KiB per stage, 5-deep ring); warps 0-3 = consumers, and
// EVERY consumer warp reads EVERY stage:
//   QK^T  warp w contracts dims [144 w, 144 w + 144) for all 16 heads x 32 keys (Q slice
//         in registers), partial scores summed through shared memory;
//   softmax  warp w owns heads 4w..4w+3 (lane = key): running max / sum, P (bf16) -> smem;
//   PV    warp w owns output columns [128 w, 128 w + 128) for all 16 heads.
// The decomposition depends on shapes only (bitwise identical for every sm_budget).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int DK = 576, DV = 512, NH = 16;
constexpr int KPS = 32;                      // keys per stage
constexpr int NSTAGE = 5;
constexpr int NCW = 4;
constexpr int NTHREADS = (NCW + 1) * 32;
constexpr int NBLK = DK / 64;                // 9 column blocks of 128 B
constexpr int STAGE_BYTES = NBLK * KPS * 128;  // 36 KiB
constexpr int KSTEPS_W = DK / 16 / NCW;      // 9 k-steps of the QK contraction per warp
constexpr int DVW = DV / NCW;                // 128 output columns per warp
constexpr int PROW = 80;                     // padded P row (bytes): conflict-free ldmatrix
constexpr int SPLIT_KEYS = 2048;  // MLA: 2.4 MB of latent per split
constexpr int SROW = 40;          // padded score row (floats): conflict-free fragment stores
constexpr float LOG2E = 1.4426950408889634f;

struct MUnit {
    int b, s, S, k0, k1, nst;  // b < 0: done
};

struct MlaParams {
    const __nv_bfloat16* q;   // [B][16][576]
    const uint4* k_new;       // [B][1][576]
    const int* req_ids;
    const int* ctx_lens;
    const int* bt;
    unsigned char* k_pool;
    __nv_bfloat16* out;       // [B][16][512] or [16][B][512]
    float* ws_m;              // [B][16][S_max]
    float* ws_l;
    float* ws_acc;            // [B][16][S_max][512]
    int* ws_cnt;              // [B]
    unsigned* sched;
    int* status;
    unsigned long long* span;  // semipd_set_spans record of this launch (or null)
    int skip_append;           // 1: the step's latent row is already in the pool (RoPE pre-pass)
    int B, lg_bs, MBR, N_B, S_max, n_units, out_head_major, G;
    float scale_log2;
    SpdTrace trace;
};

__device__ __forceinline__ void split_range(int ctx, int S, int s, int& k0, int& k1) {
    const int nk = ctx + 1;
    int len = (nk + S - 1) / S;
    len = (len + KPS - 1) / KPS * KPS;
    k0 = s * len;
    k1 = min(nk, k0 + len);
}

// byte offset of 16-byte chunk ci (0..71) of key row k inside a stage ([block][32 rows][128 B])
__device__ __forceinline__ uint32_t kchunk(int k, int ci) {
    return (uint32_t)((ci >> 3) * (KPS * 128) + k * 128 + (((ci & 7) ^ (k & 7)) << 4));
}

__global__ void __launch_bounds__(NTHREADS, 1)
    decode_mla_kernel(const __grid_constant__ CUtensorMap kmap, MlaParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* ring = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    float* scr_s = reinterpret_cast<float*>(ring + NSTAGE * STAGE_BYTES);  // [4][16][SROW]
    unsigned char* pbuf = reinterpret_cast<unsigned char*>(scr_s + NCW * NH * SROW);  // [16][80 B]
    float* alpha_s = reinterpret_cast<float*>(pbuf + NH * PROW);  // [16]
    float* m_s = alpha_s + NH;   // [16]
    float* l_s = m_s + NH;       // [16]
    uint64_t* full = reinterpret_cast<uint64_t*>(l_s + NH);
    uint64_t* empty = full + NSTAGE;
    uint64_t* ufull = empty + NSTAGE;
    uint64_t* uempty = ufull + 2;
    MUnit* units = reinterpret_cast<MUnit*>(uempty + 2);
    int* s_last = reinterpret_cast<int*>(units + 2);

    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, NCW);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(ufull + i, 1);
            mbar_init(uempty + i, NCW);
        }
        fence_mbar_init();
        span_begin(p.span);
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(2, (int)smid(), (int)blockIdx.x, 3 /* kernel kind: MLA decode */);
        }
    }
    __syncthreads();

    if (warp == NCW) {
        // =========================== producer ===========================
        if (lane == 0) tma_prefetch_desc(&kmap);
        const int oob_z = p.N_B;
        const int bs_mask = (1 << p.lg_bs) - 1;
        int gstage = 0, nunit = 0;
        for (;;) {
            int u = 0;
            if (lane == 0) u = (int)atomicAdd(p.sched, 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
            MUnit d;
            if (u >= p.n_units) {
                d.b = -1;
            } else {
                d.s = u / p.B;
                d.b = u % p.B;
                const int ctx = __ldg(p.ctx_lens + d.b);
                d.S = (ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
                if (d.s >= d.S) continue;
                split_range(ctx, d.S, d.s, d.k0, d.k1);
                d.nst = (d.k1 - d.k0 + KPS - 1) / KPS;
            }
            const int us = nunit & 1;
            if (lane == 0) {
                mbar_wait(uempty + us, ((nunit >> 1) & 1) ^ 1);
                units[us] = d;
                mbar_arrive(ufull + us);
            }
            __syncwarp();
            ++nunit;
            if (d.b < 0) break;
            const int ctx = __ldg(p.ctx_lens + d.b);
            const int* btr = p.bt + (size_t)__ldg(p.req_ids + d.b) * p.MBR;
            const int last_page = ctx >> p.lg_bs;
            if (d.s == d.S - 1 && !p.skip_append) {
                // fused append of the step's latent row (576 bf16 = 72 x 16 B) at slot ctx
                const int blk = last_page < p.MBR ? __ldg(btr + last_page) : -1;
                if (blk >= 0 && blk < p.N_B) {
                    const size_t slot = ((size_t)blk << p.lg_bs) + (ctx & bs_mask);
                    for (int c = lane; c < DK / 8; c += 32)
                        reinterpret_cast<uint4*>(p.k_pool)[slot * (DK / 8) + c] =
                            __ldg(p.k_new + (size_t)d.b * (DK / 8) + c);
                    fence_proxy_async_global();
                }
                __syncwarp();
            }
            for (int i = 0; i < d.nst; ++i, ++gstage) {
                if (lane == 0) {
                    const int st = gstage % NSTAGE;
                    mbar_wait(empty + st, ((gstage / NSTAGE) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + st, STAGE_BYTES);
                    const int key = d.k0 + i * KPS;
                    const int page = key >> p.lg_bs;
                    int z = oob_z;
                    if (page <= last_page) {
                        const int blk = page < p.MBR ? __ldg(btr + page) : -1;
                        if (blk >= 0 && blk < p.N_B) z = blk;
                        else if (p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                    }
                    tma_load_4d(ring + st * STAGE_BYTES, &kmap, full + st, 0, key & bs_mask, 0, z);
                }
                __syncwarp();
            }
        }
    } else {
        // =========================== consumers ===========================
        const int r0 = lane >> 2, c0 = (lane & 3) * 2;
        const int tid = threadIdx.x;  // 0..127
        int gstage = 0, nunit = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(ufull + us, (nunit >> 1) & 1);
            const MUnit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(uempty + us);
            ++nunit;
            if (d.b < 0) break;
            // Q fragments of this warp's contraction slice (heads >= G are zero rows)
            uint32_t qa[KSTEPS_W][4];
            {
                const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q) + (size_t)d.b * NH * (DK / 2);
                const bool va = r0 < p.G, vb = r0 + 8 < p.G;
#pragma unroll
                for (int kk = 0; kk < KSTEPS_W; ++kk) {
                    const int col = ((warp * KSTEPS_W + kk) * 16 + c0) >> 1;
                    qa[kk][0] = va ? __ldg(q32 + r0 * (DK / 2) + col) : 0u;
                    qa[kk][1] = vb ? __ldg(q32 + (r0 + 8) * (DK / 2) + col) : 0u;
                    qa[kk][2] = va ? __ldg(q32 + r0 * (DK / 2) + col + 4) : 0u;
                    qa[kk][3] = vb ? __ldg(q32 + (r0 + 8) * (DK / 2) + col + 4) : 0u;
                }
            }
            float acc[DVW / 8][4];
#pragma unroll
            for (int i = 0; i < DVW / 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
            float mrun[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};  // heads 4w + i
            float lrun[4] = {0.f, 0.f, 0.f, 0.f};
            for (int i = 0; i < d.nst; ++i, ++gstage) {
                const int st = gstage % NSTAGE;
                mbar_wait(full + st, (gstage / NSTAGE) & 1);
                const uint32_t stg = smem_u32(ring + st * STAGE_BYTES);
                // ---- partial S over this warp's 144 dims: 4 n-tiles of 8 keys
                float s[4][4];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
                    const int key = nt * 8 + (lane & 7);
#pragma unroll
                    for (int kk = 0; kk < KSTEPS_W - 1; kk += 2) {
                        const int ci = 2 * (warp * KSTEPS_W + kk) + (lane >> 3);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(stg + kchunk(key, ci), b0, b1, b2, b3);
                        mma_bf16_16816(s[nt], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                        mma_bf16_16816(s[nt], qa[kk + 1][0], qa[kk + 1][1], qa[kk + 1][2],
                                       qa[kk + 1][3], b2, b3);
                    }
                    {   // odd last k-step: x4 over the same two chunks twice (only b0, b1 used)
                        const int kk = KSTEPS_W - 1;
                        const int ci = 2 * (warp * KSTEPS_W + kk) + ((lane >> 3) & 1);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(stg + kchunk(key, ci), b0, b1, b2, b3);
                        mma_bf16_16816(s[nt], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                    }
                    float* sw = scr_s + warp * NH * SROW;
                    *reinterpret_cast<float2*>(sw + r0 * SROW + nt * 8 + c0) = make_float2(s[nt][0], s[nt][1]);
                    *reinterpret_cast<float2*>(sw + (r0 + 8) * SROW + nt * 8 + c0) = make_float2(s[nt][2], s[nt][3]);
                }
                named_bar_sync(1, NCW * 32);
                // ---- softmax: warp w owns heads 4w..4w+3, lane = key
                const int key = d.k0 + i * KPS + lane;
                const bool live = key < d.k1;
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    const int h = warp * 4 + hh;
                    float x = scr_s[h * SROW + lane] + scr_s[NH * SROW + h * SROW + lane] +
                              scr_s[2 * NH * SROW + h * SROW + lane] + scr_s[3 * NH * SROW + h * SROW + lane];
                    x = live ? x * p.scale_log2 : -INFINITY;
                    float mx = x;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                    const float mnew = fmaxf(mrun[hh], mx);
                    const float alpha = fast_exp2(mrun[hh] - mnew);
                    const float pv = fast_exp2(x - mnew);
                    float ps = pv;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
                    lrun[hh] = lrun[hh] * alpha + ps;
                    mrun[hh] = mnew;
                    reinterpret_cast<__nv_bfloat16*>(pbuf + h * PROW)[lane] = __float2bfloat16_rn(pv);
                    if (lane == 0) alpha_s[h] = alpha;
                }
                named_bar_sync(1, NCW * 32);
                // ---- O[:, 128w..] = O * alpha + P V
                const float al0 = alpha_s[r0], al1 = alpha_s[r0 + 8];
                if (__any_sync(0xffffffffu, al0 != 1.f || al1 != 1.f)) {
#pragma unroll
                    for (int nd = 0; nd < DVW / 8; ++nd) {
                        acc[nd][0] *= al0;
                        acc[nd][1] *= al0;
                        acc[nd][2] *= al1;
                        acc[nd][3] *= al1;
                    }
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    uint32_t a0, a1, a2, a3;
                    ldsm_x4(smem_u32(pbuf) + (lane & 15) * PROW + (2 * ks + (lane >> 4)) * 16, a0, a1,
                            a2, a3);
                    const int vkey = ks * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
                    for (int nd = 0; nd < DVW / 8; nd += 2) {
                        const int ch = warp * (DVW / 8) + nd + (lane >> 4);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4_t(stg + kchunk(vkey, ch), b0, b1, b2, b3);
                        mma_bf16_16816(acc[nd], a0, a1, a2, a3, b0, b1);
                        mma_bf16_16816(acc[nd + 1], a0, a1, a2, a3, b2, b3);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
                // P / alpha / scores are rewritten next stage: all warps must be past PV
                named_bar_sync(1, NCW * 32);
            }
            // ---- unit epilogue: publish per-head (m, l) of the owning warps
            if (lane == 0) {
#pragma unroll
                for (int hh = 0; hh < 4; ++hh) {
                    m_s[warp * 4 + hh] = mrun[hh];
                    l_s[warp * 4 + hh] = lrun[hh];
                }
            }
            named_bar_sync(1, NCW * 32);
            const bool split = d.S > 1;
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                const int h = r0 + half * 8;
                if (h >= p.G) continue;
                const float inv = 1.f / l_s[h];
#pragma unroll
                for (int nd = 0; nd < DVW / 8; ++nd) {
                    const int col = warp * DVW + nd * 8 + c0;
                    const float v0 = acc[nd][half * 2], v1 = acc[nd][half * 2 + 1];
                    if (!split) {
                        const size_t off = p.out_head_major ? (((size_t)h * p.B + d.b) * DV + col)
                                                            : (((size_t)d.b * p.G + h) * DV + col);
                        *reinterpret_cast<uint32_t*>(p.out + off) = pack_bf16(v0 * inv, v1 * inv);
                    } else {
                        const size_t pi = ((size_t)d.b * NH + h) * p.S_max + d.s;
                        *reinterpret_cast<float2*>(p.ws_acc + pi * DV + col) = make_float2(v0, v1);
                        if (warp == 0 && nd == 0 && c0 == 0) {
                            p.ws_m[pi] = m_s[h];
                            p.ws_l[pi] = l_s[h];
                        }
                    }
                }
            }
            if (split) {
                __threadfence();
                named_bar_sync(1, NCW * 32);
                if (tid == 0) *s_last = atomicAdd(p.ws_cnt + d.b, 1) == d.S - 1;
                named_bar_sync(1, NCW * 32);
                if (*s_last) {
                    __threadfence();
                    for (int idx = tid; idx < p.G * (DV / 4); idx += NCW * 32) {
                        const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
                        const size_t pb = ((size_t)d.b * NH + h) * p.S_max;
                        float M = -INFINITY;
                        for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb + sI));
                        float L = 0.f;
                        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int sI = 0; sI < d.S; ++sI) {
                            const float f = fast_exp2(__ldcg(p.ws_m + pb + sI) - M);
                            L += f * __ldcg(p.ws_l + pb + sI);
                            const float4 a = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + (pb + sI) * DV + c));
                            o.x += f * a.x;
                            o.y += f * a.y;
                            o.z += f * a.z;
                            o.w += f * a.w;
                        }
                        const float inv = 1.f / L;
                        const size_t off = p.out_head_major ? (((size_t)h * p.B + d.b) * DV + c)
                                                            : (((size_t)d.b * p.G + h) * DV + c);
                        uint2 v;
                        v.x = pack_bf16(o.x * inv, o.y * inv);
                        v.y = pack_bf16(o.z * inv, o.w * inv);
                        *reinterpret_cast<uint2*>(p.out + off) = v;
                    }
                    if (tid == 0) p.ws_cnt[d.b] = 0;
                }
            }
            named_bar_sync(1, NCW * 32);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        span_end(p.span);
        __threadfence();
        const unsigned done = atomicAdd(p.sched + 1, 1u);
        if (done == gridDim.x - 1) {
            p.sched[0] = 0u;
            p.sched[1] = 0u;
            __threadfence();
        }
    }
}


}  // namespace

bool spd_mla_decode_ok(const semipd_pool* p, int Hq) {
    const auto& c = p->cfg;
    const int bs = c.block_size;
    return c.dtype == SEMIPD_BF16 && c.kv_shared && c.num_kv_heads == 1 && c.head_dim_k == DK &&
           c.head_dim_v == DV && Hq <= NH && p->have_mla_map && (bs == 32 || bs == 64 || bs == 128);
}

size_t spd_mla_ws_bytes(int B, int max_ctx) {  // split partials only (see SpdWs)
    const int S_max = (max_ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
    return spd_ws_partial_bytes((size_t)B * NH, S_max, DV);
}

semipd_status spd_launch_decode_mla(semipd_pool_t pool, int layer, const void* q, const void* k_new,
                                    const int* req_ids, const int* ctx_lens, int batch,
                                    int max_ctx_len, int Hq, float scale, void* out,
                                    int out_head_major, void* workspace, size_t ws_bytes,
                                    int budget, int* status_dev, cudaStream_t st) {
    const int S_max = (max_ctx_len + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
    SpdWs w;
    if (!spd_ws_carve(workspace, ws_bytes, batch, (size_t)batch * NH, S_max, DV, &w))
        return SEMIPD_ERR_INVALID;
    MlaParams prm;
    prm.q = static_cast<const __nv_bfloat16*>(q);
    prm.k_new = static_cast<const uint4*>(k_new);
    prm.req_ids = req_ids;
    prm.ctx_lens = ctx_lens;
    prm.bt = pool->bt;
    prm.k_pool = static_cast<unsigned char*>(pool->k_layer(layer));
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.ws_cnt = w.cnt;
    prm.sched = w.sched;
    prm.ws_m = w.m;
    prm.ws_l = w.l;
    prm.ws_acc = w.acc;
    prm.status = status_dev;
    prm.span = spd_next_span(pool);
    prm.skip_append = pool->rope_on ? 1 : 0;
    prm.B = batch;
    prm.lg_bs = __builtin_ctz((unsigned)pool->cfg.block_size);
    prm.MBR = pool->cfg.max_blocks_per_req;
    prm.N_B = pool->cfg.num_blocks;
    prm.S_max = S_max;
    prm.n_units = batch * S_max;
    prm.out_head_major = out_head_major;
    prm.G = Hq;
    prm.scale_log2 = scale * LOG2E;
    prm.trace = spd_trace(pool);
    const size_t smem = 1024 + NSTAGE * STAGE_BYTES + NCW * NH * SROW * 4 + NH * PROW + 3 * NH * 4 +
                        (2 * NSTAGE + 4) * 8 + 2 * sizeof(MUnit) + 16;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(decode_mla_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr = true;
    }
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    decode_mla_kernel<<<grid, NTHREADS, smem, st>>>(pool->mla_kmap[layer], prm);
    pool->launches += 1;
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
