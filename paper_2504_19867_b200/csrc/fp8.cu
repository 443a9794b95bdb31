// fp8.cu — FP8 (E4M3) KV pages ("FP8 precision"; R31).
//
// Write rule: code = E4M3_rne_satfinite(fl32(x / s)); read rule: s * value(code); s is the
// layer's fp32 tensor scale.  This file holds every FP8-specific kernel and host call:
//   kv_write_fp8_kernel      the quantised K/V write of a prefill chunk;
//   dequant_prefix_kernel    a call's prefix pages -> bf16 staging pages, which the tcgen05
//                            prefill kernel then reads exactly as it reads a bf16 pool;
//   decode_fp8_kernel        split-K paged decode straight from E4M3 pages (fused append).
// The decode kernel is HBM-bound like the bf16 one (8 FLOP per cached byte at G = 4, far under
// the tensor / ALU ceilings), so it keeps the bf16 kernels' shape: a TMA producer warp
// streaming 32 KiB stages (one 16 KiB box = the two head pages of a (block, head pair) for K,
// one for V) into a 6-deep ring, 3 pairs of consumer warps (stage gs -> pair gs % 3, warp e of
// the pair takes head g0 + e).  Consumers convert the codes to f16 in registers (cvt
// e4m3x2 -> f16x2 is exact: every E4M3 value is an f16 value) and run swap-AB mma.sync
// m16n8k16 f16 with fp32 accumulation; k_scale is folded into the softmax scale and v_scale
// into the final 1 / l.  No shared-memory round trip for the conversion:
//   K (A operand, rows = keys): ldmatrix gives lane (r, t) bytes 4t..4t+3 of a 16-byte chunk
//     c of key row r; the MMA's k slots (2t, 2t+1) / (2t+8, 2t+9) stand for head dims
//     16c + 4t + {0,1} / {2,3} — a fixed permutation of the contraction index, applied to Q's
//     B fragments too, so every score is unchanged.
//   V (A operand of O^T = V^T P^T, rows = dv): ldmatrix.trans gives lane (g, t) the byte pairs
//     (key 2t: dv 2g, 2g+1) and (key 2t+1: dv 2g, 2g+1); one PRMT regroups them into
//     (dv 2g: keys 2t, 2t+1) and (dv 2g+1: keys 2t, 2t+1), so MMA row g is dv 16c + 2g and
//     row g + 8 is dv 16c + 2g + 1 — undone when the partials are written out.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int HD = 128;
constexpr int BS = 64;                   // FP8 pools: 64-token pages
constexpr int KPS = 64;                  // keys per stage = one page
constexpr int PAGE = KPS * HD;           // 8 KiB of codes: one (block, head) page
constexpr int STAGE = 4 * PAGE;          // K(g0) K(g0+1) V(g0) V(g0+1)
constexpr int NCW = 3;                   // consumer warp pairs (stage rotation)
constexpr int NST = 6;                   // ring depth (192 KiB)
constexpr int GMAX = 8;                  // q heads per kv head (swap-AB: MMA N = 8)
constexpr int NTHREADS = (2 * NCW + 1) * 32;
constexpr int SPLIT_KEYS = 4096;         // same split rule as the bf16 decode kernels
// SPD_F8_PIECES = 4: each split of >= 8 stages is cut further into pieces of 1/2, 1/4, 1/8, 1/8
// of its stages, handed out largest first (guided self-scheduling), aimed at the wave
// quantisation of 256 equal units (0.057 ms at 89 SMs = 2.88 -> 3 waves, 0.070 ms at 81 SMs =
// 3.16 -> 4 waves).  Parity-green but measured much SLOWER (0.091 ms at 89 SMs, 0.068 at 148;
// profiles/r2_fp8_pieces_ab.log): every unit ends in a 6-warp merge and a partial round trip,
// about 4 us per unit, far more than the tail it removes.  Default 1 (whole splits).
#ifndef SPD_F8_PIECES
#define SPD_F8_PIECES 1
#endif
constexpr int NPIECE = SPD_F8_PIECES;
constexpr float LOG2E = 1.4426950408889634f;
static_assert(NST % NCW == 0, "each ring slot must have one fixed consumer pair");
// Code -> f16 conversion per operand: 0 = cvt.rn.f16x2.e4m3x2 (F2FP, 2 per 4 codes), 1 = integer
// bit moves (f8x4_to_h2x2_alu, values / 256, about 5 LOP3 / SHF per 4 codes, and no PRMT for V).
// Measured (profiles/r2_fp8_conversion_ab.log, cfg-2 decode, ms at 44 / 89 / 148 SMs): F2FP for
// both 0.099 / 0.056 / 0.050; ALU V 0.118 / 0.064 / 0.052; ALU K 0.127 / 0.068 / 0.053; ALU both
// 0.150 / 0.081 / 0.058 — the conversion pipe is not what bounds the kernel, the extra integer
// instructions cost more than they relieve, so both stay on F2FP.
#ifndef SPD_F8_KALU
#define SPD_F8_KALU 0
#endif
#ifndef SPD_F8_VALU
#define SPD_F8_VALU 0
#endif

SPD_DEV uint32_t f8x2_to_h2(uint32_t two_codes /* low 16 bits */) {
    const __half2_raw h =
        __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)(two_codes & 0xFFFFu), __NV_E4M3);
    return (uint32_t)h.x | ((uint32_t)h.y << 16);
}

// four codes -> (f16x2 of the low two, f16x2 of the high two); exact
SPD_DEV void f8x4_to_h2x2(uint32_t x, uint32_t& lo, uint32_t& hi) {
    asm("{\n\t.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
        "cvt.rn.f16x2.e4m3x2 %0, l;\n\tcvt.rn.f16x2.e4m3x2 %1, h;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "r"(x));
}

// four codes -> f16x2 of bytes (0, 2) and f16x2 of bytes (1, 3), each value(code) / 256, exact:
// the 7 magnitude bits move one bit down onto the f16 exponent / mantissa fields and the sign
// stays on the sign bit; the bias difference (15 vs 7) leaves a factor 2^-8, subnormals included
SPD_DEV void f8x4_to_h2x2_alu(uint32_t q, uint32_t& even, uint32_t& odd) {
    odd = (q & 0x80008000u) | ((q & 0x7F007F00u) >> 1);
    const uint32_t q8 = q << 8;
    even = (q8 & 0x80008000u) | ((q8 & 0x7F007F00u) >> 1);
}

// quant2 / quant8 (the write rule above) live in common.cuh: the fused RoPE write uses them too

// 16 codes -> 16 bf16 of s * value(code) (2 x uint4 per 16 B of codes)
SPD_DEV void dequant16(uint4 c, float s, uint4& lo, uint4& hi) {
    const uint32_t w[4] = {c.x, c.y, c.z, c.w};
    uint32_t o[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t f = f8x2_to_h2(w[i] >> (16 * h));
            const float a = __half2float(__ushort_as_half((unsigned short)(f & 0xFFFFu))) * s;
            const float b = __half2float(__ushort_as_half((unsigned short)(f >> 16))) * s;
            o[2 * i + h] = pack_bf16(a, b);
        }
    }
    lo = make_uint4(o[0], o[1], o[2], o[3]);
    hi = make_uint4(o[4], o[5], o[6], o[7]);
}

SPD_DEV uint32_t pack_f16(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

SPD_DEV void mma_f16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

SPD_DEV uint32_t prmt_self(uint32_t a, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(a), "r"(sel));
    return r;
}

SPD_DEV void set_status(int* st, int v) {
    if (st) atomicMax(st, v);
}

// last request i with cu[i] <= row
SPD_DEV int row_request(const int* cu, int n, int row) {
    int i = 0, hi = n - 1;
    while (i < hi) {
        const int mid = (i + hi + 1) >> 1;
        if (__ldg(cu + mid) <= row) i = mid; else hi = mid - 1;
    }
    return i;
}

// ---------------------------------------------------------------------------------------
// Quantised K/V write of prefill rows: one warp per (row, kv head); lanes 0-15 write
// K (8 elements = 8 codes each), 16-31 V.
struct KvWriteArgs {
    const int* cu;        // [n+1]
    const int* req;       // [n]
    const int* pos0;      // [n] prefix lengths
    const int* bt;
    const uint4* k_new;   // [rows][Hkv][128] bf16
    const uint4* v_new;
    unsigned char* k_pool;
    unsigned char* v_pool;
    int* status;
    int n, rows, Hkv, MBR, N_B;
    float ks, vs;
};

constexpr int kWarps = 8;

__global__ void __launch_bounds__(kWarps * 32) kv_write_fp8_kernel(KvWriteArgs a) {
    pdl_wait();  // PDL: the previous kernel is complete; the next may launch (it waits itself)
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const long long total = (long long)a.rows * a.Hkv;
    for (long long u = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); u < total;
         u += (long long)gridDim.x * kWarps) {
        const int row = (int)(u / a.Hkv), g = (int)(u % a.Hkv);
        const int i = row_request(a.cu, a.n, row);
        const int pos = __ldg(a.pos0 + i) + row - __ldg(a.cu + i);
        const int page = pos / BS;
        const int blk = page < a.MBR ? __ldg(a.bt + (size_t)__ldg(a.req + i) * a.MBR + page) : -1;
        if (blk < 0 || blk >= a.N_B) {
            if (lane == 0) set_status(a.status, SEMIPD_ERR_BAD_BLOCK);
            continue;
        }
        const size_t slot = ((size_t)blk * a.Hkv + g) * BS + (pos % BS);
        const int c = lane & 15;
        const bool isv = lane >= 16;
        const uint4 x = __ldg((isv ? a.v_new : a.k_new) + ((size_t)row * a.Hkv + g) * (HD / 8) + c);
        reinterpret_cast<uint2*>(isv ? a.v_pool : a.k_pool)[slot * (HD / 8) + c] =
            quant8(x, isv ? a.vs : a.ks);
    }
}

// ---------------------------------------------------------------------------------------
// Prefix pages of a prefill call -> bf16 staging pages (scratch page (i * MBR + j) * Hkv + g
// for request i, page j, head g).  K pages stage value(code) exactly (every E4M3 value is a
// bf16 value; the prefill kernel applies k_scale to the prefix tiles' logits), V pages stage
// bf16(v_scale * value(code)) (one bf16 rounding of V, the order of the P rounding the PV MMA
// already has).  One warp per (i, j, g, tensor); pages past the prefix are
// skipped (the attention never reads them); a bad table entry sets BAD_BLOCK and stages zeros
// (the bf16 path's TMA zero fill).
struct DequantArgs {
    const int* req;
    const int* prefix;
    const int* bt;
    const unsigned char* k_pool;
    const unsigned char* v_pool;
    uint4* sk;            // staging K pages [cap * MBR * Hkv][64][128] bf16
    uint4* sv;
    int* status;
    int n, Hkv, MBR, N_B;
    float ks, vs;
};

__global__ void __launch_bounds__(kWarps * 32) dequant_prefix_kernel(DequantArgs a) {
    pdl_wait();  // PDL: the previous kernel is complete; the next may launch (it waits itself)
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const long long total = (long long)a.n * a.MBR * a.Hkv * 2;
    for (long long u = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); u < total;
         u += (long long)gridDim.x * kWarps) {
        const int tsel = (int)(u & 1);
        const long long w = u >> 1;
        const int g = (int)(w % a.Hkv);
        const int j = (int)((w / a.Hkv) % a.MBR);
        const int i = (int)(w / ((long long)a.Hkv * a.MBR));
        const int P = __ldg(a.prefix + i);
        if (j * BS >= P) continue;
        const int blk = __ldg(a.bt + (size_t)__ldg(a.req + i) * a.MBR + j);
        const bool ok = blk >= 0 && blk < a.N_B;
        if (!ok && lane == 0 && tsel == 0) set_status(a.status, SEMIPD_ERR_BAD_BLOCK);
        const uint4* src = reinterpret_cast<const uint4*>(tsel ? a.v_pool : a.k_pool) +
                           ((size_t)(ok ? blk : 0) * a.Hkv + g) * (PAGE / 16);
        uint4* dst = (tsel ? a.sv : a.sk) + (((size_t)i * a.MBR + j) * a.Hkv + g) * (2 * PAGE / 16);
        const float s = tsel ? a.vs : a.ks;
#pragma unroll 4
        for (int c = lane; c < PAGE / 16; c += 32) {
            uint4 lo = make_uint4(0, 0, 0, 0), hi = lo;
            if (ok) dequant16(__ldg(src + c), s, lo, hi);
            dst[2 * c] = lo;
            dst[2 * c + 1] = hi;
        }
    }
}

// ---------------------------------------------------------------------------------------
struct Unit {
    int b, g, s, S, k0, k1, base, nst;  // b < 0: no more work
};

struct DecParams {
    const __nv_bfloat16* q;      // [B][Hq][128]
    const uint4* k_new;          // [B][Hkv][128] bf16
    const uint4* v_new;
    const int* req_ids;
    const int* ctx_lens;
    const int* bt;
    unsigned char* k_pool;       // layer base (codes)
    unsigned char* v_pool;
    __nv_bfloat16* out;
    float* ws_m;                 // [B][Hq][S_max * NPIECE]
    float* ws_l;
    float* ws_acc;               // [B][Hq][S_max * NPIECE][128]
    int* ws_cnt;                 // [B][Hkv]
    unsigned* sched;             // [2]
    int* status;
    unsigned long long* span;
    int B, Hq, Hkv, G, MBR, N_B, S_max, n_units, out_head_major;
    int skip_append;  // 1: the step's rows are already in the pool (fused RoPE write, R28)
    float scale_log2;            // softmax_scale * k_scale * log2(e)
    float ks, vs;                // write scales (append)
    float v_out;                 // v_scale, applied with 1 / l
    SpdTrace trace;
    // TP head all-gather fused into the epilogue (N2, as decode.cu): every output vector is also
    // stored to each peer's gathered buffer (peer-mapped, already offset to this rank's shard)
    __nv_bfloat16* peers[SEMIPD_MAX_PEERS - 1];
    int n_peers;
};

// one bf16x4 output vector: local buffer, then every peer's gathered buffer
__device__ __forceinline__ void f8_store_out(const DecParams& p, size_t off, uint2 v) {
    *reinterpret_cast<uint2*>(p.out + off) = v;
#pragma unroll
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
        if (k < p.n_peers) *reinterpret_cast<uint2*>(p.peers[k] + off) = v;
}

__global__ void __launch_bounds__(NTHREADS, 1)
    decode_fp8_kernel(const __grid_constant__ CUtensorMap kmap, const __grid_constant__ CUtensorMap vmap,
                      DecParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ring = smem;                                           // NST x 32 KiB
    float* scr_acc = reinterpret_cast<float*>(ring + NST * STAGE);        // [6][8][128]
    float* scr_ml = scr_acc + 2 * NCW * GMAX * HD;                        // [6][8][2]
    uint64_t* full = reinterpret_cast<uint64_t*>(scr_ml + 2 * NCW * GMAX * 2);
    uint64_t* empty = full + NST;
    uint64_t* ufull = empty + NST;
    uint64_t* uempty = ufull + 2;
    Unit* units = reinterpret_cast<Unit*>(uempty + 2);
    int* s_last = reinterpret_cast<int*>(units + 2);

    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    const int NP = p.Hkv >> 1;  // head pairs per request
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 2);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(ufull + i, 1);
            mbar_init(uempty + i, 2 * NCW);
        }
        fence_mbar_init();
        if (p.trace.buf) {
            const int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(2, (int)smid(), (int)blockIdx.x, 9 /* kernel kind: FP8 decode */);
        }
    }
    __syncthreads();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (workspace, pool)
    if (threadIdx.x == 0) span_begin(p.span);

    if (warp == 2 * NCW) {
        // =========================== producer ===========================
        if (lane == 0) {
            tma_prefetch_desc(&kmap);
            tma_prefetch_desc(&vmap);
        }
        const uint64_t kv_pol = l2_policy(1);  // evict_first: the cache is read once per step
        const int oob_z = p.N_B * p.Hkv;
        int gstage = 0, nunit = 0;
        for (;;) {
            int u = 0;
            if (lane == 0) u = (int)atomicAdd(p.sched, 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
            Unit d;
            int ctx = 0;
            if (u >= p.n_units) {
                d.b = -1;
            } else {
                // unit order: piece (largest first), split, request, head pair
                const int piece = u / (p.S_max * p.B * NP);
                const int s0 = (u / (p.B * NP)) % p.S_max;
                d.b = (u / NP) % p.B;
                d.g = 2 * (u % NP);
                ctx = __ldg(p.ctx_lens + d.b);
                const int S0 = (ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
                if (s0 >= S0) continue;  // warp-uniform
                const int nk = ctx + 1;
                int len = (nk + S0 - 1) / S0;
                len = (len + KPS - 1) / KPS * KPS;
                const int np = len / KPS >= 8 ? NPIECE : 1;  // same for every split of the request
                if (piece >= np) continue;
                const int k0s = s0 * len, k1s = min(nk, k0s + len);
                const int ns = (k1s - k0s + KPS - 1) / KPS;
                int a = 0, e = ns;  // this piece's stages [a, e) of the split
                if (np > 1) {
                    const int c1 = ns / 2, c2 = c1 + (ns - c1) / 2, c3 = c2 + (ns - c2) / 2;
                    a = piece == 0 ? 0 : piece == 1 ? c1 : piece == 2 ? c2 : c3;
                    e = piece == 0 ? c1 : piece == 1 ? c2 : piece == 2 ? c3 : ns;
                }
                d.S = S0 * np;
                d.s = s0 * np + piece;
                d.k0 = k0s + a * KPS;
                d.k1 = min(k1s, k0s + e * KPS);
                if (d.k1 < d.k0) d.k1 = d.k0;  // empty piece: a (-inf, 0, 0) partial
                d.nst = (d.k1 - d.k0 + KPS - 1) / KPS;
                // align the unit's first stage to the pair rotation (R26: the stage -> warp
                // assignment depends on the unit only)
                while (gstage % NCW != 0) {
                    if (lane == 0) {
                        const int st = gstage % NST;
                        mbar_wait(empty + st, ((gstage / NST) & 1) ^ 1);
                        mbar_arrive(full + st);
                    }
                    ++gstage;
                }
                __syncwarp();
                d.base = gstage;
            }
            const int us = nunit & 1;
            if (lane == 0) {
                mbar_wait(uempty + us, ((nunit >> 1) & 1) ^ 1);
                units[us] = d;
                mbar_arrive(ufull + us);
            }
            __syncwarp();
            ++nunit;
            if (d.b < 0) {  // no more units: the next kernel on the stream may be scheduled
                pdl_trigger();
                break;
            }
            const int* btr = p.bt + (size_t)__ldg(p.req_ids + d.b) * p.MBR;
            const int last_page = ctx / BS;
            if (!p.skip_append && d.k0 <= ctx && ctx < d.k1) {
                // fused quantised append of both heads' K and V rows at slot ctx, by the
                // unit whose key range holds slot ctx (no other unit reads that slot): lane
                // = (tensor, head e, 16-element chunk c)
                const int blk = last_page < p.MBR ? __ldg(btr + last_page) : -1;
                if (blk >= 0 && blk < p.N_B) {
                    const int c = lane & 7, e = (lane >> 3) & 1;
                    const bool isv = lane >= 16;
                    const uint4* src = (isv ? p.v_new : p.k_new) + ((size_t)d.b * p.Hkv + d.g + e) * (HD / 8) + 2 * c;
                    const float s = isv ? p.vs : p.ks;
                    const uint2 lo = quant8(__ldg(src), s), hi = quant8(__ldg(src + 1), s);
                    const size_t slot = ((size_t)blk * p.Hkv + d.g + e) * BS + (ctx % BS);
                    reinterpret_cast<uint4*>(isv ? p.v_pool : p.k_pool)[slot * (HD / 16) + c] =
                        make_uint4(lo.x, lo.y, hi.x, hi.y);
                    fence_proxy_async_global();
                }
                __syncwarp();
            }
            auto lookup = [&](int i) -> int {  // raw block id of stage i (-2: past the unit)
                const int page = (d.k0 + i * KPS) / BS;
                if (i >= d.nst || page > last_page) return -2;
                return page < p.MBR ? __ldg(btr + page) : -1;
            };
            int zc = lookup(lane);
            for (int i = 0; i < d.nst; ++i, ++gstage) {
                const int st = gstage % NST;
                if (i > 0 && (i & 31) == 0) zc = lookup(i + lane);
                const int blk = __shfl_sync(0xffffffffu, zc, i & 31);
                if (lane == 0) {
                    mbar_wait(empty + st, ((gstage / NST) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + st, STAGE);
                    int z = oob_z;
                    if (blk >= 0 && blk < p.N_B) z = blk * p.Hkv + d.g;
                    else if (blk != -2) set_status(p.status, SEMIPD_ERR_BAD_BLOCK);
                    unsigned char* dst = ring + st * STAGE;
                    tma_load_3d_hint(dst, &kmap, full + st, 0, 0, z, kv_pol);
                    tma_load_3d_hint(dst + 2 * PAGE, &vmap, full + st, 0, 0, z, kv_pol);
                }
                __syncwarp();
            }
        }
    } else {
        // ================= consumers: swap-AB f16, heads are the MMA N =================
        const int pw = warp >> 1, e = warp & 1;  // pair (stage rotation), head of the pair
        const int kr = lane >> 2;                // key (S^T) / dv-pair (O^T) row in 8-row blocks
        const int t4 = lane & 3;
        const int hc = 2 * t4;                   // heads hc, hc + 1 of this lane's C values
        const int lm = (lane >> 3) & 1, lc = lane >> 4, lr = lane & 7;  // ldmatrix roles
        int nunit = 0;
        int next_gs = pw;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(ufull + us, (nunit >> 1) & 1);
            const Unit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(uempty + us);
            ++nunit;
            if (d.b < 0) break;
            const int g = d.g + e;
            // Q^T B fragments in f16: head n = kr; k slots (2t, 2t+1) / (2t+8, 2t+9) of k-step
            // c are head dims 16c + 4t + {0,1} / {2,3} (F2FP K: low / high code pair) or
            // 16c + 4t + {0,2} / {1,3} (ALU K: even / odd codes) — the K permutation above
            uint32_t qb[8][2];
            {
                const bool v = kr < p.G;
                const uint2* q2 = reinterpret_cast<const uint2*>(p.q + ((size_t)d.b * p.Hq + g * p.G + (v ? kr : 0)) * HD);
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint2 x = v ? __ldg(q2 + 4 * c + t4) : make_uint2(0u, 0u);
                    const float d0 = __uint_as_float(x.x << 16), d1 = __uint_as_float(x.x & 0xFFFF0000u);
                    const float d2 = __uint_as_float(x.y << 16), d3 = __uint_as_float(x.y & 0xFFFF0000u);
                    qb[c][0] = SPD_F8_KALU ? pack_f16(d0, d2) : pack_f16(d0, d1);
                    qb[c][1] = SPD_F8_KALU ? pack_f16(d1, d3) : pack_f16(d2, d3);
                }
            }
            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
            float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
            while (next_gs < d.base) {  // padding stages in front of this unit
                const int st = next_gs % NST;
                mbar_wait(full + st, (next_gs / NST) & 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
                next_gs += NCW;
            }
            next_gs = d.base + (pw < d.nst ? pw + ((d.nst - 1 - pw) / NCW + 1) * NCW : pw);
            for (int i = pw; i < d.nst; i += NCW) {
                const int gs = d.base + i;
                const int st = gs % NST;
                mbar_wait(full + st, (gs / NST) & 1);
                const uint32_t kst = smem_u32(ring + st * STAGE) + e * PAGE;
                const uint32_t vst = kst + 2 * PAGE;
                // ---- S^T [16 keys x 8 heads] per key tile: A = K codes -> f16
                float s[4][4];
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    s[kt][0] = s[kt][1] = s[kt][2] = s[kt][3] = 0.f;
                    const int key = kt * 16 + lm * 8 + lr;
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int c = 2 * cc + lc;
                        uint32_t r0, r1, r2, r3;
                        ldsm_x4(kst + key * 128 + ((c ^ (key & 7)) << 4), r0, r1, r2, r3);
                        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
                        if constexpr (SPD_F8_KALU) {
                            f8x4_to_h2x2_alu(r0, a0, a2);
                            f8x4_to_h2x2_alu(r1, a1, a3);
                            f8x4_to_h2x2_alu(r2, b0, b2);
                            f8x4_to_h2x2_alu(r3, b1, b3);
                        } else {
                            f8x4_to_h2x2(r0, a0, a2);
                            f8x4_to_h2x2(r1, a1, a3);
                            f8x4_to_h2x2(r2, b0, b2);
                            f8x4_to_h2x2(r3, b1, b3);
                        }
                        mma_f16_16816(s[kt], a0, a1, a2, a3, qb[2 * cc][0], qb[2 * cc][1]);
                        mma_f16_16816(s[kt], b0, b1, b2, b3, qb[2 * cc + 1][0], qb[2 * cc + 1][1]);
                    }
                }
                // ---- mask + online softmax per head (log2 domain; k_scale folded in)
                const int kbase = d.k0 + i * KPS;
                const bool tail = kbase + KPS > d.k1;
                float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
                for (int kt = 0; kt < 4; ++kt)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float x = s[kt][q] * p.scale_log2;
                        if (tail && kbase + kt * 16 + kr + (q >> 1) * 8 >= d.k1) x = -INFINITY;
                        s[kt][q] = x;
                        mx[q & 1] = fmaxf(mx[q & 1], x);
                    }
                float alpha[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 4));
                    mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 8));
                    mx[j] = fmaxf(mx[j], __shfl_xor_sync(0xffffffffu, mx[j], 16));
                    const float mnew = fmaxf(mrow[j], mx[j]);
                    alpha[j] = fast_exp2(mrow[j] - mnew);
                    mrow[j] = mnew;
                }
                float ls[2] = {0.f, 0.f};
                uint32_t pb[4][2];
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    const float p0 = fast_exp2(s[kt][0] - mrow[0]);
                    const float p1 = fast_exp2(s[kt][1] - mrow[1]);
                    const float p2 = fast_exp2(s[kt][2] - mrow[0]);
                    const float p3 = fast_exp2(s[kt][3] - mrow[1]);
                    ls[0] += p0 + p2;
                    ls[1] += p1 + p3;
                    pb[kt][0] = movmatrix_t(pack_f16(p0, p1));  // C (keys x heads) -> B (k, n)
                    pb[kt][1] = movmatrix_t(pack_f16(p2, p3));
                }
                lrow[0] = lrow[0] * alpha[0] + ls[0];
                lrow[1] = lrow[1] * alpha[1] + ls[1];
                if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
                    for (int dt = 0; dt < 8; ++dt) {
                        acc[dt][0] *= alpha[0];
                        acc[dt][1] *= alpha[1];
                        acc[dt][2] *= alpha[0];
                        acc[dt][3] *= alpha[1];
                    }
                }
                // ---- O^T [16 dv x 8 heads] += V^T P^T per dv tile: A = V codes (trans) -> f16
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    const int key = kt * 16 + lm * 8 + lr;
#pragma unroll
                    for (int dc = 0; dc < 4; ++dc) {
                        const int c = 2 * dc + lc;
                        uint32_t r0, r1, r2, r3;
                        ldsm_x4_t(vst + key * 128 + ((c ^ (key & 7)) << 4), r0, r1, r2, r3);
                        uint32_t a0, a1, a2, a3, b0, b1, b2, b3;
                        if constexpr (SPD_F8_VALU) {  // even codes = dv 2g, odd = dv 2g + 1
                            f8x4_to_h2x2_alu(r0, a0, a1);
                            f8x4_to_h2x2_alu(r1, a2, a3);
                            f8x4_to_h2x2_alu(r2, b0, b1);
                            f8x4_to_h2x2_alu(r3, b2, b3);
                        } else {
                            f8x4_to_h2x2(prmt_self(r0, 0x3120), a0, a1);
                            f8x4_to_h2x2(prmt_self(r1, 0x3120), a2, a3);
                            f8x4_to_h2x2(prmt_self(r2, 0x3120), b0, b1);
                            f8x4_to_h2x2(prmt_self(r3, 0x3120), b2, b3);
                        }
                        mma_f16_16816(acc[2 * dc], a0, a1, a2, a3, pb[kt][0], pb[kt][1]);
                        mma_f16_16816(acc[2 * dc + 1], b0, b1, b2, b3, pb[kt][0], pb[kt][1]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
            }
            // ---- per-warp partial -> shared scratch (rows = heads, dv un-permuted)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 4);
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 8);
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 16);
            }
            const int wi = pw * 2 + e;
            float* wacc = scr_acc + wi * GMAX * HD;
#pragma unroll
            for (int dt = 0; dt < 8; ++dt) {
                const int dv = dt * 16 + 2 * kr;
                *reinterpret_cast<float2*>(wacc + hc * HD + dv) = make_float2(acc[dt][0], acc[dt][2]);
                *reinterpret_cast<float2*>(wacc + (hc + 1) * HD + dv) = make_float2(acc[dt][1], acc[dt][3]);
            }
            if (kr == 0) {
                scr_ml[(wi * GMAX + hc) * 2 + 0] = mrow[0];
                scr_ml[(wi * GMAX + hc) * 2 + 1] = lrow[0];
                scr_ml[(wi * GMAX + hc + 1) * 2 + 0] = mrow[1];
                scr_ml[(wi * GMAX + hc + 1) * 2 + 1] = lrow[1];
            }
            named_bar_sync(1, 2 * NCW * 32);
            // ---- cross-warp merge: thread handles (head e of the pair, q head h, 4 columns)
            const int tid = threadIdx.x;
            const bool split = d.S > 1;
            for (int idx = tid; idx < 2 * p.G * (HD / 4); idx += 2 * NCW * 32) {
                const int ee = idx / (p.G * (HD / 4));
                const int h = (idx / (HD / 4)) % p.G, c = (idx % (HD / 4)) * 4;
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < NCW; ++w) M = fmaxf(M, scr_ml[((w * 2 + ee) * GMAX + h) * 2]);
                float L = 0.f;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < NCW; ++w) {
                    const int wj = w * 2 + ee;
                    const float mw = scr_ml[(wj * GMAX + h) * 2];
                    const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
                    L += f * scr_ml[(wj * GMAX + h) * 2 + 1];
                    const float4 a = *reinterpret_cast<const float4*>(scr_acc + (wj * GMAX + h) * HD + c);
                    o.x += f * a.x;
                    o.y += f * a.y;
                    o.z += f * a.z;
                    o.w += f * a.w;
                }
                const int hq = (d.g + ee) * p.G + h;
                if (!split) {
                    const float inv = p.v_out / L;
                    const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                        : (((size_t)d.b * p.Hq + hq) * HD + c);
                    uint2 v;
                    v.x = pack_bf16(o.x * inv, o.y * inv);
                    v.y = pack_bf16(o.z * inv, o.w * inv);
                    f8_store_out(p, off, v);
                } else {
                    const size_t pi = ((size_t)d.b * p.Hq + hq) * (p.S_max * NPIECE) + d.s;
                    *reinterpret_cast<float4*>(p.ws_acc + pi * HD + c) = o;
                    if (c == 0) {
                        p.ws_m[pi] = M;
                        p.ws_l[pi] = L;
                    }
                }
            }
            if (split) {
                __threadfence();
                named_bar_sync(1, 2 * NCW * 32);
                if (tid == 0) *s_last = atomicAdd(p.ws_cnt + d.b * p.Hkv + d.g, 1) == d.S - 1;
                named_bar_sync(1, 2 * NCW * 32);
                if (*s_last) {
                    __threadfence();
                    // merge over splits in split-index order (flash-decoding)
                    for (int idx = tid; idx < 2 * p.G * (HD / 4); idx += 2 * NCW * 32) {
                        const int ee = idx / (p.G * (HD / 4));
                        const int h = (idx / (HD / 4)) % p.G, c = (idx % (HD / 4)) * 4;
                        const int hq = (d.g + ee) * p.G + h;
                        const size_t pb0 = ((size_t)d.b * p.Hq + hq) * (p.S_max * NPIECE);
                        float M = -INFINITY;
                        for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb0 + sI));
                        float L = 0.f;
                        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int sI = 0; sI < d.S; ++sI) {
                            const float f = fast_exp2(__ldcg(p.ws_m + pb0 + sI) - M);
                            L += f * __ldcg(p.ws_l + pb0 + sI);
                            const float4 a = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + (pb0 + sI) * HD + c));
                            o.x += f * a.x;
                            o.y += f * a.y;
                            o.z += f * a.z;
                            o.w += f * a.w;
                        }
                        const float inv = p.v_out / L;
                        const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                            : (((size_t)d.b * p.Hq + hq) * HD + c);
                        uint2 v;
                        v.x = pack_bf16(o.x * inv, o.y * inv);
                        v.y = pack_bf16(o.z * inv, o.w * inv);
                        f8_store_out(p, off, v);
                    }
                    if (tid == 0) p.ws_cnt[d.b * p.Hkv + d.g] = 0;  // ready for the next call
                }
            }
            named_bar_sync(1, 2 * NCW * 32);  // scratch reuse
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        span_end(p.span);
        __threadfence();
        const unsigned done = atomicAdd(p.sched + 1, 1u);
        if (done == gridDim.x - 1) {  // last CTA: reset the work counter for the next launch
            p.sched[0] = 0u;
            p.sched[1] = 0u;
            __threadfence();
        }
    }
}

size_t decode_fp8_smem_bytes() {
    return 1024 + NST * STAGE + 2 * NCW * GMAX * HD * 4 + 2 * NCW * GMAX * 2 * 4 + (2 * NST + 4) * 8 +
           2 * sizeof(Unit) + 16;
}

// staging layout inside the caller's scratch: [ids int32[cap] | bt int32[cap][MBR] | K pages |
// V pages], every region 1 KiB aligned
struct ScratchLayout {
    size_t ids, bt, k, v, total;
};
size_t al1k(size_t x) { return (x + 1023) / 1024 * 1024; }
ScratchLayout scratch_layout(const semipd_pool* p, int cap) {
    const auto& c = p->cfg;
    ScratchLayout L{};
    const size_t pages = (size_t)cap * c.max_blocks_per_req * c.num_kv_heads;
    L.ids = 0;
    L.bt = al1k(sizeof(int) * (size_t)cap);
    L.k = L.bt + al1k(sizeof(int) * (size_t)cap * c.max_blocks_per_req);
    L.v = L.k + al1k(pages * BS * HD * 2);
    L.total = L.v + al1k(pages * BS * HD * 2);
    return L;
}

}  // namespace

int spd_fp8_pieces() { return NPIECE; }

bool spd_fp8_geometry_ok(const semipd_pool_config* c) {
    return c->head_dim_k == HD && c->head_dim_v == HD && c->block_size == BS &&
           c->num_kv_heads % 2 == 0 && !c->kv_shared;
}

bool spd_fp8_init_maps(semipd_pool* p) {
    const auto& c = p->cfg;
    const uint64_t pages = (uint64_t)c.num_blocks * c.num_kv_heads;
    p->f8kmap.resize(c.num_layers);
    p->f8vmap.resize(c.num_layers);
    p->k_scale.assign(c.num_layers, 1.0f);
    p->v_scale.assign(c.num_layers, 1.0f);
    p->box_rows = BS;
    for (int l = 0; l < c.num_layers; ++l) {
        // (128 code bytes, 64 rows, pages); box = the two head pages of a (block, head pair)
        if (!spd_encode_tiled_3d(&p->f8kmap[l], CU_TENSOR_MAP_DATA_TYPE_UINT8, p->k_layer(l), HD, BS,
                                 pages, HD, HD * BS, HD, BS, 2, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !spd_encode_tiled_3d(&p->f8vmap[l], CU_TENSOR_MAP_DATA_TYPE_UINT8, p->v_layer(l), HD, BS,
                                 pages, HD, HD * BS, HD, BS, 2, CU_TENSOR_MAP_SWIZZLE_128B))
            return false;
    }
    p->have_f8_maps = true;
    return true;
}

semipd_status spd_launch_kv_write_fp8(semipd_pool_t p, int layer, const void* k_new, const void* v_new,
                                      const int* cu_seqlens, const int* req_ids, const int* pos0,
                                      int n, int total_rows, int* status_dev, cudaStream_t s) {
    if (total_rows <= 0) return SEMIPD_OK;
    const auto& c = p->cfg;
    KvWriteArgs a;
    a.cu = cu_seqlens;
    a.req = req_ids;
    a.pos0 = pos0;
    a.bt = p->bt;
    a.k_new = static_cast<const uint4*>(k_new);
    a.v_new = static_cast<const uint4*>(v_new);
    a.k_pool = static_cast<unsigned char*>(p->k_layer(layer));
    a.v_pool = static_cast<unsigned char*>(p->v_layer(layer));
    a.status = status_dev;
    a.n = n;
    a.rows = total_rows;
    a.Hkv = c.num_kv_heads;
    a.MBR = c.max_blocks_per_req;
    a.N_B = c.num_blocks;
    a.ks = p->k_scale[layer];
    a.vs = p->v_scale[layer];
    long long grid = ((long long)total_rows * c.num_kv_heads + kWarps - 1) / kWarps;
    if (grid > 16LL * p->num_sms) grid = 16LL * p->num_sms;
    const cudaError_t le = spd_launch_pdl(kv_write_fp8_kernel, dim3((unsigned)grid), dim3(kWarps * 32), 0, s, a);
    p->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

semipd_status spd_launch_dequant_prefix(semipd_pool_t p, int layer, const int* req_ids,
                                        const int* prefix_lens, int n, int budget, int* status_dev,
                                        cudaStream_t s) {
    const auto& c = p->cfg;
    const ScratchLayout L = scratch_layout(p, p->f8s_cap);
    DequantArgs a;
    a.req = req_ids;
    a.prefix = prefix_lens;
    a.bt = p->bt;
    a.k_pool = static_cast<const unsigned char*>(p->k_layer(layer));
    a.v_pool = static_cast<const unsigned char*>(p->v_layer(layer));
    a.sk = reinterpret_cast<uint4*>(p->f8s + L.k);
    a.sv = reinterpret_cast<uint4*>(p->f8s + L.v);
    a.status = status_dev;
    a.n = n;
    a.Hkv = c.num_kv_heads;
    a.MBR = c.max_blocks_per_req;
    a.N_B = c.num_blocks;
    a.ks = 1.0f;  // exact codes; k_scale is applied to the logits (scale_log2_pre)
    a.vs = p->v_scale[layer];
    const long long work = (long long)n * c.max_blocks_per_req * c.num_kv_heads * 2;
    long long grid = (work + kWarps - 1) / kWarps;
    const long long cap = budget > 0 ? 4LL * budget : 4LL * p->num_sms;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    const cudaError_t le = spd_launch_pdl(dequant_prefix_kernel, dim3((unsigned)grid), dim3(kWarps * 32), 0, s, a);
    p->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

void spd_fp8_prefill_view(const semipd_pool* p, const int** ids, const int** bt, int* n_pages_blocks) {
    const ScratchLayout L = scratch_layout(p, p->f8s_cap);
    *ids = reinterpret_cast<const int*>(p->f8s + L.ids);
    *bt = reinterpret_cast<const int*>(p->f8s + L.bt);
    *n_pages_blocks = p->f8s_cap * p->cfg.max_blocks_per_req;
}

semipd_status spd_launch_decode_fp8(semipd_pool_t pool, int layer, const void* q, const void* k_new,
                                    const void* v_new, const int* req_ids, const int* ctx_lens,
                                    int batch, int max_ctx_len, int Hq, float scale, void* out,
                                    int out_head_major, void* workspace, size_t ws_bytes, int budget,
                                    int* status_dev, cudaStream_t st) {
    const auto& c = pool->cfg;
    const int G = Hq / c.num_kv_heads;
    if (G > GMAX || !pool->have_f8_maps) return SEMIPD_ERR_UNSUPPORTED;
    const int S0_max = (max_ctx_len + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
    SpdWs w;
    if (!spd_ws_carve(workspace, ws_bytes, (size_t)batch * c.num_kv_heads, (size_t)batch * Hq,
                      (size_t)S0_max * NPIECE, HD, &w))
        return SEMIPD_ERR_INVALID;
    DecParams prm;
    prm.q = static_cast<const __nv_bfloat16*>(q);
    prm.k_new = static_cast<const uint4*>(k_new);
    prm.v_new = static_cast<const uint4*>(v_new);
    prm.req_ids = req_ids;
    prm.ctx_lens = ctx_lens;
    prm.bt = pool->bt;
    prm.k_pool = static_cast<unsigned char*>(pool->k_layer(layer));
    prm.v_pool = static_cast<unsigned char*>(pool->v_layer(layer));
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.ws_m = w.m;
    prm.ws_l = w.l;
    prm.ws_acc = w.acc;
    prm.ws_cnt = w.cnt;
    prm.sched = w.sched;
    prm.status = status_dev;
    prm.span = spd_next_span(pool);
    prm.B = batch;
    prm.Hq = Hq;
    prm.Hkv = c.num_kv_heads;
    prm.G = G;
    prm.MBR = c.max_blocks_per_req;
    prm.N_B = c.num_blocks;
    prm.S_max = S0_max;  // unit enumeration; partial rows are indexed [B][Hq][S_max * NPIECE]
    prm.n_units = NPIECE * S0_max * batch * (c.num_kv_heads / 2);
    prm.out_head_major = out_head_major;
    prm.skip_append = pool->rope_on ? 1 : 0;
    prm.n_peers = pool->dec_n_peers;
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
        prm.peers[k] = k < pool->dec_n_peers ? static_cast<__nv_bfloat16*>(pool->dec_peers[k]) : nullptr;
    prm.scale_log2 = scale * pool->k_scale[layer] * LOG2E * (SPD_F8_KALU ? 256.f : 1.f);
    prm.ks = pool->k_scale[layer];
    prm.vs = pool->v_scale[layer];
    prm.v_out = pool->v_scale[layer] * (SPD_F8_VALU ? 256.f : 1.f);  // ALU codes are value / 256
    prm.trace = spd_trace(pool);
    const size_t smem = decode_fp8_smem_bytes();
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(decode_fp8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr = true;
    }
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    if (spd_launch_pdl(decode_fp8_kernel, dim3(grid), dim3(NTHREADS), smem, st, pool->f8kmap[layer],
                       pool->f8vmap[layer], prm) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    if (cudaGetLastError() != cudaSuccess) return SEMIPD_ERR_CUDA;
    pool->launches += 1;
    return SEMIPD_OK;
}

extern "C" {

semipd_status semipd_set_kv_scales(semipd_pool_t pool, const float* k_scales, const float* v_scales) {
    if (!pool || pool->cfg.dtype != SEMIPD_FP8_E4M3) return SEMIPD_ERR_INVALID;
    const int L = pool->cfg.num_layers;
    for (const float* a : {k_scales, v_scales})
        if (a)
            for (int l = 0; l < L; ++l)
                if (!(a[l] > 0.f) || !std::isfinite(a[l])) return SEMIPD_ERR_INVALID;
    for (int l = 0; l < L; ++l) {
        if (k_scales) pool->k_scale[l] = k_scales[l];
        if (v_scales) pool->v_scale[l] = v_scales[l];
    }
    return SEMIPD_OK;
}

size_t semipd_fp8_prefill_scratch_bytes(semipd_pool_t pool, int32_t max_reqs_per_call) {
    if (!pool || pool->cfg.dtype != SEMIPD_FP8_E4M3 || max_reqs_per_call < 1) return 0;
    return scratch_layout(pool, max_reqs_per_call).total;
}

semipd_status semipd_set_fp8_prefill_scratch(semipd_pool_t pool, void* mem, size_t bytes,
                                             int32_t max_reqs_per_call) {
    if (!pool || pool->cfg.dtype != SEMIPD_FP8_E4M3) return SEMIPD_ERR_INVALID;
    if (!mem) {
        pool->f8s = nullptr;
        pool->f8s_cap = 0;
        pool->have_f8s_maps = false;
        return SEMIPD_OK;
    }
    if (max_reqs_per_call < 1 || reinterpret_cast<uintptr_t>(mem) % 1024) return SEMIPD_ERR_INVALID;
    const ScratchLayout L = scratch_layout(pool, max_reqs_per_call);
    if (bytes < L.total) return SEMIPD_ERR_INVALID;
    const auto& c = pool->cfg;
    const int MBR = c.max_blocks_per_req;
    unsigned char* base = static_cast<unsigned char*>(mem);
    // identity tables: request i of a call -> staging pages i * MBR + j
    std::vector<int> ids(max_reqs_per_call), bt((size_t)max_reqs_per_call * MBR);
    for (int i = 0; i < max_reqs_per_call; ++i) {
        ids[i] = i;
        for (int j = 0; j < MBR; ++j) bt[(size_t)i * MBR + j] = i * MBR + j;
    }
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess || cudaSetDevice(c.device) != cudaSuccess) return SEMIPD_ERR_CUDA;
    const bool okc = cudaMemcpy(base + L.ids, ids.data(), ids.size() * sizeof(int), cudaMemcpyHostToDevice) ==
                         cudaSuccess &&
                     cudaMemcpy(base + L.bt, bt.data(), bt.size() * sizeof(int), cudaMemcpyHostToDevice) ==
                         cudaSuccess;
    cudaSetDevice(prev);
    if (!okc) return SEMIPD_ERR_CUDA;
    // the bf16 prefill kernel's prefix page maps (as the bf16 pool's), over the staging pages
    const uint64_t pages = (uint64_t)max_reqs_per_call * MBR * c.num_kv_heads;
    const uint64_t kr = HD * 2;
    if (!spd_encode_tiled_3d(&pool->f8s_kmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base + L.k, HD, BS, pages, kr,
                             kr * BS, 64, BS, 1, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !spd_encode_tiled_3d(&pool->f8s_vmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, base + L.v, HD, BS, pages, kr,
                             kr * BS, 64, BS, 1, CU_TENSOR_MAP_SWIZZLE_128B))
        return SEMIPD_ERR_CUDA;
    pool->f8s = base;
    pool->f8s_cap = max_reqs_per_call;
    pool->have_f8s_maps = true;
    return SEMIPD_OK;
}

}  // extern "C"
