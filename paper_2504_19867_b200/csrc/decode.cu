// decode.cu — split-K paged decode attention (PagedAttention P:229, GQA P:355,
// flash-decoding split-K cited P:127) with the K/V append fused ("at each
// decode iteration, the KV cache of the request is updated").
//
// Persistent grid capped to the decode SM budget (P:195 x/y partition), dynamic
// work counter; a work unit is (request b, kv head g, split s).  Per CTA:
//   warp 3 (producer): fetches units, appends k_new/v_new for the unit
//     owning slot ctx, streams 64-key stages of K and V pages with TMA (128-B
//     swizzle, one 4-D box = min(bs,64) rows x all 128 columns of one (block, head)
//     page) into a 6-deep shared-memory ring (192 KiB: Little's law for HBM latency
//     on a minority of SMs);
//   consumer warps 0-2: global stage gs goes to warp gs % 3; QK^T and PV on
//     mma.sync m16n8k16 (the G <= 16 query heads of one kv head fill M = 16, so
//     each K/V byte is read once for all G heads), warp-shuffle online softmax in
//     the log2 domain, then a cross-warp merge in shared memory and, for split
//     units, a last-CTA-done merge over splits in split-index order.
// The decomposition depends on shapes only, so results are bitwise identical for
// every sm_budget and under co-run (S26).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

// L2 policy of the KV page stream: evict_first keeps the co-running prefill's
// reused chunk K/V tiles resident in L2 while decode streams the cache through it
#ifndef SPD_DEC_L2
#define SPD_DEC_L2 1
#endif
constexpr int kDecL2 = SPD_DEC_L2;

using namespace spd;

constexpr int HD = 128;           // head dim (dk == dv)
// SPD_DEC_CPASYNC = 1: 16-token pages streamed by the producer warp with 16-byte cp.async
// (LDGSTS) instead of one TMA box per 4 KiB (page, head).  Parity-green, but measured 9-10 %
// SLOWER at every SM budget (cfg-2 decode, bs 16: 3.58 vs 3.95 TB/s at 104 SMs, 4.46 vs 4.92 at
// 148; profiles/r2_decode_bs16_cpasync_ab.log): the 4 KiB TMA box is not what limits 16-token
// pages, so the default stays 0 (TMA).
// SPD_DEC_PF = D > 0: the producer also prefetches the boxes D stages ahead of the one it loads
// into L2 (cp.async.bulk.prefetch.tensor: no smem, no barrier), so the ring's own loads hit
// L2 and a slot is held for less than the HBM round trip.  Measured (profiles/r2_l2_prefetch_ab.log):
// D = 2 / 4 are 13-37 % SLOWER (bs 16: 3.96 -> 2.47 TB/s at 104 SMs; bs 64: 6.02 -> 5.20 at 89):
// a prefetch costs the SM's TMA engine as much as a load, and that engine is what bounds
// small pages.  Default 0.
#ifndef SPD_DEC_PF
#define SPD_DEC_PF 0
#endif
// SPD_DEC_PAIR16 = 1: 16-token pages with an even Hkv run the head-pair wide-box kernel
// (MODE 2): one 8 KiB TMA box per (block, head pair) and tensor
#ifndef SPD_DEC_PAIR16
#define SPD_DEC_PAIR16 1
#endif
#ifndef SPD_DEC_CPASYNC
#define SPD_DEC_CPASYNC 0
#endif
constexpr int KPS = 64;           // keys per stage
constexpr int NSTAGE = 6;
constexpr int KV_BYTES = KPS * HD * 2;         // 16 KiB of K (or V) per stage
constexpr int STAGE_BYTES = 2 * KV_BYTES;      // K + V
// SPD_DEC_SPLIT_KEYS: finer splits of the cfg-2 contexts (1024 / 2048 keys, with or without the
// head-pair wide boxes, SEMIPD_DECODE_PAIR64=1) are 10-70 % slower than whole-context units at
// 74-148 SMs (isolated, B 64 ctx 2048; profiles/r2_decode_split_pair_ab.log).  Default 4096.
#ifndef SPD_DEC_SPLIT_KEYS
#define SPD_DEC_SPLIT_KEYS 4096
#endif
constexpr int SPLIT_KEYS = SPD_DEC_SPLIT_KEYS;  // maximum keys per split (shape-only decomposition)
constexpr float LOG2E = 1.4426950408889634f;

struct UnitDesc {
    int b, g, s, S, k0, k1, base, nst;  // b < 0 : no more work
};

struct DecodeParams {
    const __nv_bfloat16* q;      // [B][Hq][128]
    const uint4* k_new;          // [B][Hkv][128] bf16
    const uint4* v_new;
    const int* req_ids;
    const int* ctx_lens;
    const int* bt;
    unsigned char* k_pool;       // layer base
    unsigned char* v_pool;
    __nv_bfloat16* out;
    float* ws_m;                 // [B][Hq][S_max]
    float* ws_l;
    float* ws_acc;               // [B][Hq][S_max][128]
    int* ws_cnt;                 // [B][Hkv]
    unsigned* sched;             // [2]: next unit, finished CTAs
    int* status;
    unsigned long long* span;  // semipd_set_spans record of this launch (or null)
    int skip_append;           // 1: the step's K/V rows are already in the pool (RoPE pre-pass)
    int B, Hq, Hkv, G, lg_bs, MBR, N_B, S_max, n_units, out_head_major;
    // TP head all-gather fused into the epilogue: every output vector is also
    // stored to each peer's gathered buffer (peer-mapped, already offset to this rank's shard)
    __nv_bfloat16* peers[SEMIPD_MAX_PEERS - 1];
    int n_peers;
    float scale_log2;
    SpdTrace trace;
    long long* tl;  // SPD_TIMELINE builds only: per-stage clock64 stamps of CTA 0
    int* tl_ctr;
};

// one bf16x4 output vector: local buffer, then every peer's gathered buffer (NVLink posted
// stores; the caller's "landed" handshake after the kernel publishes them)
__device__ __forceinline__ void store_out(const DecodeParams& p, size_t off, uint2 v) {
    *reinterpret_cast<uint2*>(p.out + off) = v;
#pragma unroll
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
        if (k < p.n_peers) *reinterpret_cast<uint2*>(p.peers[k] + off) = v;
}

#ifdef SPD_TIMELINE
#define TL_REC(a, b, c, d, e)                                                              \
    do {                                                                                   \
        if (p.tl && blockIdx.x == 0 && (b) < 2048) {                                       \
            long long* _r = p.tl + 8 * ((a) * 2048 + (b));                                 \
            _r[0] = a; _r[1] = b; _r[2] = c; _r[3] = d; _r[4] = e;                         \
        }                                                                                  \
    } while (0)
#define TL_NOW() clock64()
#else
#define TL_REC(a, b, c, d, e) do { } while (0)
#define TL_NOW() 0LL
#endif

__device__ __forceinline__ void split_range(int ctx, int S, int s, int& k0, int& k1) {
    const int nk = ctx + 1;
    int len = (nk + S - 1) / S;
    len = (len + KPS - 1) / KPS * KPS;
    k0 = s * len;
    k1 = min(nk, k0 + len);
}

// byte offset of (key, 64-column half h) inside a stage's K or V buffer:
// TMA box b (LG_R rows of one page, both halves) lands as [half][R rows][128 B]
template <int LG_R>
__device__ __forceinline__ uint32_t kv_off(int key, int h) {
    return ((uint32_t)(key >> LG_R) << (LG_R + 8)) + ((uint32_t)h << (LG_R + 7)) +
           ((uint32_t)(key & ((1 << LG_R) - 1)) << 7);
}

// offset of (key, 64-column half h) in a wide-box stage: MODE 0 / 1 as kv_off; MODE 2
// (16-token pages, one 8 KiB box = both heads' 16 rows): [box][head][half][16 rows][128 B],
// the head's own 4 KiB already added to the base
template <int MODE, int LG_R>
__device__ __forceinline__ uint32_t pair_off(int key, int h) {
    if constexpr (MODE == 2)
        return ((uint32_t)(key >> 4) << 13) + ((uint32_t)h << 11) + ((uint32_t)(key & 15) << 7);
    else
        return kv_off<LG_R>(key, h);
}

// SPD_DEC_KSPLIT = 1: separate barriers for a stage's K and V halves (see KS below).  Parity-
// green (62 decode / co-run tests) but measured SLOWER (isolated, bs 64: 3274 / 5437 / 6032 vs
// 3604 / 5702 / 6076 GB/s at 44 / 74 / 89 SMs; profiles/r2_decode_ksplit_ab.log): the one
// producer lane now blocks on the V slot of every stage after issuing its K, so the next
// stage's K goes out no earlier than before and the extra waits cost.  = 2 issues each V half
// after the next stage's K (no producer blocking): parity-green (62 tests), slower still (3068 /
// 5111 / 5864 GB/s at 44 / 74 / 89 SMs; profiles/r2_decode_ksplit_ab.log).  At 89 SMs the
// isolated kernel already streams 6.0 TB/s (0.92 of the copy peak): the ring is not what limits
// it there.  Default 0.
#ifndef SPD_DEC_KSPLIT
#define SPD_DEC_KSPLIT 0
#endif
template <int LG_R, bool SWAP>
__global__ void __launch_bounds__(4 * 32, 1)
    decode_bf16_kernel(const __grid_constant__ CUtensorMap kmap,
                       const __grid_constant__ CUtensorMap vmap, DecodeParams p) {
    constexpr int R = 1 << LG_R;     // rows per TMA box (= min(bs, 64))
    constexpr int NB = KPS / R;      // boxes per stage per tensor
    // 16-token pages: a 4 KiB (page, head) box costs the SM's TMA unit about as much as a
    // 16 KiB one, so the producer warp streams them with 16-byte cp.async (LDGSTS) instead,
    // into the same 128-B-swizzled stage layout, 32 lanes arriving on the stage barrier
    constexpr bool CPA = LG_R == 4 && SPD_DEC_CPASYNC;
    // KS: a stage's K and V halves have their own full / empty barriers, so a consumer hands
    // the K half back to the producer as soon as S is computed (before softmax and P V): one
    // more half-stage of loads in flight per held stage (SPD_DEC_KSPLIT, TMA path only)
    constexpr bool KS = SPD_DEC_KSPLIT && !CPA;
    // KS2 (SPD_DEC_KSPLIT = 2): the V half of stage i is issued after the K half of stage i + 1,
    // so the producer never blocks on a V slot before the next K goes out
    constexpr bool KS2 = KS && SPD_DEC_KSPLIT == 2;
    // consumer warps and scratch rows (the swap-AB partials have G <= 8 rows); 6 swap-AB
    // consumer warps measured 2-5 % slower than 3 (more padding stages and merge work)
    constexpr int CW = 3;
    constexpr int SR = SWAP ? 8 : 16;
    static_assert(NSTAGE % CW == 0, "each ring slot must have one fixed consumer warp");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ring = smem;                                   // NSTAGE x 32 KiB
    float* scr_acc = reinterpret_cast<float*>(ring + NSTAGE * STAGE_BYTES);  // [CW][16][128]
    float* scr_ml = scr_acc + CW * SR * HD;                       // [CW][16][2]
    uint64_t* full = reinterpret_cast<uint64_t*>(scr_ml + CW * SR * 2);
    uint64_t* empty = full + NSTAGE;
    uint64_t* fullV = KS ? empty + NSTAGE : full;   // V half (KS), else the stage barrier
    uint64_t* emptyV = KS ? fullV + NSTAGE : empty;
    uint64_t* ufull = KS ? emptyV + NSTAGE : empty + NSTAGE;
    uint64_t* uempty = ufull + 2;
    UnitDesc* units = reinterpret_cast<UnitDesc*>(uempty + 2);
    int* s_last = reinterpret_cast<int*>(units + 2);

    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    const uint64_t kv_pol = l2_policy(kDecL2);  // KV stream: read once per step
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(full + i, CPA ? 32 : 1);
            mbar_init(empty + i, 1);
            if (KS) {
                mbar_init(fullV + i, 1);
                mbar_init(emptyV + i, 1);
            }
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(ufull + i, 1);
            mbar_init(uempty + i, CW);
        }
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(2, (int)smid(), (int)blockIdx.x, 2 /* kernel kind: split-K decode */);
        }
    }
    __syncthreads();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (workspace, pool)
    if (threadIdx.x == 0) span_begin(p.span);

    // cross-warp merge of the consumer warps' partials (scratch rows = q heads of the group),
    // then the output (or the split partial and, by the last split, the split-order merge)
    auto merge_and_store = [&](const UnitDesc& d) {
        // ---- cross-warp merge: thread t handles (head h, 4 columns)
        const int tid = threadIdx.x;  // 0..127
        const bool split = d.S > 1;
        for (int idx = tid; idx < p.G * (HD / 4); idx += CW * 32) {
            const int h = idx / (HD / 4), c = (idx % (HD / 4)) * 4;
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < CW; ++w) M = fmaxf(M, scr_ml[(w * SR + h) * 2]);
            float L = 0.f;
            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                const float mw = scr_ml[(w * SR + h) * 2];
                const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
                L += f * scr_ml[(w * SR + h) * 2 + 1];
                const float4 a = *reinterpret_cast<const float4*>(scr_acc + (w * SR + h) * HD + c);
                o.x += f * a.x;
                o.y += f * a.y;
                o.z += f * a.z;
                o.w += f * a.w;
            }
            const int hq = d.g * p.G + h;
            if (!split) {
                const float inv = 1.f / L;
                const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                    : (((size_t)d.b * p.Hq + hq) * HD + c);
                uint2 v;
                v.x = pack_bf16(o.x * inv, o.y * inv);
                v.y = pack_bf16(o.z * inv, o.w * inv);
                store_out(p, off, v);
            } else {
                const size_t pi = ((size_t)d.b * p.Hq + hq) * p.S_max + d.s;
                *reinterpret_cast<float4*>(p.ws_acc + pi * HD + c) = o;
                if (c == 0) {
                    p.ws_m[pi] = M;
                    p.ws_l[pi] = L;
                }
            }
        }
        if (split) {
            __threadfence();
            named_bar_sync(1, CW * 32);
            if (tid == 0) {
                const int prev = atomicAdd(p.ws_cnt + d.b * p.Hkv + d.g, 1);
                *s_last = prev == d.S - 1;
            }
            named_bar_sync(1, CW * 32);
            if (*s_last) {
                __threadfence();
                // merge over splits in split-index order (flash-decoding)
                for (int idx = tid; idx < p.G * (HD / 4); idx += CW * 32) {
                    const int h = idx / (HD / 4), c = (idx % (HD / 4)) * 4;
                    const int hq = d.g * p.G + h;
                    const size_t pb = ((size_t)d.b * p.Hq + hq) * p.S_max;
                    float M = -INFINITY;
                    for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb + sI));
                    float L = 0.f;
                    float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int sI = 0; sI < d.S; ++sI) {
                        const float f = fast_exp2(__ldcg(p.ws_m + pb + sI) - M);
                        L += f * __ldcg(p.ws_l + pb + sI);
                        const float4 a = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + (pb + sI) * HD + c));
                        o.x += f * a.x;
                        o.y += f * a.y;
                        o.z += f * a.z;
                        o.w += f * a.w;
                    }
                    const float inv = 1.f / L;
                    const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                        : (((size_t)d.b * p.Hq + hq) * HD + c);
                    uint2 v;
                    v.x = pack_bf16(o.x * inv, o.y * inv);
                    v.y = pack_bf16(o.z * inv, o.w * inv);
                    store_out(p, off, v);
                }
                if (tid == 0) p.ws_cnt[d.b * p.Hkv + d.g] = 0;  // ready for the next call
            }
        }
        named_bar_sync(1, CW * 32);  // scratch reuse
    };
    if (warp == CW) {
        // =========================== producer ===========================
        // Whole warp: lane l holds the raw block id of box (32*batch + l) of the unit,
        // loaded one batch ahead (block-table reads off the TMA issue path); lane 0
        // issues one TMA per (page, tensor) per box; the K/V append uses 32 lanes.
        if (lane == 0) {
            tma_prefetch_desc(&kmap);
            tma_prefetch_desc(&vmap);
        }
        const int oob_z = p.N_B * p.Hkv;  // first page index past the tensor -> zero fill
        const int bs_mask = (1 << p.lg_bs) - 1;
        int gstage = 0, nunit = 0;
        // first unit of each CTA is static (blockIdx.x); later ones come from the counter,
        // fetched one unit ahead so the atomic's round trip overlaps the current unit
        // lane 0 holds the next unit index; the atomic's result is first read one unit later
        int u_next = blockIdx.x;
        // consecutive units are mostly the next kv head of the same (request, split): keep
        // the last request's metadata and first 64 block ids to skip the global round trips
        int prev_b = -1, prev_ctx = 0, prev_rid = 0, prev_k0 = -1, zc0 = -2, zn0 = -2;
        for (;;) {
            [[maybe_unused]] const long long tu0 = TL_NOW();
            const int u = __shfl_sync(0xffffffffu, u_next, 0);
            if (lane == 0) u_next = (int)gridDim.x + (int)atomicAdd(p.sched, 1u);
            UnitDesc d;
            int ctx = 0, rid = 0;
            if (u >= p.n_units) {
                d.b = -1;
            } else {
                // unit order: split-major, then request, then kv head
                d.s = u / (p.B * p.Hkv);
                d.b = (u / p.Hkv) % p.B;
                d.g = u % p.Hkv;
                if (d.b == prev_b) {
                    ctx = prev_ctx;
                    rid = prev_rid;
                } else {
                    ctx = __ldg(p.ctx_lens + d.b);
                    rid = __ldg(p.req_ids + d.b);
                }
                d.S = (ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
                if (d.s >= d.S) continue;  // warp-uniform
                split_range(ctx, d.S, d.s, d.k0, d.k1);
                d.nst = (d.k1 - d.k0 + KPS - 1) / KPS;
                // align the unit's first stage to a multiple of CW with data-less padding
                // stages, so the stage -> warp split depends on the unit only (bitwise
                // identical results for every grid size / schedule)
                while (gstage % CW != 0) {
                    const int st = gstage % NSTAGE;
                    if (lane == 0) mbar_wait(empty + st, ((gstage / NSTAGE) & 1) ^ 1);
                    __syncwarp();
                    if (CPA || lane == 0) mbar_arrive(full + st);
                    if (KS && lane == 0) {
                        mbar_wait(emptyV + st, ((gstage / NSTAGE) & 1) ^ 1);
                        mbar_arrive(fullV + st);
                    }
                    ++gstage;
                }
                __syncwarp();
                d.base = gstage;
            }
            const int us = nunit & 1;
            [[maybe_unused]] const long long tu1 = TL_NOW();
            if (lane == 0) {
                mbar_wait(uempty + us, ((nunit >> 1) & 1) ^ 1);
                units[us] = d;
                mbar_arrive(ufull + us);
            }
            __syncwarp();
            if (lane == 0) TL_REC(3, nunit, tu0, tu1, TL_NOW());
            ++nunit;
            if (d.b < 0) {  // no more units: the next kernel on the stream may be scheduled
                pdl_trigger();
                break;
            }
            const int* btr = p.bt + (size_t)rid * p.MBR;
            const int last_page = ctx >> p.lg_bs;
            // fused append of this step's K/V at slot ctx (last split only, bit-exact): the
            // rows are loaded now and stored right before the TMA of the stage holding slot
            // ctx (lanes 0-15 K, 16-31 V, 16 B each), then handed to the async proxy
            const bool append = d.s == d.S - 1 && !p.skip_append;
            const int app_stage = (ctx - d.k0) / KPS;
            uint4 app_v = make_uint4(0, 0, 0, 0);
            if (append) {
                const size_t src = ((size_t)d.b * p.Hkv + d.g) * (HD / 8);
                app_v = __ldg((lane < 16 ? p.k_new : p.v_new) + src + (lane & 15));
            }
            const int nbox = d.nst * NB;
            // raw block id for box bi (-2 = past the request's last page: zero fill, no error)
            auto lookup = [&](int bi) -> int {
                const int page = (d.k0 + bi * R) >> p.lg_bs;
                if (bi >= nbox || page > last_page) return -2;
                return page < p.MBR ? __ldg(btr + page) : -1;
            };
            int zc, zn;
            if (d.b == prev_b && d.k0 == prev_k0) {
                zc = zc0;
                zn = zn0;
            } else {
                zc = lookup(lane);
                zn = lookup(32 + lane);
            }
            prev_b = d.b;
            prev_ctx = ctx;
            prev_rid = rid;
            prev_k0 = d.k0;
            zc0 = zc;
            zn0 = zn;
            // KS2: the V half of the latest stage, issued after the next stage's K
            bool pv_ok = false;
            int pv_st = 0, pv_gs = 0, pv_y[NB], pv_z[NB];
            auto issue_v = [&]() {
                mbar_wait(emptyV + pv_st, ((pv_gs / NSTAGE) & 1) ^ 1);
                mbar_arrive_expect_tx(fullV + pv_st, KV_BYTES);
                unsigned char* vst_p = ring + pv_st * STAGE_BYTES + KV_BYTES;
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    tma_load_4d_hint(vst_p + b * (R * 256), &vmap, fullV + pv_st, 0, pv_y[b], 0, pv_z[b], kv_pol);
            };
            for (int i = 0; i < d.nst; ++i, ++gstage) {
                const int bb0 = i * NB;
                if (bb0 > 0 && (bb0 & 31) == 0) {
                    zc = zn;
                    zn = lookup(bb0 + 32 + lane);
                }
                const int st = gstage % NSTAGE;
                unsigned char* kst = ring + st * STAGE_BYTES;
                if (append && i == app_stage) {
                    const int blk = last_page < p.MBR ? __ldg(btr + last_page) : -1;
                    if (blk >= 0 && blk < p.N_B) {
                        const size_t slot = (((size_t)blk * p.Hkv + d.g) << p.lg_bs) + (ctx & bs_mask);
                        reinterpret_cast<uint4*>(lane < 16 ? p.k_pool : p.v_pool)[slot * (HD / 8) + (lane & 15)] = app_v;
                        fence_proxy_async_global();
                    }
                    __syncwarp();
                }
                [[maybe_unused]] long long tp0 = TL_NOW(), tp1 = 0;
                if (lane == 0) {
                    mbar_wait(empty + st, ((gstage / NSTAGE) & 1) ^ 1);
                    tp1 = TL_NOW();
                    if (!CPA) mbar_arrive_expect_tx(full + st, KS ? KV_BYTES : STAGE_BYTES);
                }
                if constexpr (CPA) {
                    // every lane copies 8 of the 256 16-byte chunks of each 4 KiB K and V page
                    // (consecutive lanes: consecutive 16 B of a row), swizzled as the TMA box
                    // would land: [half][16 rows][128 B], chunk cc of row r at cc ^ (r & 7)
                    __syncwarp();
                    const uint32_t kst_a = smem_u32(kst);
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const int blk = __shfl_sync(0xffffffffu, zc, (bb0 & 31) + b);
                        const bool ok = blk >= 0 && blk < p.N_B;
                        if (lane == 0 && !ok && blk != -2 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                        const size_t pg = ok ? ((size_t)blk * p.Hkv + d.g) * (R * 256) : 0;
                        const uint32_t nbytes = ok ? 16u : 0u;  // 0: zero fill
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int idx = lane + 32 * e;      // chunk of the page, 0..255
                            const int r = idx >> 4, c = idx & 15;
                            const uint32_t so = (uint32_t)(b * (R * 256) + (c >> 3) * (R * 128) + r * 128 +
                                                           (((c & 7) ^ (r & 7)) << 4));
                            const size_t go = pg + (size_t)(r * 256 + c * 16);
                            cp_async16_hint(kst_a + so, p.k_pool + go, nbytes, kv_pol);
                            cp_async16_hint(kst_a + KV_BYTES + so, p.v_pool + go, nbytes, kv_pol);
                        }
                    }
                    cp_async_mbar_arrive_noinc(full + st);
                } else {
                int zb[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const int blk = __shfl_sync(0xffffffffu, zc, (bb0 & 31) + b);
                    zb[b] = oob_z;
                    if (blk >= 0 && blk < p.N_B) zb[b] = blk * p.Hkv + d.g;
                    else if (lane == 0 && blk != -2 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                }
                if (lane == 0) {
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const int y = (d.k0 + i * KPS + b * R) & bs_mask;
                        tma_load_4d_hint(kst + b * (R * 256), &kmap, full + st, 0, y, 0, zb[b], kv_pol);
                        if (!KS)
                            tma_load_4d_hint(kst + KV_BYTES + b * (R * 256), &vmap, full + st, 0, y, 0, zb[b], kv_pol);
                    }
                    if (KS2) {  // the previous stage's V, then remember this one's
                        if (pv_ok) issue_v();
                        pv_ok = true;
                        pv_st = st;
                        pv_gs = gstage;
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            pv_y[b] = (d.k0 + i * KPS + b * R) & bs_mask;
                            pv_z[b] = zb[b];
                        }
                    } else if (KS) {  // the V half goes out once its own slot is free
                        mbar_wait(emptyV + st, ((gstage / NSTAGE) & 1) ^ 1);
                        mbar_arrive_expect_tx(fullV + st, KV_BYTES);
#pragma unroll
                        for (int b = 0; b < NB; ++b) {
                            const int y = (d.k0 + i * KPS + b * R) & bs_mask;
                            tma_load_4d_hint(kst + KV_BYTES + b * (R * 256), &vmap, fullV + st, 0, y, 0, zb[b], kv_pol);
                        }
                    }
                }
                if constexpr (SPD_DEC_PF > 0) {
                    // boxes SPD_DEC_PF stages ahead: in this 32-box batch (zc) or the next (zn)
#pragma unroll
                    for (int b = 0; b < NB; ++b) {
                        const int pbi = bb0 + SPD_DEC_PF * NB + b;
                        const int src = pbi - (bb0 & ~31);
                        const int v = __shfl_sync(0xffffffffu, src < 32 ? zc : zn, src & 31);
                        if (lane == 0 && pbi < nbox && src < 64 && v >= 0 && v < p.N_B) {
                            const int y = (d.k0 + i * KPS + SPD_DEC_PF * KPS + b * R) & bs_mask;
                            const int z = v * p.Hkv + d.g;
                            tma_prefetch_l2_4d(&kmap, 0, y, 0, z);
                            tma_prefetch_l2_4d(&vmap, 0, y, 0, z);
                        }
                    }
                }
                }
                if (lane == 0) TL_REC(1, gstage, tp0, tp1, TL_NOW());
                __syncwarp();
            }
            if (KS2 && lane == 0 && pv_ok) issue_v();  // the unit's last V
            __syncwarp();
        }
    } else if (SWAP) {
        // ================= consumers, swap-AB (G <= 8): heads are the MMA N =================
        // S^T[16 keys x 8 heads] = K . Q^T and O^T[16 dv x 8 heads] += V^T . P^T with
        // m16n8k16: half the MMAs of the q-heads-as-M form, which pads G <= 8 rows to 16.
        // The C fragment of S^T is turned into the B fragment of P^T by an 8x8 transpose.
        const int kr = lane >> 2;         // key (S^T) / dv (O^T) row within an 8-row block
        const int hc = (lane & 3) * 2;    // heads hc, hc + 1 of this thread's C values
        int nunit = 0;
        int next_gs = warp;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(ufull + us, (nunit >> 1) & 1);
            const UnitDesc d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(uempty + us);
            ++nunit;
            if (d.b < 0) break;
            // Q^T B fragments: head n = lane / 4, dims 16 kk + 2 (lane % 4) (+8)
            uint32_t qb[8][2];
            {
                const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q);
                const bool v = kr < p.G;
                const size_t row = ((size_t)d.b * p.Hq + d.g * p.G + kr) * (HD / 2);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int col = (kk * 16 + hc) >> 1;
                    qb[kk][0] = v ? __ldg(q32 + row + col) : 0u;
                    qb[kk][1] = v ? __ldg(q32 + row + col + 4) : 0u;
                }
            }
            float acc[8][4];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
            float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
            while (next_gs < d.base) {
                const int st = next_gs % NSTAGE;
                mbar_wait(full + st, (next_gs / NSTAGE) & 1);
                if (KS) mbar_wait(fullV + st, (next_gs / NSTAGE) & 1);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(empty + st);
                    if (KS) mbar_arrive(emptyV + st);
                }
                next_gs += CW;
            }
            next_gs = d.base + (warp < d.nst ? warp + ((d.nst - 1 - warp) / CW + 1) * CW : warp);
            const int lm = lane >> 3, lr = lane & 7;  // ldmatrix: matrix / row of this lane
            for (int i = warp; i < d.nst; i += CW) {
                const int gs = d.base + i;
                const int st = gs % NSTAGE;
                [[maybe_unused]] const long long tc0 = TL_NOW();
                mbar_wait(full + st, (gs / NSTAGE) & 1);
                [[maybe_unused]] const long long tc1 = TL_NOW();
                const uint32_t kst = smem_u32(ring + st * STAGE_BYTES);
                const uint32_t vst = kst + KV_BYTES;
                // ---- S^T: 4 key tiles x 8 k-steps; A = K rows (keys) via ldmatrix
                float s[4][4];
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    s[kt][0] = s[kt][1] = s[kt][2] = s[kt][3] = 0.f;
                    const int key = kt * 16 + (lm & 1) * 8 + lr;
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) {
                        const int ci = kk * 2 + (lm >> 1);  // 16-byte chunk (dims / 8)
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4(kst + kv_off<LG_R>(key, ci >> 3) + (((ci & 7) ^ (key & 7)) << 4), a0, a1,
                                a2, a3);
                        mma_bf16_16816(s[kt], a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
                    }
                }
                if (KS) {  // every K ldmatrix of this stage has retired: hand the K half back
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st);
                }
                // ---- mask + online softmax over keys, per head (log2 domain)
                const int kbase = d.k0 + i * KPS;
                const bool tail = kbase + KPS > d.k1;
                float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
                for (int kt = 0; kt < 4; ++kt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float x = s[kt][e] * p.scale_log2;
                        if (tail && kbase + kt * 16 + kr + (e >> 1) * 8 >= d.k1) x = -INFINITY;
                        s[kt][e] = x;
                        mx[e & 1] = fmaxf(mx[e & 1], x);
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
                    // C (key row, head cols) -> B (key k, head n): 8x8 transposes
                    pb[kt][0] = movmatrix_t(pack_bf16(p0, p1));
                    pb[kt][1] = movmatrix_t(pack_bf16(p2, p3));
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
                if (KS) mbar_wait(fullV + st, (gs / NSTAGE) & 1);
                // ---- O^T += V^T P^T: 8 dv tiles x 4 key steps; A = V^T via ldmatrix.trans
#pragma unroll
                for (int kt = 0; kt < 4; ++kt) {
                    const int key = kt * 16 + (lm >> 1) * 8 + lr;
#pragma unroll
                    for (int dt = 0; dt < 8; ++dt) {
                        const int ch = dt * 2 + (lm & 1);
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4_t(vst + kv_off<LG_R>(key, ch >> 3) + (((ch & 7) ^ (key & 7)) << 4), a0, a1,
                                  a2, a3);
                        mma_bf16_16816(acc[dt], a0, a1, a2, a3, pb[kt][0], pb[kt][1]);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(KS ? emptyV + st : empty + st);
                if (lane == 0) TL_REC(2, gs, tc0, tc1, TL_NOW());
            }
            // ---- per-warp partial -> shared scratch (rows = heads)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 4);
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 8);
                lrow[j] += __shfl_xor_sync(0xffffffffu, lrow[j], 16);
            }
            float* wacc = scr_acc + warp * SR * HD;
#pragma unroll
            for (int dt = 0; dt < 8; ++dt) {
                const int dv = dt * 16 + kr;
                wacc[hc * HD + dv] = acc[dt][0];
                wacc[(hc + 1) * HD + dv] = acc[dt][1];
                wacc[hc * HD + dv + 8] = acc[dt][2];
                wacc[(hc + 1) * HD + dv + 8] = acc[dt][3];
            }
            if (kr == 0) {
                scr_ml[(warp * SR + hc) * 2 + 0] = mrow[0];
                scr_ml[(warp * SR + hc) * 2 + 1] = lrow[0];
                scr_ml[(warp * SR + hc + 1) * 2 + 0] = mrow[1];
                scr_ml[(warp * SR + hc + 1) * 2 + 1] = lrow[1];
            }
            named_bar_sync(1, CW * 32);
            merge_and_store(d);
        }
    } else {
        // =========================== consumers ===========================
        const int r0 = lane >> 2;       // row (q head within group) of c0/c1
        const int c0 = (lane & 3) * 2;  // column pair
        int nunit = 0;
        int next_gs = warp;             // next global stage this warp must consume
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(ufull + us, (nunit >> 1) & 1);
            const UnitDesc d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(uempty + us);
            ++nunit;
            if (d.b < 0) break;
            // ---- Q fragments (rows >= G are zero)
            uint32_t qa[8][4];
            {
                const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q);
                const size_t rowA = ((size_t)d.b * p.Hq + d.g * p.G + r0) * (HD / 2);
                const size_t rowB = rowA + 8 * (HD / 2);
                const bool va = r0 < p.G, vb = r0 + 8 < p.G;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int col = (kk * 16 + c0) >> 1;
                    qa[kk][0] = va ? __ldg(q32 + rowA + col) : 0u;
                    qa[kk][1] = vb ? __ldg(q32 + rowB + col) : 0u;
                    qa[kk][2] = va ? __ldg(q32 + rowA + col + 4) : 0u;
                    qa[kk][3] = vb ? __ldg(q32 + rowB + col + 4) : 0u;
                }
            }
            float acc[16][4];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
            float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};

            // global stage gs goes to warp gs % CW, so every ring slot is consumed by one
            // warp in order (each full/empty phase is waited for exactly once); first
            // release the padding stages in front of this unit
            while (next_gs < d.base) {
                const int st = next_gs % NSTAGE;
                mbar_wait(full + st, (next_gs / NSTAGE) & 1);
                if (KS) mbar_wait(fullV + st, (next_gs / NSTAGE) & 1);
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(empty + st);
                    if (KS) mbar_arrive(emptyV + st);
                }
                next_gs += CW;
            }
            next_gs = d.base + (warp < d.nst ? warp + ((d.nst - 1 - warp) / CW + 1) * CW : warp);
            for (int i = warp; i < d.nst; i += CW) {
                const int gs = d.base + i;
                const int st = gs % NSTAGE;
                mbar_wait(full + st, (gs / NSTAGE) & 1);
                const uint32_t kst = smem_u32(ring + st * STAGE_BYTES);
                const uint32_t vst = kst + KV_BYTES;
                // ---- S = Q K^T : 8 n-tiles of 8 keys
                float s[8][4];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
                    const int key = nt * 8 + (lane & 7);
#pragma unroll
                    for (int kk = 0; kk < 8; kk += 2) {
                        const int ci = 2 * kk + (lane >> 3);
                        const uint32_t addr = kst + kv_off<LG_R>(key, ci >> 3) +
                                              (((ci & 7) ^ (key & 7)) << 4);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(addr, b0, b1, b2, b3);
                        mma_bf16_16816(s[nt], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                        mma_bf16_16816(s[nt], qa[kk + 1][0], qa[kk + 1][1], qa[kk + 1][2],
                                       qa[kk + 1][3], b2, b3);
                    }
                }
                if (KS) {  // every K ldmatrix of this stage has retired: hand the K half back
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st);
                }
                // ---- mask + online softmax (log2 domain); rows r0 (idx 0,1) and r0+8 (2,3)
                const int kbase = d.k0 + i * KPS;
                const bool tail = kbase + KPS > d.k1;
                float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        float x = s[nt][e] * p.scale_log2;
                        if (tail && kbase + nt * 8 + c0 + (e & 1) >= d.k1) x = -INFINITY;
                        s[nt][e] = x;
                        mx[e >> 1] = fmaxf(mx[e >> 1], x);
                    }
                float alpha[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 1));
                    mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 2));
                    const float mnew = fmaxf(mrow[h], mx[h]);
                    alpha[h] = fast_exp2(mrow[h] - mnew);  // exp2(-inf) = 0 on first stage
                    mrow[h] = mnew;
                }
                float ls[2] = {0.f, 0.f};
                uint32_t pa[4][4];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    const float p0 = fast_exp2(s[nt][0] - mrow[0]);
                    const float p1 = fast_exp2(s[nt][1] - mrow[0]);
                    const float p2 = fast_exp2(s[nt][2] - mrow[1]);
                    const float p3 = fast_exp2(s[nt][3] - mrow[1]);
                    ls[0] += p0 + p1;
                    ls[1] += p2 + p3;
                    const int ks = nt >> 1, hi = nt & 1;
                    pa[ks][hi * 2 + 0] = pack_bf16(p0, p1);
                    pa[ks][hi * 2 + 1] = pack_bf16(p2, p3);
                }
                lrow[0] = lrow[0] * alpha[0] + ls[0];
                lrow[1] = lrow[1] * alpha[1] + ls[1];
                if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
#pragma unroll
                    for (int nd = 0; nd < 16; ++nd) {
                        acc[nd][0] *= alpha[0];
                        acc[nd][1] *= alpha[0];
                        acc[nd][2] *= alpha[1];
                        acc[nd][3] *= alpha[1];
                    }
                }
                if (KS) mbar_wait(fullV + st, (gs / NSTAGE) & 1);
                // ---- O += P V : 16 dv n-tiles x 4 k-steps of 16 keys
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const int key = ks * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
                    for (int nd = 0; nd < 16; nd += 2) {
                        const int ch = nd + (lane >> 4);
                        const uint32_t addr = vst + kv_off<LG_R>(key, ch >> 3) +
                                              (((ch & 7) ^ (key & 7)) << 4);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4_t(addr, b0, b1, b2, b3);
                        mma_bf16_16816(acc[nd], pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3], b0, b1);
                        mma_bf16_16816(acc[nd + 1], pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3], b2, b3);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(KS ? emptyV + st : empty + st);
            }
            // ---- per-warp partial -> shared scratch
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 1);
                lrow[h] += __shfl_xor_sync(0xffffffffu, lrow[h], 2);
            }
            float* wacc = scr_acc + warp * SR * HD;
#pragma unroll
            for (int nd = 0; nd < 16; ++nd) {
                const int col = nd * 8 + c0;
                *reinterpret_cast<float2*>(wacc + r0 * HD + col) = make_float2(acc[nd][0], acc[nd][1]);
                *reinterpret_cast<float2*>(wacc + (r0 + 8) * HD + col) =
                    make_float2(acc[nd][2], acc[nd][3]);
            }
            if ((lane & 3) == 0) {
                scr_ml[(warp * SR + r0) * 2 + 0] = mrow[0];
                scr_ml[(warp * SR + r0) * 2 + 1] = lrow[0];
                scr_ml[(warp * SR + r0 + 8) * 2 + 0] = mrow[1];
                scr_ml[(warp * SR + r0 + 8) * 2 + 1] = lrow[1];
            }
            named_bar_sync(1, CW * 32);
            merge_and_store(d);
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

// ---------------------------------------------------------------------------------------
// Wide-box variants (G <= 8).  A TMA box costs ~800 cycles of its SM's TMA unit regardless of
// size up to ~24 KiB, so 16 KiB boxes cap an SM at ~20 B/clk.  Both variants
// move 32 KiB of K + 32 KiB of V per stage in two boxes, 3-deep ring, 3 warp pairs: stage gs
// goes to pair gs % 3 and warp 2p + e of the pair takes half e of the stage.
//   MODE 0 (64-token pages, even Hkv): unit = (request, kv heads g0 and g0 + 1, split); a box
//          covers the two adjacent (block, head) pages; half e = head g0 + e, 64 keys.
//   MODE 1 (128-token pages): unit = (request, kv head, split); a box is one whole page,
//          128 keys; half e = keys [64 e, 64 e + 64) of the stage.
// Per-warp math is decode_bf16_kernel's; partials of the 6 warps merge in smem.
constexpr int P_NCW = 3;                       // warp pairs (stage rotation)
constexpr int P_NSTAGE = 3;
constexpr int P_NTHREADS = (2 * P_NCW + 1) * 32;
constexpr int P_STAGE = 4 * KV_BYTES;          // K(g0) K(g0+1) V(g0) V(g0+1)
constexpr int P_GMAX = 8;

template <int MODE>
__global__ void __launch_bounds__(P_NTHREADS, 1)
    decode_pair_kernel(const __grid_constant__ CUtensorMap kmap2,
                       const __grid_constant__ CUtensorMap vmap2, DecodeParams p) {
    constexpr int LG_R = MODE == 0 ? 6 : MODE == 1 ? 7 : 4;  // rows per box (= per page)
    constexpr int KPS_M = MODE == 1 ? 128 : 64;               // keys per stage
    constexpr int NHU = MODE == 1 ? 1 : 2;                    // kv heads per unit
    constexpr int NBX = KPS_M >> LG_R;                        // boxes per stage per tensor
    constexpr bool PAIR = MODE != 1;                          // two heads per unit
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ring = smem;                                                     // 3 x 64 KiB
    float* scr_acc = reinterpret_cast<float*>(ring + P_NSTAGE * P_STAGE);          // [6][8][128]
    float* scr_ml = scr_acc + 2 * P_NCW * P_GMAX * HD;                             // [6][8][2]
    uint64_t* full = reinterpret_cast<uint64_t*>(scr_ml + 2 * P_NCW * P_GMAX * 2);
    uint64_t* empty = full + P_NSTAGE;
    uint64_t* ufull = empty + P_NSTAGE;
    uint64_t* uempty = ufull + 2;
    UnitDesc* units = reinterpret_cast<UnitDesc*>(uempty + 2);
    int* s_last = reinterpret_cast<int*>(units + 2);

    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    const uint64_t kv_pol = l2_policy(kDecL2);  // KV stream: read once per step
    const int NP = PAIR ? p.Hkv >> 1 : p.Hkv;  // head groups per request
    if (threadIdx.x == 0) {
        for (int i = 0; i < P_NSTAGE; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 2);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(ufull + i, 1);
            mbar_init(uempty + i, 2 * P_NCW);
        }
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(2, (int)smid(), (int)blockIdx.x, 6 + MODE /* kernel kind: wide-box split-K decode */);
        }
    }
    __syncthreads();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (workspace, pool)
    if (threadIdx.x == 0) span_begin(p.span);

    if (warp == 2 * P_NCW) {
        // =========================== producer ===========================
        if (lane == 0) {
            tma_prefetch_desc(&kmap2);
            tma_prefetch_desc(&vmap2);
        }
        const int oob_z = p.N_B * p.Hkv;
        const int bs_mask = (1 << p.lg_bs) - 1;
        int gstage = 0, nunit = 0;
        for (;;) {
            int u = 0;
            if (lane == 0) u = (int)atomicAdd(p.sched, 1u);
            u = __shfl_sync(0xffffffffu, u, 0);
            UnitDesc d;
            if (u >= p.n_units) {
                d.b = -1;
            } else {
                d.s = u / (p.B * NP);
                d.b = (u / NP) % p.B;
                d.g = NHU * (u % NP);  // first head of the unit
                const int ctx = __ldg(p.ctx_lens + d.b);
                d.S = (ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
                if (d.s >= d.S) continue;
                {
                    const int nk = ctx + 1;
                    int len = (nk + d.S - 1) / d.S;
                    len = (len + KPS_M - 1) / KPS_M * KPS_M;
                    d.k0 = d.s * len;
                    d.k1 = min(nk, d.k0 + len);
                }
                d.nst = (d.k1 - d.k0 + KPS_M - 1) / KPS_M;
                while (gstage % P_NCW != 0) {  // align to the pair rotation (R26)
                    if (lane == 0) {
                        const int st = gstage % P_NSTAGE;
                        mbar_wait(empty + st, ((gstage / P_NSTAGE) & 1) ^ 1);
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
            const int ctx = __ldg(p.ctx_lens + d.b);
            const int* btr = p.bt + (size_t)__ldg(p.req_ids + d.b) * p.MBR;
            const int last_page = ctx >> p.lg_bs;
            if (d.s == d.S - 1 && !p.skip_append) {
                // fused append of the unit's heads' K and V rows at slot ctx (16 B per lane per
                // copy; MODE 0: lanes 16-31 take the second head, MODE 1: they take V)
                const int blk = last_page < p.MBR ? __ldg(btr + last_page) : -1;
                if (blk >= 0 && blk < p.N_B) {
                    const int c = lane & 15, e = lane >> 4;
                    if (PAIR) {
                        const size_t slot = (((size_t)blk * p.Hkv + d.g + e) << p.lg_bs) + (ctx & bs_mask);
                        const size_t src = ((size_t)d.b * p.Hkv + d.g + e) * (HD / 8);
                        reinterpret_cast<uint4*>(p.k_pool)[slot * (HD / 8) + c] = __ldg(p.k_new + src + c);
                        reinterpret_cast<uint4*>(p.v_pool)[slot * (HD / 8) + c] = __ldg(p.v_new + src + c);
                    } else {
                        const size_t slot = (((size_t)blk * p.Hkv + d.g) << p.lg_bs) + (ctx & bs_mask);
                        const size_t src = ((size_t)d.b * p.Hkv + d.g) * (HD / 8);
                        unsigned char* pool = e ? p.v_pool : p.k_pool;
                        const uint4* nw = e ? p.v_new : p.k_new;
                        reinterpret_cast<uint4*>(pool)[slot * (HD / 8) + c] = __ldg(nw + src + c);
                    }
                    fence_proxy_async_global();
                }
                __syncwarp();
            }
            // raw block id of box bi (NBX boxes per stage; -2: past the request)
            const int nbox = d.nst * NBX;
            auto lookup = [&](int bi) -> int {
                const int page = (d.k0 + bi * (KPS_M / NBX)) >> p.lg_bs;
                if (bi >= nbox || page > last_page) return -2;
                return page < p.MBR ? __ldg(btr + page) : -1;
            };
            int zc = lookup(lane);
            for (int i = 0; i < d.nst; ++i, ++gstage) {
                const int st = gstage % P_NSTAGE;
                if (lane == 0) {
                    mbar_wait(empty + st, ((gstage / P_NSTAGE) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + st, P_STAGE);
                }
#pragma unroll
                for (int b = 0; b < NBX; ++b) {
                    const int bi = i * NBX + b;
                    if (bi > 0 && (bi & 31) == 0) zc = lookup(bi + lane);
                    const int blk = __shfl_sync(0xffffffffu, zc, bi & 31);
                    if (lane == 0) {
                        unsigned char* kst = ring + st * P_STAGE + b * (KV_BYTES * 2 / NBX);
                        int z = oob_z;
                        if (blk >= 0 && blk < p.N_B) z = blk * p.Hkv + d.g;
                        else if (blk != -2 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                        const int y = (d.k0 + bi * (KPS_M / NBX)) & bs_mask;
                        tma_load_4d_hint(kst, &kmap2, full + st, 0, y, 0, z, kv_pol);
                        tma_load_4d_hint(kst + 2 * KV_BYTES, &vmap2, full + st, 0, y, 0, z, kv_pol);
                    }
                }
                __syncwarp();
            }
        }
    } else {
        // =========================== consumers ===========================
        const int pw = warp >> 1, e = warp & 1;  // pair (stage rotation), head of the pair
        const int r0 = lane >> 2;
        const int c0 = (lane & 3) * 2;
        int nunit = 0;
        int next_gs = pw;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(ufull + us, (nunit >> 1) & 1);
            const UnitDesc d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(uempty + us);
            ++nunit;
            if (d.b < 0) break;
            const int g = d.g + (PAIR ? e : 0);
            uint32_t qa[8][4];
            {
                const uint32_t* q32 = reinterpret_cast<const uint32_t*>(p.q);
                const size_t rowA = ((size_t)d.b * p.Hq + g * p.G + r0) * (HD / 2);
                const bool va = r0 < p.G;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int col = (kk * 16 + c0) >> 1;
                    qa[kk][0] = va ? __ldg(q32 + rowA + col) : 0u;
                    qa[kk][1] = 0u;  // rows 8-15: G <= 8
                    qa[kk][2] = va ? __ldg(q32 + rowA + col + 4) : 0u;
                    qa[kk][3] = 0u;
                }
            }
            float acc[16][2];
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[i][0] = acc[i][1] = 0.f;
            float mrow = -INFINITY, lrow = 0.f;
            while (next_gs < d.base) {
                const int st = next_gs % P_NSTAGE;
                mbar_wait(full + st, (next_gs / P_NSTAGE) & 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
                next_gs += P_NCW;
            }
            next_gs = d.base + (pw < d.nst ? pw + ((d.nst - 1 - pw) / P_NCW + 1) * P_NCW : pw);
            for (int i = pw; i < d.nst; i += P_NCW) {
                const int gs = d.base + i;
                const int st = gs % P_NSTAGE;
                mbar_wait(full + st, (gs / P_NSTAGE) & 1);
                // MODE 0: [K g0 | K g0+1 | V g0 | V g0+1], 64-row pages; MODE 1: [K | V], one
                // 128-row page each ([half][128 rows][128 B]); this warp's keys start at koff
                // MODE 2: [box b][head e][half][16 rows][128 B] (8 KiB per box), K then V
                const uint32_t kst = smem_u32(ring + st * P_STAGE) +
                                     (MODE == 0 ? e * KV_BYTES : MODE == 2 ? e * 4096 : 0);
                const uint32_t vst = kst + 2 * KV_BYTES;
                const int koff = MODE == 1 ? 64 * e : 0;
                float s[8][4];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    s[nt][0] = s[nt][1] = s[nt][2] = s[nt][3] = 0.f;
                    const int key = koff + nt * 8 + (lane & 7);
#pragma unroll
                    for (int kk = 0; kk < 8; kk += 2) {
                        const int ci = 2 * kk + (lane >> 3);
                        const uint32_t addr = kst + pair_off<MODE, LG_R>(key, ci >> 3) + (((ci & 7) ^ (key & 7)) << 4);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4(addr, b0, b1, b2, b3);
                        mma_bf16_16816(s[nt], qa[kk][0], qa[kk][1], qa[kk][2], qa[kk][3], b0, b1);
                        mma_bf16_16816(s[nt], qa[kk + 1][0], qa[kk + 1][1], qa[kk + 1][2],
                                       qa[kk + 1][3], b2, b3);
                    }
                }
                const int kbase = d.k0 + i * KPS_M + koff;
                const bool tail = kbase + KPS > d.k1;
                float mx = -INFINITY;
#pragma unroll
                for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                    for (int q2 = 0; q2 < 2; ++q2) {  // rows r0 only (rows >= 8 are padding)
                        float x = s[nt][q2] * p.scale_log2;
                        if (tail && kbase + nt * 8 + c0 + q2 >= d.k1) x = -INFINITY;
                        s[nt][q2] = x;
                        mx = fmaxf(mx, x);
                    }
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
                if (MODE == 1 && mx == -INFINITY) {  // this half lies past the unit's last key
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + st);
                    continue;
                }
                const float mnew = fmaxf(mrow, mx);
                const float alpha = fast_exp2(mrow - mnew);
                mrow = mnew;
                float ls = 0.f;
                uint32_t pa[4][4];
#pragma unroll
                for (int nt = 0; nt < 8; ++nt) {
                    const float p0 = fast_exp2(s[nt][0] - mrow);
                    const float p1 = fast_exp2(s[nt][1] - mrow);
                    ls += p0 + p1;
                    const int ks = nt >> 1, hi = nt & 1;
                    pa[ks][hi * 2 + 0] = pack_bf16(p0, p1);
                    pa[ks][hi * 2 + 1] = 0u;
                }
                lrow = lrow * alpha + ls;
                if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
                    for (int nd = 0; nd < 16; ++nd) {
                        acc[nd][0] *= alpha;
                        acc[nd][1] *= alpha;
                    }
                }
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const int key = koff + ks * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
                    for (int nd = 0; nd < 16; nd += 2) {
                        const int ch = nd + (lane >> 4);
                        const uint32_t addr = vst + pair_off<MODE, LG_R>(key, ch >> 3) + (((ch & 7) ^ (key & 7)) << 4);
                        uint32_t b0, b1, b2, b3;
                        ldsm_x4_t(addr, b0, b1, b2, b3);
                        float t0[4] = {acc[nd][0], acc[nd][1], 0.f, 0.f};
                        float t1[4] = {acc[nd + 1][0], acc[nd + 1][1], 0.f, 0.f};
                        mma_bf16_16816(t0, pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3], b0, b1);
                        mma_bf16_16816(t1, pa[ks][0], pa[ks][1], pa[ks][2], pa[ks][3], b2, b3);
                        acc[nd][0] = t0[0];
                        acc[nd][1] = t0[1];
                        acc[nd + 1][0] = t1[0];
                        acc[nd + 1][1] = t1[1];
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + st);
            }
            lrow += __shfl_xor_sync(0xffffffffu, lrow, 1);
            lrow += __shfl_xor_sync(0xffffffffu, lrow, 2);
            const int wi = pw * 2 + e;  // scratch slot of this warp
            float* wacc = scr_acc + wi * P_GMAX * HD;
            if (r0 < P_GMAX) {
#pragma unroll
                for (int nd = 0; nd < 16; ++nd)
                    *reinterpret_cast<float2*>(wacc + r0 * HD + nd * 8 + c0) = make_float2(acc[nd][0], acc[nd][1]);
                if ((lane & 3) == 0) {
                    scr_ml[(wi * P_GMAX + r0) * 2 + 0] = mrow;
                    scr_ml[(wi * P_GMAX + r0) * 2 + 1] = lrow;
                }
            }
            named_bar_sync(1, 2 * P_NCW * 32);
            // cross-warp merge: thread t handles (head e of the pair, q head h, 4 columns)
            const int tid = threadIdx.x;  // 0..191
            const bool split = d.S > 1;
            constexpr int WPH = 2 * P_NCW / NHU;  // warps per head
            for (int idx = tid; idx < NHU * p.G * (HD / 4); idx += 2 * P_NCW * 32) {
                const int ee = idx / (p.G * (HD / 4));
                const int h = (idx / (HD / 4)) % p.G, c = (idx % (HD / 4)) * 4;
                float M = -INFINITY;
#pragma unroll
                for (int w = 0; w < WPH; ++w)
                    M = fmaxf(M, scr_ml[(((PAIR ? w * 2 + ee : w)) * P_GMAX + h) * 2]);
                float L = 0.f;
                float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int w = 0; w < WPH; ++w) {
                    const int wj = PAIR ? w * 2 + ee : w;
                    const float mw = scr_ml[(wj * P_GMAX + h) * 2];
                    const float f = mw == -INFINITY ? 0.f : fast_exp2(mw - M);
                    L += f * scr_ml[(wj * P_GMAX + h) * 2 + 1];
                    const float4 a = *reinterpret_cast<const float4*>(scr_acc + (wj * P_GMAX + h) * HD + c);
                    o.x += f * a.x;
                    o.y += f * a.y;
                    o.z += f * a.z;
                    o.w += f * a.w;
                }
                const int hq = (d.g + ee) * p.G + h;
                if (!split) {
                    const float inv = 1.f / L;
                    const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                        : (((size_t)d.b * p.Hq + hq) * HD + c);
                    uint2 v;
                    v.x = pack_bf16(o.x * inv, o.y * inv);
                    v.y = pack_bf16(o.z * inv, o.w * inv);
                    store_out(p, off, v);
                } else {
                    const size_t pi = ((size_t)d.b * p.Hq + hq) * p.S_max + d.s;
                    *reinterpret_cast<float4*>(p.ws_acc + pi * HD + c) = o;
                    if (c == 0) {
                        p.ws_m[pi] = M;
                        p.ws_l[pi] = L;
                    }
                }
            }
            if (split) {
                __threadfence();
                named_bar_sync(1, 2 * P_NCW * 32);
                if (tid == 0) *s_last = atomicAdd(p.ws_cnt + d.b * p.Hkv + d.g, 1) == d.S - 1;
                named_bar_sync(1, 2 * P_NCW * 32);
                if (*s_last) {
                    __threadfence();
                    for (int idx = tid; idx < NHU * p.G * (HD / 4); idx += 2 * P_NCW * 32) {
                        const int ee = idx / (p.G * (HD / 4));
                        const int h = (idx / (HD / 4)) % p.G, c = (idx % (HD / 4)) * 4;
                        const int hq = (d.g + ee) * p.G + h;
                        const size_t pb = ((size_t)d.b * p.Hq + hq) * p.S_max;
                        float M = -INFINITY;
                        for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb + sI));
                        float L = 0.f;
                        float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int sI = 0; sI < d.S; ++sI) {
                            const float f = fast_exp2(__ldcg(p.ws_m + pb + sI) - M);
                            L += f * __ldcg(p.ws_l + pb + sI);
                            const float4 a = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + (pb + sI) * HD + c));
                            o.x += f * a.x;
                            o.y += f * a.y;
                            o.z += f * a.z;
                            o.w += f * a.w;
                        }
                        const float inv = 1.f / L;
                        const size_t off = p.out_head_major ? (((size_t)hq * p.B + d.b) * HD + c)
                                                            : (((size_t)d.b * p.Hq + hq) * HD + c);
                        uint2 v;
                        v.x = pack_bf16(o.x * inv, o.y * inv);
                        v.y = pack_bf16(o.z * inv, o.w * inv);
                        store_out(p, off, v);
                    }
                    if (tid == 0) p.ws_cnt[d.b * p.Hkv + d.g] = 0;
                }
            }
            named_bar_sync(1, 2 * P_NCW * 32);
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

size_t decode_pair_smem_bytes() {
    return 1024 + P_NSTAGE * P_STAGE + 2 * P_NCW * P_GMAX * HD * 4 + 2 * P_NCW * P_GMAX * 2 * 4 +
           (2 * P_NSTAGE + 4) * 8 + 2 * sizeof(UnitDesc) + 16;
}

size_t decode_smem_bytes(bool swap) {
    const int cw = 3, sr = swap ? 8 : 16;
    return 1024 + NSTAGE * STAGE_BYTES + cw * sr * HD * 4 + cw * sr * 2 * 4 +
           (4 * NSTAGE + 4) * 8 + 2 * sizeof(UnitDesc) + 16;  // (K, V) full / empty + unit barriers
}

bool fast_path_ok(const semipd_pool* p, int Hq) {
    const auto& c = p->cfg;
    const int bs = c.block_size;
    return c.dtype == SEMIPD_BF16 && !c.kv_shared && c.head_dim_k == HD && c.head_dim_v == HD &&
           p->have_dmaps && Hq % c.num_kv_heads == 0 && Hq / c.num_kv_heads <= 16 &&
           (bs == 16 || bs == 32 || bs == 64 || bs == 128);
}

}  // namespace

extern "C" {

size_t semipd_decode_workspace_bytes(semipd_pool_t pool, int32_t max_batch, int32_t num_q_heads,
                                     int32_t max_ctx) {
    if (!pool || max_batch < 0 || num_q_heads <= 0 || max_ctx < 0) return 0;
    // SpdWs: counters for max_batch x Hkv at the front + the largest split-partial set of any
    // decode kernel / batch <= max_batch at the back
    int S_max = (max_ctx + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
    if (pool->cfg.dtype == SEMIPD_FP8_E4M3) S_max *= spd_fp8_pieces();  // FP8: split pieces
    size_t part = spd_ws_partial_bytes((size_t)max_batch * num_q_heads, S_max, pool->cfg.head_dim_v);
    if (pool->cfg.kv_shared) {
        const size_t m = spd_mla_ws_bytes(max_batch, max_ctx);
        const size_t m2 = spd_mla_tc_ws_bytes(max_batch, max_ctx);
        if (m > part) part = m;
        if (m2 > part) part = m2;
    }
    const int hkv = pool->cfg.num_kv_heads > 0 ? pool->cfg.num_kv_heads : 1;
    return spd_ws_counter_bytes((size_t)max_batch * hkv) + part;
}

semipd_status semipd_decode_attn(semipd_pool_t pool, int32_t layer, const void* q,
                                 const void* k_new, const void* v_new, const int32_t* req_ids,
                                 const int32_t* ctx_lens, int32_t batch, int32_t max_ctx_len,
                                 int32_t num_q_heads, float softmax_scale, void* out,
                                 int32_t out_head_major, void* workspace, size_t ws_bytes,
                                 int32_t sm_budget, int32_t* status_dev, semipd_stream_t s) {
    if (!pool || layer < 0 || layer >= pool->cfg.num_layers || batch < 0 || max_ctx_len < 0)
        return SEMIPD_ERR_INVALID;
    const auto& c = pool->cfg;
    if (num_q_heads <= 0 || num_q_heads % c.num_kv_heads) return SEMIPD_ERR_INVALID;
    if (sm_budget < -1 || sm_budget > pool->num_sms) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (status_dev && cudaMemsetAsync(status_dev, 0, sizeof(int), st) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    if (batch == 0) return SEMIPD_OK;
    if (!q || !k_new || (!v_new && !c.kv_shared) || !req_ids || !ctx_lens || !out)
        return SEMIPD_ERR_INVALID;
    const int budget = spd_resolve_budget(pool, sm_budget, false);
    // the split-K kernels (bf16 and E4M3 pages) support peers
    const bool f8_pool = c.dtype == SEMIPD_FP8_E4M3;
    if (pool->dec_n_peers > 0 && (!out_head_major || (!f8_pool && !fast_path_ok(pool, num_q_heads)) ||
                                  spd_mla_tc_ok(pool, num_q_heads) ||
                                  spd_mla_decode_ok(pool, num_q_heads)))
        return pool->dec_n_peers > 0 && !out_head_major ? SEMIPD_ERR_INVALID : SEMIPD_ERR_UNSUPPORTED;
    // the peer offsets were fixed for the gathered buffers' batch: any other batch would store
    // at wrong head / token positions or past a peer's buffer
    if (pool->dec_n_peers > 0 && batch != pool->dec_peer_tokens) return SEMIPD_ERR_INVALID;
    if (f8_pool) {  // E4M3 pages (reading R31): quantised append + decode
        if (pool->rope_on) {
            // RoPE of q / k_new in place at ctx, fused with the quantised append of the rotated
            // rows (R28 + R31); the FP8 kernel skips its own append
            semipd_status r = spd_launch_rope_write(pool, layer, const_cast<void*>(q),
                                                    const_cast<void*>(k_new), v_new, nullptr, req_ids,
                                                    ctx_lens, batch, batch, num_q_heads, status_dev, st);
            if (r != SEMIPD_OK) return r;
        }
        return spd_launch_decode_fp8(pool, layer, q, k_new, v_new, req_ids, ctx_lens, batch,
                                     max_ctx_len, num_q_heads, softmax_scale, out, out_head_major,
                                     workspace, ws_bytes, budget, status_dev, st);
    }
    if (pool->rope_on) {
        // RoPE of q / k_new (in place) at position ctx, fused with the append of the rotated
        // rows (R28): the attention kernels below skip their own append
        semipd_status r = spd_launch_rope_write(pool, layer, const_cast<void*>(q),
                                                const_cast<void*>(k_new), v_new, nullptr, req_ids,
                                                ctx_lens, batch, batch, num_q_heads, status_dev, st);
        if (r != SEMIPD_OK) return r;
    }
    if (spd_mla_tc_ok(pool, num_q_heads))  // absorbed MLA latent cache, 64-token pages (cfg 5)
        return spd_launch_decode_mla_tc(pool, layer, q, k_new, req_ids, ctx_lens, batch,
                                        max_ctx_len, num_q_heads, softmax_scale, out,
                                        out_head_major, workspace, ws_bytes, budget, status_dev, st);
    if (spd_mla_decode_ok(pool, num_q_heads))  // latent cache with 32/128-token pages
        return spd_launch_decode_mla(pool, layer, q, k_new, req_ids, ctx_lens, batch, max_ctx_len,
                                     num_q_heads, softmax_scale, out, out_head_major, workspace,
                                     ws_bytes, budget, status_dev, st);
    if (!fast_path_ok(pool, num_q_heads)) {
        // generic CUDA-core path: append, then attention (same stream)
        if (!pool->rope_on) {
            semipd_status r = spd_launch_kv_write(pool, layer, k_new, v_new, nullptr, req_ids,
                                                  ctx_lens, batch, batch, 1, status_dev, st);
            if (r != SEMIPD_OK) return r;
        }
        return spd_launch_simt_attn(pool, layer, q, nullptr, req_ids, ctx_lens, batch, batch, 1,
                                    num_q_heads, softmax_scale, out, out_head_major, budget,
                                    status_dev, st);
    }
    const int S_max = (max_ctx_len + 1 + SPLIT_KEYS - 1) / SPLIT_KEYS;
    SpdWs w;
    if (!spd_ws_carve(workspace, ws_bytes, (size_t)batch * c.num_kv_heads, (size_t)batch * num_q_heads,
                      S_max, HD, &w))
        return SEMIPD_ERR_INVALID;
    DecodeParams prm;
    prm.q = static_cast<const __nv_bfloat16*>(q);
    prm.k_new = static_cast<const uint4*>(k_new);
    prm.v_new = static_cast<const uint4*>(v_new);
    prm.req_ids = req_ids;
    prm.ctx_lens = ctx_lens;
    prm.bt = pool->bt;
    prm.k_pool = static_cast<unsigned char*>(pool->k_layer(layer));
    prm.v_pool = static_cast<unsigned char*>(pool->v_layer(layer));
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
    prm.Hq = num_q_heads;
    prm.Hkv = c.num_kv_heads;
    prm.G = num_q_heads / c.num_kv_heads;
    prm.lg_bs = __builtin_ctz((unsigned)c.block_size);
    prm.MBR = c.max_blocks_per_req;
    prm.N_B = c.num_blocks;
    prm.S_max = S_max;
    prm.n_units = batch * c.num_kv_heads * S_max;
    prm.out_head_major = out_head_major;
    prm.n_peers = pool->dec_n_peers;
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
        prm.peers[k] = k < pool->dec_n_peers ? static_cast<__nv_bfloat16*>(pool->dec_peers[k]) : nullptr;
    prm.scale_log2 = softmax_scale * LOG2E;
    prm.trace = spd_trace(pool);
    prm.tl = reinterpret_cast<long long*>(pool->timeline);
    prm.tl_ctr = pool->timeline_ctr;
    // wide-box kernels (G <= 8): 128-token pages always (MODE 1, one whole page per box);
    // 64-token pages with even Hkv only when the batch alone gives >= 2 x 148 head-pair
    // units (MODE 0: with fewer, the coarser units cost more in grid-tail imbalance than the
    // bigger boxes gain).  Shape-only rules, so the kernel choice never depends on the SM
    // budget (R26).
    const bool mode1 = pool->have_wide_maps && c.block_size == 128 && prm.G <= P_GMAX;
    const bool mode0 = pool->have_wide_maps && c.block_size == 64 && prm.G <= P_GMAX &&
                       c.num_kv_heads % 2 == 0 &&
                       (batch * (c.num_kv_heads / 2) >= 2 * 148 || pool->force_pair);
    // 16-token pages, even Hkv (SPD_DEC_PAIR16): one 8 KiB box carries both heads of a
    // (block, head-pair), half the TMA operations of the one-head kernel's 4 KiB boxes
    const bool mode2 = SPD_DEC_PAIR16 && pool->have_wide_maps && c.block_size == 16 &&
                       prm.G <= P_GMAX && c.num_kv_heads % 2 == 0;
    if ((mode0 || mode1 || mode2) && !pool->force_single) {
        prm.n_units = batch * (mode1 ? c.num_kv_heads : c.num_kv_heads / 2) * S_max;
        const size_t smem = decode_pair_smem_bytes();
        static bool attr_pair[3] = {false, false, false};
        const int mi = mode0 ? 0 : mode1 ? 1 : 2;
        auto kern = mode0 ? decode_pair_kernel<0> : mode1 ? decode_pair_kernel<1> : decode_pair_kernel<2>;
        if (!attr_pair[mi]) {
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
                cudaSuccess)
                return SEMIPD_ERR_CUDA;
            attr_pair[mi] = true;
        }
        int grid = budget > 0 ? budget : prm.n_units;
        if (grid > prm.n_units) grid = prm.n_units;
        if (spd_launch_pdl(kern, dim3(grid), dim3(P_NTHREADS), smem, st, pool->dkmap2[layer], pool->dvmap2[layer],
                           prm) != cudaSuccess ||
            cudaGetLastError() != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        pool->launches += 1;
        return SEMIPD_OK;
    }
    const bool swap = prm.G <= 8;  // heads fit the MMA N = 8: swap-AB consumers
    const size_t smem = decode_smem_bytes(swap);
    const int nthreads = 4 * 32;
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    const int lg_r = __builtin_ctz((unsigned)pool->dbox_rows);
    cudaError_t e = cudaSuccess;
    auto launch = [&](auto kern) {
        static bool attr_set[6] = {false, false, false, false, false, false};
        const int ai = (lg_r - 4) * 2 + (prm.G <= 8);
        if (!attr_set[ai]) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return;
            attr_set[ai] = true;
        }
        e = spd_launch_pdl(kern, dim3(grid), dim3(nthreads), smem, st, pool->dkmap[layer], pool->dvmap[layer], prm);
        if (e == cudaSuccess) e = cudaGetLastError();
    };
    if (lg_r == 4) swap ? launch(decode_bf16_kernel<4, true>) : launch(decode_bf16_kernel<4, false>);
    else if (lg_r == 5) swap ? launch(decode_bf16_kernel<5, true>) : launch(decode_bf16_kernel<5, false>);
    else swap ? launch(decode_bf16_kernel<6, true>) : launch(decode_bf16_kernel<6, false>);
    if (e != cudaSuccess) return SEMIPD_ERR_CUDA;
    pool->launches += 1;
    return SEMIPD_OK;
}

semipd_status semipd_set_decode_peers(semipd_pool_t pool, void* const* peer_out, int32_t n,
                                      int32_t tokens) {
    if (!pool || n < 0 || n > SEMIPD_MAX_PEERS - 1 || (n > 0 && (!peer_out || tokens <= 0)))
        return SEMIPD_ERR_INVALID;
    for (int k = 0; k < n; ++k)
        if (!peer_out[k] || reinterpret_cast<uintptr_t>(peer_out[k]) % 8) return SEMIPD_ERR_INVALID;
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k) pool->dec_peers[k] = k < n ? peer_out[k] : nullptr;
    pool->dec_n_peers = n;
    pool->dec_peer_tokens = n > 0 ? tokens : 0;
    return SEMIPD_OK;
}

}  // extern "C"
