// decode_mla_tc.cu — absorbed-MLA decode attention on the 5th-gen tensor cores (cfg 5:
// 16 q heads share ONE latent KV head, dk = 576 (512 latent + 64 rope), dv = 512,
// V = K[..., :512]; R19).  Same hot-path contract as decode.cu: fused append of
// the step's latent row, paged access through the block table, split-K
// with a last-CTA merge in split-index order (flash-decoding, cited P:127).
//
// AI ~ 30 FLOP/B (SURVEY §8(d) cfg 5: "tensor cores in decode").  Swap-AB so the 16 heads
// are the MMA N dimension and keys / value columns fill M:
//   S^T[64 keys x 16]  = C_page[64 x 576] . Q^T        M=64  N=16, 36 x K16, SS
//   O^T[512 x 16]     += V^T[512 x 64] . P^T[64 x 16]   M=128 N=16, 4 blocks x 4 K16, SS
// C_page is one 64-token page, landed by two 4-D TMA boxes (column blocks [0,4) = 32 KiB
// and [4,9) = 40 KiB) into 40 KiB ring slots: [column block][64 keys][128 B], 128-B
// swizzle — K-major A for QK and, read transposed (LBO = 8 KiB between 64-column blocks,
// SBO = 1 KiB between 8-key groups), MN-major A for PV.  Q (18 KiB) arrives by TMA per
// unit; P^T ([16 heads][64 keys] bf16, K-major) is written by the softmax warps.
// TMEM: S^T double-buffered (2 x 16 cols), O^T 4 x 16 cols.  For M = 64, D row 16w + i
// sits in TMEM lane 32w + i (measured, scripts/probe_umma_m64.cu).
//
// Warps: 0 producer (units, append, TMA), 1 MMA issuer (one thread), 2-5 softmax +
// epilogue (warp w reads TMEM lane quadrant w % 4).  The work list depends on shapes
// only, so outputs are bitwise identical for every sm_budget (R26).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int DK = 576, DV = 512, NH = 16;
constexpr int PAGE = 64;                                // keys per tile = one page (bs 64)
constexpr int NCB = DK / 64;                            // 9 column blocks of 128 B
constexpr int CB_LO = 4;                                // boxes: cb [0,4) and [4,9)
constexpr uint32_t LO_BYTES = CB_LO * PAGE * 128;       // 32 KiB
constexpr uint32_t HI_BYTES = (NCB - CB_LO) * PAGE * 128;  // 40 KiB
// SPD_MLA_DQ = 1: two Q buffers (the next unit's Q lands while the current unit still runs
// QK, so the unit boundary no longer waits a Q TMA round trip) and a 4-slot ring of exactly
// sized halves (even slots 32 KiB = LO boxes, odd slots 40 KiB = HI boxes: 2 pages in flight);
// 0: one Q buffer and 5 uniform 40 KiB slots (2.5 pages in flight).  Measured (same box,
// microbench, 2 reps): DQ = 1 is 1-6 % SLOWER at every shape (B 256 ctx 350 at 44 / 104 /
// 148 SMs, B 256 ctx 1000, B 64 ctx 4000): the unit boundary is not held by the Q load, and
// the shallower ring costs more than the second Q buffer gains.  Default 0.
// SPD_MLA_PF = D > 0: the producer prefetches page i + D (both boxes) into L2 after loading
// page i, so a ring slot is held for an L2 hit instead of the HBM round trip.  Measured 1-12 %
// SLOWER (B 256 ctx 350: 3.17 -> 2.81 TB/s at 148 SMs; profiles/r2_l2_prefetch_ab.log).
// Default 0.
#ifndef SPD_MLA_PF
#define SPD_MLA_PF 0
#endif
// SPD_MLA_LOOKAHEAD = 1: while streaming a unit, the producer already resolves the next one
// (its context, request id and first 32 block ids, in two steps so no load stalls the page
// loop), so the next unit's first page goes out as soon as a ring slot frees.  Parity-green
// but neutral (+-0.5 %, profiles/r2_mla_decode_lookahead_ab.log), as in round 1: default 0.
#ifndef SPD_MLA_LOOKAHEAD
#define SPD_MLA_LOOKAHEAD 0
#endif
#ifndef SPD_MLA_DQ
#define SPD_MLA_DQ 0
#endif
constexpr uint32_t SLOT_BYTES = HI_BYTES;
constexpr int NSLOT = SPD_MLA_DQ ? 4 : 5;
constexpr int NQBUF = SPD_MLA_DQ ? 2 : 1;
constexpr uint32_t RING_BYTES = SPD_MLA_DQ ? 2 * (LO_BYTES + HI_BYTES) : NSLOT * SLOT_BYTES;
__host__ __device__ constexpr uint32_t slot_off(int s) {
    return SPD_MLA_DQ ? (uint32_t)(s >> 1) * (LO_BYTES + HI_BYTES) + (uint32_t)(s & 1) * LO_BYTES
                      : (uint32_t)s * SLOT_BYTES;
}
constexpr uint32_t Q_BYTES = NCB * NH * 128;            // 18 KiB
constexpr uint32_t P_BYTES = NH * 128;                  // 2 KiB per buffer (2 buffers)
constexpr int NTHREADS = 192;
constexpr int NSOFT = 128;
// SPD_MLA_SPLIT_PAGES: finer splits (8 / 12 / 16 pages) shorten the longest units' chains but
// their partial write-back and merge cost more at every budget (cfg-5 lognormal batch at 104 SMs:
// 0.052 / 0.048 / 0.044 vs 0.042 ms; profiles/r2_mla_decode_split_pages_ab.log).  Default 20.
#ifndef SPD_MLA_SPLIT_PAGES
#define SPD_MLA_SPLIT_PAGES 20
#endif
constexpr int SPLIT_PAGES = SPD_MLA_SPLIT_PAGES;  // a split spans at most this many pages (20: 1280 keys)

// number of splits of a request with ctx cached tokens (ctx + 1 keys): a function of the
// shape only (R26).  At least ceil(pages / 20) (1025 keys = 17 pages stay one unit).  The
// S_fill hook splits small batches further (up to S_fill splits of >= 2 pages); with
// S_fill = ceil(148 / B) the cfg-5 trace ran 7 % slower (per-split partials + merges cost
// more than the extra SMs gain), so fill_splits() returns 1.
// Splits are whole pages: pps = ceil(pages / S) pages each, and the count is re-derived from
// pps so that no split is empty (ceil(pages / ceil(pages / S)) <= S).
__host__ __device__ __forceinline__ int n_splits(int ctx, int S_fill) {
    const int pages = (ctx + 1 + PAGE - 1) / PAGE;
    const int s_len = (pages + SPLIT_PAGES - 1) / SPLIT_PAGES;
    const int s_f = S_fill < (pages + 1) / 2 ? S_fill : (pages + 1) / 2;
    int S = s_len > s_f ? s_len : s_f;
    if (S < 1) S = 1;
    const int pps = (pages + S - 1) / S;
    return (pages + pps - 1) / pps;
}
__host__ __device__ __forceinline__ int fill_splits(int B) { return B > 0 ? 1 : 1; }
// n_splits is not monotone in ctx (re-deriving the count from whole pages can drop one), so the
// workspace / unit-grid bound is the maximum over every page count up to max_ctx's
inline int max_splits(int max_ctx, int S_fill) {
    const int pages = (max_ctx + 1 + PAGE - 1) / PAGE;
    int m = 1;
    for (int pg = 1; pg <= pages; ++pg) {
        const int sp = n_splits(pg * PAGE - 1, S_fill);
        m = sp > m ? sp : m;
    }
    return m;
}
constexpr float LOG2E = 1.4426950408889634f;
// SPD_MLA_DEFER = 1: an unsplit unit's O^T read-out is deferred into the next unit: its four
// 128-dv blocks are stored after the next unit's first four P writes (one block per tile), so
// the softmax warps go straight on to the next unit's first tile instead of idling through the
// epilogue.  O^T then has one double buffer per unit parity (TMEM 512 columns).  Measured
// (profiles/r2_mla_decode_defer_ab.log, parity 36/36): +1-2 % on the lognormal cfg-5 batch,
// +4 % at B 64 / ctx 4000, within noise at ctx 1000.
#ifndef SPD_MLA_DEFER
#define SPD_MLA_DEFER 1
#endif
constexpr uint32_t TM_S = 0, TM_O = 64;              // S^T 2 x 16 cols; O^T 2 x (4 x 16) per set
constexpr uint32_t TM_OSET = SPD_MLA_DEFER ? 128 : 0;  // column offset of the odd units' O^T set
constexpr uint32_t TM_COLS = SPD_MLA_DEFER ? 512 : 256;

struct TUnit {
    int b, s, S, k0, k1, nt;  // b < 0: done
};

// SPD_MLA_SORT = 1: the launch's real units in longest-first order, built in shared memory by
// every CTA before its first unit (mla_unit_order).  The default enumeration walks the
// (split level, request) grid, S_max x B entries, and a request with fewer splits than S_max
// leaves empty entries that each cost the producer a counter atomic and a context load before
// the next real unit (cfg-5 lognormal batch: 253 of 512 entries empty, most of them handed out
// first).  Used when S_max x B <= SORT_CAP (uint16 entries b | s << 11, so B <= 2048, S <= 32).
// Measured (profiles/r2_mla_decode_sort_ab.log, MLA parity 70/70): 2-5 % SLOWER at every shape
// (cfg-5 lognormal batch 0.0410 vs 0.0391 ms at 148 SMs, 0.0684 vs 0.0668 at 44; uniform
// ctx 1000, where the order is unchanged, +2 %: the prologue's context loads and barriers delay
// every CTA's first TMA by about as much as the empty entries cost).  Finer splits stay slower
// with it (SPLIT_PAGES 10 / 14: +12-70 %).  With the builder out of line (__noinline__) the MMA
// warp's descriptors left the uniform datapath (R2UR per MMA, +25-30 %).  Default 0.
#ifndef SPD_MLA_SORT
#define SPD_MLA_SORT 0
#endif
constexpr int SORT_CAP = 1024;

struct TcParams {
    const uint4* k_new;       // [B][1][576]
    const int* req_ids;
    const int* ctx_lens;
    const int* bt;
    unsigned char* k_pool;
    __nv_bfloat16* out;       // [B][Hq][512] or [Hq][B][512]
    float* ws_m;              // [B][16][S_max]
    float* ws_l;
    float* ws_acc;            // [B][16][S_max][512]
    int* ws_cnt;              // [B]
    unsigned* sched;
    int* status;
    unsigned long long* span;  // semipd_set_spans record of this launch (or null)
    int skip_append;           // 1: the step's latent row is already in the pool (RoPE pre-pass)
    int B, MBR, N_B, S_max, n_units, out_head_major, G, S_fill;
    int sorted;  // 1: units come from the in-smem longest-first order (SPD_MLA_SORT)
    float scale_log2;
    SpdTrace trace;
    long long* tl;  // SPD_TIMELINE builds only: pipeline clock64 stamps of CTA 0
    int* tl_ctr;
};

#ifdef SPD_TIMELINE
// record slot = kind * 512 + tile: plain stores, no atomics (keeps the pipeline unperturbed)
#define TL_REC(a, b, c, d, e)                                                              \
    do {                                                                                   \
        if (p.tl && (int)blockIdx.x == tl_cta && (b) < 512) {                                        \
            long long* _r = p.tl + 8 * ((a) * 512 + (b));                                  \
            _r[0] = a; _r[1] = b; _r[2] = c; _r[3] = d; _r[4] = e;                         \
        }                                                                                  \
    } while (0)
#define TL_NOW() clock64()
#else
#define TL_REC(a, b, c, d, e) do { } while (0)
#define TL_NOW() 0LL
#endif

struct Bars {
    uint64_t full[NSLOT], empty[NSLOT], s_full[2], s_empty[2], p_full[2], o_done[2], q_full[NQBUF],
        q_empty[NQBUF], ufull[2], uempty[2];
};

constexpr uint32_t OFF_Q = RING_BYTES;
constexpr uint32_t OFF_P = OFF_Q + NQBUF * Q_BYTES;
constexpr uint32_t OFF_RED = OFF_P + 2 * P_BYTES;            // [2][64] maxima, [64] sums
constexpr uint32_t OFF_BARS = OFF_RED + 5 * 64 * 4;
constexpr uint32_t OFF_UNITS = OFF_BARS + sizeof(Bars);
constexpr uint32_t OFF_MISC = OFF_UNITS + 2 * sizeof(TUnit);
constexpr uint32_t OFF_PERM = OFF_MISC + 16;                 // [SORT_CAP] uint16 unit order
constexpr uint32_t SMEM_BYTES = 1024 + OFF_PERM + (SPD_MLA_SORT ? SORT_CAP * 2 : 0);
static_assert(OFF_Q % 1024 == 0 && OFF_P % 1024 == 0, "UMMA operands need 1 KiB alignment");
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KiB opt-in shared memory");

__device__ __forceinline__ void split_range(int ctx, int S, int s, int& k0, int& k1) {
    const int nk = ctx + 1;
    const int pages = (nk + PAGE - 1) / PAGE;
    const int pps = (pages + S - 1) / S;  // pages per split (n_splits keeps every split non-empty)
    k0 = s * pps * PAGE;
    k1 = min(nk, k0 + pps * PAGE);
}

// SPD_MLA_MERGE_FN = 1 (default): the last split's merge as a separate (non-inlined) function,
// so its registers do not enter the page loop's allocation (255 -> 244 registers, no spill),
// with (m, l) loaded by 8 threads per head at once and two splits' partials in flight (instead
// of 2 S + S serialised L2 round trips).  +1-2 % on the lognormal cfg-5 batch, neutral on split
// batches (profiles/r2_mla_decode_merge_fn_ab.log); finer splits stay slower with it.
#ifndef SPD_MLA_MERGE_FN
#define SPD_MLA_MERGE_FN 1
#endif
__device__ __noinline__ void mla_split_merge(const float* ws_m, const float* ws_l, const float* ws_acc,
                                             __nv_bfloat16* out, int* ws_cnt, int b, int S, int S_max, int G,
                                             int B, int out_head_major, int tid, float* wsm) {
    // pass 1: w[h][s] = 2^(m_s - M_h) / L_h into smem, 8 threads per head (S <= 32: 4 splits each)
    const int h1 = tid >> 3, j8 = tid & 7;
    const size_t pb1 = ((size_t)b * NH + h1) * S_max;
    float mv[4], lv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int sI = j8 + 8 * k;
        const bool ok = h1 < G && sI < S;
        mv[k] = ok ? __ldcg(ws_m + pb1 + sI) : -INFINITY;
        lv[k] = ok ? __ldcg(ws_l + pb1 + sI) : 0.f;
    }
    float M = fmaxf(fmaxf(mv[0], mv[1]), fmaxf(mv[2], mv[3]));
    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 1));
    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 2));
    M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 4));
    float f[4], Ls = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f[k] = j8 + 8 * k < S ? fast_exp2(mv[k] - M) : 0.f;
        Ls += f[k] * lv[k];
    }
    Ls += __shfl_xor_sync(0xffffffffu, Ls, 1);
    Ls += __shfl_xor_sync(0xffffffffu, Ls, 2);
    Ls += __shfl_xor_sync(0xffffffffu, Ls, 4);
    const float inv = 1.f / Ls;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (h1 < G && j8 + 8 * k < S) wsm[h1 * 32 + j8 + 8 * k] = f[k] * inv;
    named_bar_sync(1, NSOFT);
    // pass 2: each thread owns 16 float4 columns; two splits' loads in flight
    constexpr int PER = NH * (DV / 4) / NSOFT;
    float4 o[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 2
    for (int sI = 0; sI < S; ++sI) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const int idx = tid + j * NSOFT;
            const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
            if (h < G) {
                const float w = wsm[h * 32 + sI];
                const float4 a = __ldcg(reinterpret_cast<const float4*>(ws_acc + (((size_t)b * NH + h) * S_max + sI) * DV + c));
                o[j].x += w * a.x;
                o[j].y += w * a.y;
                o[j].z += w * a.z;
                o[j].w += w * a.w;
            }
        }
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int idx = tid + j * NSOFT;
        const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
        if (h >= G) continue;
        const size_t off = out_head_major ? (((size_t)h * B + b) * DV + c) : (((size_t)b * G + h) * DV + c);
        uint2 v;
        v.x = pack_bf16(o[j].x, o[j].y);
        v.y = pack_bf16(o[j].z, o[j].w);
        *reinterpret_cast<uint2*>(out + off) = v;
    }
    if (tid == 0) ws_cnt[b] = 0;
}

// Longest-first order of the launch's real (request, split) units (SPD_MLA_SORT): a stable
// counting sort by page count, descending, ties in (b, s) order.  A function of the shapes only,
// so every CTA builds the same list and outputs stay bitwise identical for every sm_budget (R26;
// the order only decides which CTA runs a unit, never its arithmetic).  All NTHREADS threads;
// the scratch is the still-idle ring.  Needs B <= 6 * NTHREADS (implied by S_max x B <= SORT_CAP).
__device__ __forceinline__ void mla_unit_order(const int* ctx_lens, int B, int S_fill, unsigned char* scratch,
                                            uint16_t* perm, int* s_ntot) {
    constexpr int NW = NTHREADS / 32;
    constexpr int PER = 6;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    int* wsum = reinterpret_cast<int*>(scratch);                      // [8]
    int* wcnt = wsum + 8;                                             // [NW][32]: counts, then bases
    uint16_t* ccode = reinterpret_cast<uint16_t*>(wcnt + NW * 32);    // [SORT_CAP] canonical units
    uint8_t* ckey = reinterpret_cast<uint8_t*>(ccode + SORT_CAP);     // [SORT_CAP] their page counts
    for (int i = tid; i < NW * 32; i += NTHREADS) wcnt[i] = 0;
    // 1. splits of this thread's consecutive requests; block exclusive scan -> canonical offsets
    const int per = (B + NTHREADS - 1) / NTHREADS;
    int cl[PER], sl[PER], loc = 0;
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        const int b = tid * per + j;
        cl[j] = (j < per && b < B) ? __ldg(ctx_lens + b) : -1;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        sl[j] = cl[j] >= 0 ? n_splits(cl[j], S_fill) : 0;
        loc += sl[j];
    }
    int inc = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    int c = inc - loc, tot = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const int v = wsum[i];
        if (i < w) c += v;
        tot += v;
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
        for (int sI = 0; sI < sl[j]; ++sI, ++c) {
            int k0, k1;
            split_range(cl[j], sl[j], sI, k0, k1);
            const int nt = (k1 - k0 + PAGE - 1) / PAGE;
            ccode[c] = (uint16_t)((tid * per + j) | (sI << 11));
            ckey[c] = (uint8_t)(nt < 31 ? nt : 31);
        }
    }
    __syncthreads();
    // 2. per-warp key counts over warp w's canonical range
    const int L = ((tot + NW - 1) / NW + 31) & ~31;
    const int r0 = w * L, r1 = min(tot, r0 + L);
    for (int c0 = r0; c0 < r1; c0 += 32) {
        const int cc = c0 + lane;
        const int key = cc < r1 ? (int)ckey[cc] : -1;
        const unsigned m = __match_any_sync(0xffffffffu, key);
        if (key >= 0 && lane == __ffs(m) - 1) wcnt[w * 32 + key] += __popc(m);
        __syncwarp();
    }
    __syncthreads();
    // 3. bases: keys in descending order, warps in canonical order within a key
    if (w == 0) {
        int pw[NW], t = 0;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            pw[i] = wcnt[i * 32 + lane];
            t += pw[i];
        }
        int suf = t;  // sum over keys >= lane
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_down_sync(0xffffffffu, suf, o);
            if (lane + o < 32) suf += v;
        }
        int base = suf - t;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            wcnt[i * 32 + lane] = base;
            base += pw[i];
        }
    }
    __syncthreads();
    // 4. placement: rank among equal keys, stable within the warp's range
    for (int c0 = r0; c0 < r1; c0 += 32) {
        const int cc = c0 + lane;
        const int key = cc < r1 ? (int)ckey[cc] : -1;
        const unsigned m = __match_any_sync(0xffffffffu, key);
        if (key >= 0) perm[wcnt[w * 32 + key] + __popc(m & ((1u << lane) - 1u))] = ccode[cc];
        __syncwarp();
        if (key >= 0 && lane == __ffs(m) - 1) wcnt[w * 32 + key] += __popc(m);
        __syncwarp();
    }
    if (tid == 0) *s_ntot = tot;
    fence_proxy_async_smem();  // the ring's generic scratch writes before its TMA fills
    __syncthreads();
}

__global__ void __launch_bounds__(NTHREADS, 1)
    decode_mla_tc_kernel(const __grid_constant__ CUtensorMap map_lo,
                         const __grid_constant__ CUtensorMap map_hi,
                         const __grid_constant__ CUtensorMap qmap, TcParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ring = base;
    unsigned char* qs = base + OFF_Q;
    unsigned char* ps = base + OFF_P;
    float* red = reinterpret_cast<float*>(base + OFF_RED);
    Bars& bar = *reinterpret_cast<Bars*>(base + OFF_BARS);
    TUnit* units = reinterpret_cast<TUnit*>(base + OFF_UNITS);
    int* s_last = reinterpret_cast<int*>(base + OFF_MISC);
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(base + OFF_MISC + 4);

    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    if (threadIdx.x == 0) {
        for (int i = 0; i < NSLOT; ++i) {
            mbar_init(bar.full + i, 1);
            mbar_init(bar.empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar.s_full + i, 1);
            mbar_init(bar.s_empty + i, 4);
            mbar_init(bar.ufull + i, 1);
            mbar_init(bar.uempty + i, 5);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(bar.p_full + i, 4);
            mbar_init(bar.o_done + i, 1);
        }
        for (int i = 0; i < NQBUF; ++i) {
            mbar_init(bar.q_full + i, 1);
            mbar_init(bar.q_empty + i, 1);
        }
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(2, (int)smid(), (int)blockIdx.x, 4 /* kernel kind: MLA tcgen05 */);
        }
    }
#ifdef SPD_TIMELINE
    const int tl_cta = p.tl ? *p.tl_ctr : -1;  // which CTA records its pipeline
    unsigned long long g_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
    int n_units_done = 0;
#endif
    if (warp == 1) tmem_alloc(tmem_base, TM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (workspace counters, pool)
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = *tmem_base;
    uint16_t* perm = reinterpret_cast<uint16_t*>(base + OFF_PERM);
    int* s_ntot = reinterpret_cast<int*>(base + OFF_MISC + 8);
    const bool sorted = SPD_MLA_SORT && p.sorted;
    if (sorted) mla_unit_order(p.ctx_lens, p.B, p.S_fill, ring, perm, s_ntot);
    const int n_lim = sorted ? *s_ntot : p.n_units;

    if (warp == 0) {
        // =========================== producer ===========================
        if (lane == 0) {
            tma_prefetch_desc(&map_lo);
            tma_prefetch_desc(&map_hi);
            tma_prefetch_desc(&qmap);
        }
        int gh = 0, nunit = 0, nq = 0;
        // first unit of each CTA is static (blockIdx.x); later ones come from the counter,
        // fetched one unit ahead so the atomic's round trip overlaps the current unit
        int u_next = blockIdx.x;
        // lookahead state: the unit la_u's context / request id (step 1) and its first 32 block
        // ids (step 2, la_ok)
        int la_u = -1, la_ctx = 0, la_rid = 0, la_blk = -1;
        bool la_ok = false;
        for (;;) {
            const int u = u_next;
            if (lane == 0) u_next = (int)gridDim.x + (int)atomicAdd(p.sched, 1u);
            u_next = __shfl_sync(0xffffffffu, u_next, 0);
            TUnit d;
            int ctx = 0, rid = 0;
            const bool have_la = SPD_MLA_LOOKAHEAD && u == la_u;
            if (u >= n_lim) {
                d.b = -1;
            } else {
                if (sorted) {
                    const unsigned code = perm[u];
                    d.b = (int)(code & 2047u);
                    d.s = (int)(code >> 11);
                } else {
                    // longest-first: units of the highest split index (full-length splits of
                    // the longest requests) are handed out first
                    d.s = p.S_max - 1 - u / p.B;
                    d.b = u % p.B;
                }
                ctx = have_la ? la_ctx : __ldg(p.ctx_lens + d.b);
                rid = have_la ? la_rid : __ldg(p.req_ids + d.b);
                d.S = n_splits(ctx, p.S_fill);
                if (d.s >= d.S) continue;
                split_range(ctx, d.S, d.s, d.k0, d.k1);
                d.nt = (d.k1 - d.k0 + PAGE - 1) / PAGE;
            }
            const int us = nunit & 1;
            if (lane == 0) {
                mbar_wait(bar.uempty + us, ((nunit >> 1) & 1) ^ 1);
                units[us] = d;
                mbar_arrive(bar.ufull + us);
            }
            __syncwarp();
            ++nunit;
            if (d.b < 0) {  // no more units: the next kernel on the stream may be scheduled
                pdl_trigger();
                break;
            }
            const int* btr = p.bt + (size_t)rid * p.MBR;
            const int last_page = ctx / PAGE;
            // fused append (last split only): the step's latent row (576 bf16 = 72 x 16 B) goes
            // to slot ctx right before the TMA of the page holding it
            const bool append = d.s == d.S - 1 && !p.skip_append;
            uint4 kn[3];
            if (append) {
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int c = lane + 32 * j;
                    kn[j] = c < DK / 8 ? __ldg(p.k_new + (size_t)d.b * (DK / 8) + c) : make_uint4(0, 0, 0, 0);
                }
            }
            const int page0 = d.k0 / PAGE;
            int blk_l = -1;
            const bool use_la_blk = have_la && la_ok;
            la_u = -1;
            la_ok = false;
            for (int i = 0; i < d.nt; ++i, gh += 2) {
                if ((i & 31) == 0) {
                    if (i == 0 && use_la_blk) {
                        blk_l = la_blk;
                    } else {
                        const int pg = page0 + i + lane;
                        blk_l = (pg <= last_page && pg < p.MBR) ? __ldg(btr + pg) : -1;
                    }
                }
                const int blk = __shfl_sync(0xffffffffu, blk_l, i & 31);
                if (append && page0 + i == last_page && blk >= 0 && blk < p.N_B) {
                    uint4* dst = reinterpret_cast<uint4*>(p.k_pool) + ((size_t)blk * PAGE + (ctx % PAGE)) * (DK / 8);
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        if (lane + 32 * j < DK / 8) dst[lane + 32 * j] = kn[j];
                    fence_proxy_async_global();
                    __syncwarp();
                }
                if (lane == 0) {
                    int z = p.N_B;  // out of range: zero fill
                    if (blk >= 0 && blk < p.N_B) z = blk;
                    else if (p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                    const int s0 = gh % NSLOT, s1 = (gh + 1) % NSLOT;
                    [[maybe_unused]] const long long tp0 = TL_NOW();
                    mbar_wait(bar.empty + s0, ((gh / NSLOT) & 1) ^ 1);
                    [[maybe_unused]] const long long tp1 = TL_NOW();
                    mbar_arrive_expect_tx(bar.full + s0, LO_BYTES);
                    tma_load_4d(ring + slot_off(s0), &map_lo, bar.full + s0, 0, 0, 0, z);
                    if (i == 0) {
                        // Q of this unit: its buffer frees when the last QK of the unit that
                        // used it before completes (issued before this tile: no deadlock)
                        const int qb = nq % NQBUF;
                        mbar_wait(bar.q_empty + qb, ((nq / NQBUF) & 1) ^ 1);
                        mbar_arrive_expect_tx(bar.q_full + qb, Q_BYTES);
                        tma_load_4d(qs + qb * Q_BYTES, &qmap, bar.q_full + qb, 0, 0, 0, d.b);
                    }
                    mbar_wait(bar.empty + s1, (((gh + 1) / NSLOT) & 1) ^ 1);
                    mbar_arrive_expect_tx(bar.full + s1, HI_BYTES);
                    tma_load_4d(ring + slot_off(s1), &map_hi, bar.full + s1, 0, 0, CB_LO, z);
                    TL_REC(1, gh / 2, tp0, tp1, TL_NOW());
                }
                if constexpr (SPD_MLA_PF > 0) {
                    // page i + D of this unit, if its block id is in the current 32-page batch
                    const int ip = i + SPD_MLA_PF;
                    const int bp = __shfl_sync(0xffffffffu, blk_l, ip & 31);
                    if (lane == 0 && ip < d.nt && (ip >> 5) == (i >> 5) && bp >= 0 && bp < p.N_B) {
                        tma_prefetch_l2_4d(&map_lo, 0, 0, 0, bp);
                        tma_prefetch_l2_4d(&map_hi, 0, 0, CB_LO, bp);
                    }
                }
                // after this page's TMA issue, so no lookahead load delays it
                if (SPD_MLA_LOOKAHEAD && !sorted && i == 0 && u_next < p.n_units) {
                    // step 1: the next unit's context and request id (consumed at step 2)
                    la_u = u_next;
                    const int b2 = u_next % p.B;
                    la_ctx = __ldg(p.ctx_lens + b2);
                    la_rid = __ldg(p.req_ids + b2);
                }
                if (SPD_MLA_LOOKAHEAD && i == (d.nt > 1 ? 1 : 0) && la_u >= 0) {
                    // step 2 (a page later): its split range and first 32 block ids
                    const int s2 = p.S_max - 1 - la_u / p.B;
                    const int S2 = n_splits(la_ctx, p.S_fill);
                    if (s2 < S2) {
                        int k0b, k1b;
                        split_range(la_ctx, S2, s2, k0b, k1b);
                        const int pg = k0b / PAGE + lane;
                        la_blk = (pg <= la_ctx / PAGE && pg < p.MBR) ? __ldg(p.bt + (size_t)la_rid * p.MBR + pg) : -1;
                        la_ok = true;
                    }
                }
                __syncwarp();
            }
            ++nq;
        }
    } else if (warp == 1) {
        // =========================== MMA issuer (warp-collective) ===========================
        // The whole warp runs this loop with uniform state; elect.sync inside the asm picks
        // the issuing lane, so descriptors stay in uniform registers.  Barrier probes are
        // taken by lane 0 and broadcast so every lane takes the same branch.
        constexpr uint32_t ID_QK = umma_idesc_bf16_f32_ab(64, NH, 0, 0);
        constexpr uint32_t ID_PV = umma_idesc_bf16_f32_ab(128, NH, 1, 0);
        const uint32_t ring_a = smem_u32(ring), q_a = smem_u32(qs), p_a = smem_u32(ps);
        // smem descriptors as (low, high) words: the K16 / block offsets are 32-bit adds to the
        // low word on the uniform datapath (umma_ss_warp2)
        const uint32_t dq0 = desc_lo(q_a, 16);
        const uint32_t dp0 = desc_lo(p_a, 16);
        constexpr uint32_t DH = DESC_HI_SBO1K;
        auto probe = [&](const uint64_t* b, uint32_t par) {
            bool r = false;
            if (lane == 0) r = mbar_test_wait(b, par);
            return __shfl_sync(0xffffffffu, r ? 1 : 0, 0) != 0;
        };
        int gh = 0, gt = 0, nunit = 0, nq = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(bar.ufull + us, (nunit >> 1) & 1);
            const TUnit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(bar.uempty + us);
            ++nunit;
            if (d.b < 0) break;
            // PV(t) as soon as P(t) is written (it releases tile t's ring slots), else QK(t)
            // as soon as tile t has landed.
            bool q_ok = false, qk_lo = false;
            int nqk = 0, npv = 0;
            while (npv < d.nt) {
                const int tp = gt + npv, ob = tp & 1;
                if (npv < nqk && probe(bar.p_full + ob, (tp >> 1) & 1)) {
                    const int h0 = gh + 2 * npv;
                    const int s0 = h0 % NSLOT, s1 = (h0 + 1) % NSLOT;
                    tc_fence_after();
                    const uint32_t lo = ring_a + slot_off(s0), hi = ring_a + slot_off(s1);
#pragma unroll
                    for (int m = 0; m < DV / 128; ++m) {
                        // dv block m = column blocks 2m, 2m+1 (both in the same half-page)
                        const uint32_t a0 = m < 2 ? lo + m * (2 * PAGE * 128)
                                                  : hi + (2 * m - CB_LO) * (PAGE * 128);
                        const uint32_t da = desc_lo(a0, PAGE * 128);
#pragma unroll
                        for (int ks = 0; ks < PAGE / 16; ++ks)
                            umma_ss_warp2(tmem + TM_O + ((nunit - 1) & 1) * TM_OSET + ob * 64 + m * NH,
                                          da + (uint32_t)(ks * 128), DH,
                                          dp0 + (uint32_t)(ob * (P_BYTES / 16) + ks * 2), DH, ID_PV,
                                          (npv > 1 || ks > 0) ? 1u : 0u);
                        if (m == 1) umma_commit_warp(bar.empty + s0);  // blocks 0,1 read the first box
                    }
                    umma_commit_warp(bar.o_done + ob);
                    umma_commit_warp(bar.empty + s1);
                    if (lane == 0) TL_REC(3, gt + npv, TL_NOW(), 0, 0);
                    ++npv;
                    continue;
                }
                if (nqk < d.nt) {
                    // QK(t) in two halves: column blocks [0,4) as soon as the first box has
                    // landed, [4,9) when the second has
                    const int t = gt + nqk, sb = t & 1, h0 = gh + 2 * nqk;
                    const int s0 = h0 % NSLOT, s1 = (h0 + 1) % NSLOT;
                    const int qb = nq % NQBUF;
                    if (!q_ok) q_ok = probe(bar.q_full + qb, (nq / NQBUF) & 1);
                    if (q_ok && !qk_lo && probe(bar.s_empty + sb, ((t >> 1) & 1) ^ 1) &&
                        probe(bar.full + s0, (h0 / NSLOT) & 1)) {
                        tc_fence_after();
                        const uint32_t dlo = desc_lo(ring_a + slot_off(s0), 16);
                        const uint32_t dq = dq0 + (uint32_t)(qb * (Q_BYTES / 16));
#pragma unroll
                        for (int k = 0; k < CB_LO * 4; ++k) {
                            const int cb = k >> 2;
                            // descriptor start address is in 16-byte units
                            umma_ss_warp2(tmem + TM_S + sb * NH, dlo + (uint32_t)(cb * (PAGE * 128 / 16) + (k & 3) * 2), DH,
                                          dq + (uint32_t)(cb * (NH * 128 / 16) + (k & 3) * 2), DH, ID_QK, k > 0);
                        }
                        qk_lo = true;
                        continue;
                    }
                    if (qk_lo && probe(bar.full + s1, ((h0 + 1) / NSLOT) & 1)) {
                        tc_fence_after();
                        const uint32_t dhi = desc_lo(ring_a + slot_off(s1), 16);
                        const uint32_t dq = dq0 + (uint32_t)(qb * (Q_BYTES / 16));
#pragma unroll
                        for (int k = CB_LO * 4; k < DK / 16; ++k) {
                            const int cb = k >> 2;
                            umma_ss_warp2(tmem + TM_S + sb * NH, dhi + (uint32_t)((cb - CB_LO) * (PAGE * 128 / 16) + (k & 3) * 2), DH,
                                          dq + (uint32_t)(cb * (NH * 128 / 16) + (k & 3) * 2), DH, ID_QK, 1u);
                        }
                        umma_commit_warp(bar.s_full + sb);
                        if (lane == 0) TL_REC(2, t, TL_NOW(), 0, 0);
                        if (nqk == d.nt - 1) umma_commit_warp(bar.q_empty + qb);
                        qk_lo = false;
                        ++nqk;
                        continue;
                    }
                }
                __nanosleep(32);  // nothing ready: yield issue slots to the softmax warp
                                  // sharing this SM sub-partition
            }
            ++nq;
            gt += d.nt;
            gh += 2 * d.nt;
        }
    } else {
        // =========================== softmax + epilogue ===========================
        const int qd = warp & 3;                       // TMEM lane quadrant
        const int tid = threadIdx.x - 64;              // 0..127
        const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
        float* red_l = red + 128;
        const bool odd = lane & 1;
        const size_t ohs = p.out_head_major ? (size_t)p.B * DV : (size_t)DV;
        const size_t whs = (size_t)p.S_max * DV;
        // one 128-dv block of a unit's O^T read-out: combine the two buffers of set upx with the
        // per-head factors facp (smem), then store bf16 output (unsplit) or fp32 partials (split).
        // Lane pairs (dv, dv + 1) exchange so each lane stores bf16x2 for 8 of the 16 heads
        // (even lane: heads 0-7, odd lane: heads 8-15)
        auto store_block = [&](int m, int b, int s_idx, int upx, int bl, bool two, bool split,
                               const float* facp) {
            uint32_t o[NH], o2[NH];
            const uint32_t ob0 = tmem + lane_base + TM_O + upx * TM_OSET;
            tmem_ld16(ob0 + bl * 64 + m * NH, o);
            if (two) tmem_ld16(ob0 + (bl ^ 1) * 64 + m * NH, o2);
            tmem_wait_ld();
            const int dv = m * 128 + qd * 32 + lane;
            auto val = [&](int h) {
                const float x = __uint_as_float(o[h]) * facp[h];
                return two ? fmaf(__uint_as_float(o2[h]), facp[NH + h], x) : x;
            };
            if (!split) {
                __nv_bfloat16* op = p.out + (p.out_head_major ? (size_t)b * DV : (size_t)b * p.G * DV) +
                                    (dv & ~1) + (odd ? 8 * ohs : 0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    // even lanes store head j, odd lanes head j + 8
                    const float a0 = val(j), a1 = val(j + 8);
                    const float send = odd ? a0 : a1;
                    const float got = __shfl_xor_sync(0xffffffffu, send, 1);
                    const int h = odd ? j + 8 : j;
                    if (h < p.G)
                        *reinterpret_cast<uint32_t*>(op + j * ohs) =
                            odd ? pack_bf16(got, a1) : pack_bf16(a0, got);
                }
            } else {
                float* wp = p.ws_acc + ((size_t)b * NH * p.S_max + s_idx) * DV + dv;
#pragma unroll
                for (int h = 0; h < NH; ++h)
                    if (h < p.G) wp[h * whs] = val(h);
            }
        };
        // the deferred read-out of the previous unsplit unit (SPD_MLA_DEFER)
        bool pend = false, pend_ready = false, pend_two = false;
        int pend_b = 0, pend_up = 0, pend_bl = 0, pend_chunk = 0;
        int gt = 0, nunit = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(bar.ufull + us, (nunit >> 1) & 1);
            const TUnit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(bar.uempty + us);
            const int up = nunit & 1;  // this unit's O^T set
            ++nunit;
            if (d.b < 0) break;
            // O^T is double-buffered: PV(t) accumulates into buffer t & 1 with P(t) from P
            // buffer t & 1, so writing P(t) / rescaling O_(t&1) waits only for PV(t-2) and
            // the softmax of tile t overlaps PV(t-1).  Buffer contents are relative to the
            // running max at their last update (mold2 for tile t-2); the epilogue combines.
            float mrun[NH], mold2[NH], lpart[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                mrun[h] = -INFINITY;
                mold2[h] = -INFINITY;
                lpart[h] = 0.f;
            }
            for (int i = 0; i < d.nt; ++i) {
                const int t = gt + i, sb = t & 1;
                [[maybe_unused]] const long long ts0 = TL_NOW();
                mbar_wait(bar.s_full + sb, (t >> 1) & 1);
                [[maybe_unused]] const long long ts1 = TL_NOW();
                tc_fence_after();
                uint32_t r[NH];
                tmem_ld16(tmem + lane_base + TM_S + sb * NH, r);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar.s_empty + sb);
                const int key = d.k0 + i * PAGE + qd * 16 + lane;
                const bool valid = lane < 16 && key < d.k1;
                float x[NH];
                float mine = -INFINITY;
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    x[h] = valid ? __uint_as_float(r[h]) * p.scale_log2 : -INFINITY;
                    const float mx = redux_max_f32(x[h]);
                    mine = lane == h ? mx : mine;
                }
                float* rm = red + (t & 1) * 64;
                if (lane < NH) rm[qd * NH + lane] = mine;
                named_bar_sync(1, NSOFT);
                float mn[NH];
#pragma unroll
                for (int h4 = 0; h4 < NH / 4; ++h4) {
                    const float4 a = reinterpret_cast<const float4*>(rm)[h4];
                    const float4 b = reinterpret_cast<const float4*>(rm + NH)[h4];
                    const float4 c = reinterpret_cast<const float4*>(rm + 2 * NH)[h4];
                    const float4 e = reinterpret_cast<const float4*>(rm + 3 * NH)[h4];
                    mn[h4 * 4 + 0] = fmaxf(mrun[h4 * 4 + 0], fmaxf(fmax3(a.x, b.x, c.x), e.x));
                    mn[h4 * 4 + 1] = fmaxf(mrun[h4 * 4 + 1], fmaxf(fmax3(a.y, b.y, c.y), e.y));
                    mn[h4 * 4 + 2] = fmaxf(mrun[h4 * 4 + 2], fmaxf(fmax3(a.z, b.z, c.z), e.z));
                    mn[h4 * 4 + 3] = fmaxf(mrun[h4 * 4 + 3], fmaxf(fmax3(a.w, b.w, c.w), e.w));
                }
                // the 32 per-head factors are warp-uniform: lane h computes 2^(mrun - mn) (the
                // l rescale) and lane 16 + h 2^(mold2 - mn) (the O_(t&1) rescale), one MUFU
                // op per lane instead of 32, then broadcast
                float scl[NH];
                bool grow = false;
                {
                    float e_in = 0.f;
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        e_in = lane == h ? mrun[h] - mn[h] : e_in;
                        e_in = lane == h + 16 ? mold2[h] - mn[h] : e_in;
                        grow |= mn[h] > mold2[h];
                    }
                    const float e = fast_exp2(e_in);
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        lpart[h] *= __shfl_sync(0xffffffffu, e, h);
                        scl[h] = __shfl_sync(0xffffffffu, e, h + 16);
                        mold2[h] = mrun[h];
                        mrun[h] = mn[h];
                    }
                }
                uint32_t pb[NH];
#pragma unroll
                for (int h = 0; h < NH; ++h) {
                    const __nv_bfloat16 pv = __float2bfloat16_rn(fast_exp2(x[h] - mrun[h]));
                    pb[h] = (uint32_t)__bfloat16_as_ushort(pv);
                    lpart[h] += __bfloat162float(pv);
                }
                // P buffer / O buffer t & 1 are free once PV(t-2) completed
                const int ob = t & 1;
                [[maybe_unused]] const long long ts2 = TL_NOW();
                if (t >= 2) mbar_wait(bar.o_done + ob, ((t >> 1) & 1) ^ 1);
                [[maybe_unused]] const long long ts3 = TL_NOW();
                tc_fence_after();
                if (grow && i >= 2) {
                    const uint32_t ta = tmem + lane_base + TM_O + up * TM_OSET + ob * 64;
                    uint32_t o[4][NH];
#pragma unroll
                    for (int m = 0; m < DV / 128; ++m) tmem_ld16(ta + m * NH, o[m]);
                    tmem_wait_ld();
#pragma unroll
                    for (int m = 0; m < DV / 128; ++m) {
#pragma unroll
                        for (int h = 0; h < NH; ++h) o[m][h] = __float_as_uint(__uint_as_float(o[m][h]) * scl[h]);
                        tmem_st16(ta + m * NH, o[m]);
                    }
                    tmem_wait_st();
                }
                // P^T [16 heads][64 keys] bf16, K-major 128-B swizzle; lane pairs store 4 B
                {
                    unsigned char* pbuf = ps + ob * P_BYTES;
                    const int kk = qd * 16 + (lane & ~1);
                    const bool odd = lane & 1;
#pragma unroll
                    for (int h = 0; h < NH; ++h) {
                        const uint32_t other = __shfl_xor_sync(0xffffffffu, pb[h], 1);
                        const bool mine_h = odd ? (h >= 8) : (h < 8);
                        if (lane < 16 && mine_h) {
                            const uint32_t v = odd ? (other | (pb[h] << 16)) : (pb[h] | (other << 16));
                            const uint32_t off = h * 128 + ((((kk >> 3) ^ (h & 7)) << 4) | ((kk & 7) << 1));
                            *reinterpret_cast<uint32_t*>(pbuf + off) = v;
                        }
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar.p_full + ob);
                if (pend) {
                    if (!pend_ready) {
                        // the previous unit's last PV (tile gt - 1): its barrier cannot have
                        // moved on, the next PV of that parity needs a P not yet written; the
                        // one before (gt - 2) was waited for above
                        mbar_wait(bar.o_done + ((gt - 1) & 1), ((gt - 1) >> 1) & 1);
                        tc_fence_after();
                        pend_ready = true;
                    }
                    store_block(pend_chunk, pend_b, 0, pend_up, pend_bl, pend_two, false,
                                red + 192 + pend_up * 48);
                    if (++pend_chunk == DV / 128) pend = false;
                    tc_fence_before();
                }
                if (lane == 0 && qd == 2) {
                    TL_REC(4, t, ts0, ts1, ts2);
                    TL_REC(5, t, ts3, TL_NOW(), 0);
                }
            }
            gt += d.nt;
            // the previous unit's blocks this (short) unit had no tiles left for
            if (pend) {
                while (pend_chunk < DV / 128)
                    store_block(pend_chunk++, pend_b, 0, pend_up, pend_bl, pend_two, false,
                                red + 192 + pend_up * 48);
                pend = false;
                tc_fence_before();
            }
            // ---- unit epilogue: l totals, O^T from TMEM (combining the two buffers)
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                float v = lpart[h];
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 2);
                v += __shfl_xor_sync(0xffffffffu, v, 1);
                lpart[h] = v;  // lanes 0..15 hold the warp's total (lanes 16..31 contribute 0)
            }
            {
                float mine = 0.f;
#pragma unroll
                for (int h = 0; h < NH; ++h) mine = lane == h ? lpart[h] : mine;
                if (lane < NH) red_l[qd * NH + lane] = mine;
            }
            [[maybe_unused]] const long long te0 = TL_NOW();
            const int bl = (gt - 1) & 1;  // buffer of the last tile (relative to mrun)
            const bool two = d.nt >= 2;   // the other buffer holds tiles <= nt-2 (mold2)
            const bool split = d.S > 1;
            const bool defer = SPD_MLA_DEFER && !split;
            if (!defer) {
                mbar_wait(bar.o_done + bl, ((gt - 1) >> 1) & 1);
                if (two) mbar_wait(bar.o_done + (bl ^ 1), ((gt - 2) >> 1) & 1);
                tc_fence_after();
            }
            named_bar_sync(1, NSOFT);
            // per-head factors, formed once by 16 threads into smem (registers stay free for
            // the O^T tiles): fac[h] multiplies the last tile's buffer, fac[16 + h] the other
            // one (its contents are relative to mold2); unsplit units fold in 1 / L.  One slot
            // per O^T set, so a deferred unit's factors survive the next unit's
            float* fac = red + 192 + up * 48;  // [3][16]: factor, other-buffer factor, L
            if (tid < NH) {
                float mr = mrun[0], mo = mold2[0];
#pragma unroll
                for (int h = 1; h < NH; ++h) {
                    mr = tid == h ? mrun[h] : mr;
                    mo = tid == h ? mold2[h] : mo;
                }
                const float Lh = red_l[tid] + red_l[NH + tid] + red_l[2 * NH + tid] + red_l[3 * NH + tid];
                const float f2 = two ? fast_exp2(mo - mr) : 0.f;
                const float r = split ? 1.f : __fdividef(1.f, Lh);
                fac[tid] = r;
                fac[NH + tid] = f2 * r;
                fac[2 * NH + tid] = Lh;
            }
            named_bar_sync(1, NSOFT);
            [[maybe_unused]] const long long te1 = TL_NOW();
            if (defer) {
                pend = true;
                pend_ready = false;
                pend_b = d.b;
                pend_up = up;
                pend_bl = bl;
                pend_two = two;
                pend_chunk = 0;
            } else {
#pragma unroll 1
                for (int m = 0; m < DV / 128; ++m) store_block(m, d.b, d.s, up, bl, two, split, fac);
            }
            tc_fence_before();
            if (split) {
                if (tid < p.G) {
                    const size_t pi = ((size_t)d.b * NH + tid) * p.S_max + d.s;
                    float mv = mrun[0];
#pragma unroll
                    for (int h = 1; h < NH; ++h) mv = tid == h ? mrun[h] : mv;
                    p.ws_m[pi] = mv;
                    p.ws_l[pi] = fac[2 * NH + tid];
                }
                __threadfence();
                named_bar_sync(1, NSOFT);
                if (tid == 0) *s_last = atomicAdd(p.ws_cnt + d.b, 1) == d.S - 1;
                named_bar_sync(1, NSOFT);
                if (*s_last) {
                    __threadfence();
#if SPD_MLA_MERGE_FN
                    mla_split_merge(p.ws_m, p.ws_l, p.ws_acc, p.out, p.ws_cnt, d.b, d.S, p.S_max, p.G, p.B,
                                    p.out_head_major, tid, reinterpret_cast<float*>(ps));
#else
                    // merge in split-index order.  Pass 1 (one thread per head): weights
                    // w[h][s] = 2^(m_s - M) / L into smem (the P buffer is idle here: PV of
                    // the unit's last tile completed).  Pass 2: each thread owns 16 float4
                    // columns and streams the S partials with 16 loads in flight.
                    float* wsm = reinterpret_cast<float*>(ps);  // [16][S], S <= 32
                    const bool staged = d.S <= 32;
                    if (staged && tid < p.G) {
                        const size_t pb0 = ((size_t)d.b * NH + tid) * p.S_max;
                        float M = -INFINITY;
                        for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb0 + sI));
                        float Ls = 0.f;
                        for (int sI = 0; sI < d.S; ++sI) {
                            const float f = fast_exp2(__ldcg(p.ws_m + pb0 + sI) - M);
                            wsm[tid * 32 + sI] = f;
                            Ls += f * __ldcg(p.ws_l + pb0 + sI);
                        }
                        const float inv = 1.f / Ls;
                        for (int sI = 0; sI < d.S; ++sI) wsm[tid * 32 + sI] *= inv;
                    }
                    named_bar_sync(1, NSOFT);
                    if (staged) {
                        constexpr int PER = NH * (DV / 4) / NSOFT;  // 16 float4 per thread
                        float4 o[PER];
#pragma unroll
                        for (int j = 0; j < PER; ++j) o[j] = make_float4(0.f, 0.f, 0.f, 0.f);
                        for (int sI = 0; sI < d.S; ++sI) {
#pragma unroll
                            for (int j = 0; j < PER; ++j) {
                                const int idx = tid + j * NSOFT;
                                const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
                                if (h < p.G) {
                                    const float w = wsm[h * 32 + sI];
                                    const float4 a = __ldcg(reinterpret_cast<const float4*>(
                                        p.ws_acc + (((size_t)d.b * NH + h) * p.S_max + sI) * DV + c));
                                    o[j].x += w * a.x;
                                    o[j].y += w * a.y;
                                    o[j].z += w * a.z;
                                    o[j].w += w * a.w;
                                }
                            }
                        }
#pragma unroll
                        for (int j = 0; j < PER; ++j) {
                            const int idx = tid + j * NSOFT;
                            const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
                            if (h >= p.G) continue;
                            const size_t off = p.out_head_major ? (((size_t)h * p.B + d.b) * DV + c)
                                                                : (((size_t)d.b * p.G + h) * DV + c);
                            uint2 v;
                            v.x = pack_bf16(o[j].x, o[j].y);
                            v.y = pack_bf16(o[j].z, o[j].w);
                            *reinterpret_cast<uint2*>(p.out + off) = v;
                        }
                    } else {
                        for (int idx = tid; idx < p.G * (DV / 4); idx += NSOFT) {
                            const int h = idx / (DV / 4), c = (idx % (DV / 4)) * 4;
                            const size_t pb0 = ((size_t)d.b * NH + h) * p.S_max;
                            float M = -INFINITY;
                            for (int sI = 0; sI < d.S; ++sI) M = fmaxf(M, __ldcg(p.ws_m + pb0 + sI));
                            float Ls = 0.f;
                            float4 o = make_float4(0.f, 0.f, 0.f, 0.f);
                            for (int sI = 0; sI < d.S; ++sI) {
                                const float f = fast_exp2(__ldcg(p.ws_m + pb0 + sI) - M);
                                Ls += f * __ldcg(p.ws_l + pb0 + sI);
                                const float4 a = __ldcg(reinterpret_cast<const float4*>(p.ws_acc + (pb0 + sI) * DV + c));
                                o.x += f * a.x;
                                o.y += f * a.y;
                                o.z += f * a.z;
                                o.w += f * a.w;
                            }
                            const float inv = 1.f / Ls;
                            const size_t off = p.out_head_major ? (((size_t)h * p.B + d.b) * DV + c)
                                                                : (((size_t)d.b * p.G + h) * DV + c);
                            uint2 v;
                            v.x = pack_bf16(o.x * inv, o.y * inv);
                            v.y = pack_bf16(o.z * inv, o.w * inv);
                            *reinterpret_cast<uint2*>(p.out + off) = v;
                        }
                    }
                    if (tid == 0) p.ws_cnt[d.b] = 0;
#endif
                }
            }
            [[maybe_unused]] const long long te2 = TL_NOW();
            // red_l / s_last are rewritten by the next unit
            named_bar_sync(1, NSOFT);
            if (lane == 0 && qd == 2) TL_REC(6, nunit, te0, te1, te2);
            if (lane == 0 && qd == 2) TL_REC(7, nunit, TL_NOW(), 0, 0);
        }
        if (pend) {  // the last unit's read-out: no next unit to carry it
            if (!pend_ready) {
                mbar_wait(bar.o_done + ((gt - 1) & 1), ((gt - 1) >> 1) & 1);
                if (pend_two) mbar_wait(bar.o_done + ((gt - 2) & 1), ((gt - 2) >> 1) & 1);
                tc_fence_after();
            }
            while (pend_chunk < DV / 128)
                store_block(pend_chunk++, pend_b, 0, pend_up, pend_bl, pend_two, false,
                            red + 192 + pend_up * 48);
        }
    }
    tc_fence_before();
    __syncthreads();
#ifdef SPD_TIMELINE
    if (threadIdx.x == 0 && p.tl && blockIdx.x < 512) {
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        long long* _r = p.tl + 8 * (8 * 512 + blockIdx.x);
        _r[0] = 8; _r[1] = blockIdx.x; _r[2] = (long long)g_start; _r[3] = (long long)g_end; _r[4] = smid();
    }
#endif
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, TM_COLS);
    }
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

bool spd_mla_tc_ok(const semipd_pool* p, int Hq) {
    const auto& c = p->cfg;
    return c.dtype == SEMIPD_BF16 && c.kv_shared && c.num_kv_heads == 1 && c.head_dim_k == DK &&
           c.head_dim_v == DV && Hq <= NH && c.block_size == PAGE && p->have_mla_tc_maps;
}

size_t spd_mla_tc_ws_bytes(int B, int max_ctx) {
    // split partials only (see SpdWs); any batch b <= B may be launched with this workspace,
    // and small batches split more: size for the largest b x S_max(b)
    size_t best = 0;
    for (int b = 1; b <= (B > 0 ? B : 1); ++b) {
        const size_t need = spd_ws_partial_bytes((size_t)b * NH, max_splits(max_ctx, fill_splits(b)), DV);
        if (need > best) best = need;
    }
    return best;
}

semipd_status spd_launch_decode_mla_tc(semipd_pool_t pool, int layer, const void* q,
                                       const void* k_new, const int* req_ids, const int* ctx_lens,
                                       int batch, int max_ctx_len, int Hq, float scale, void* out,
                                       int out_head_major, void* workspace, size_t ws_bytes,
                                       int budget, int* status_dev, cudaStream_t st) {
    const int S_fill = fill_splits(batch);
    const int S_max = max_splits(max_ctx_len, S_fill);
    SpdWs w;
    if (!spd_ws_carve(workspace, ws_bytes, batch, (size_t)batch * NH, S_max, DV, &w))
        return SEMIPD_ERR_INVALID;
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) return SEMIPD_ERR_INVALID;
    // Q [B][Hq][576] as (64 cols, Hq heads, 9 column blocks, B): box lands [cb][16 rows][128 B];
    // rows >= Hq are out of range and zero-filled by TMA
    CUtensorMap qmap;
    {
        const uint64_t dims[4] = {64, (uint64_t)Hq, NCB, (uint64_t)batch};
        const uint64_t strides[3] = {DK * 2, 128, (uint64_t)Hq * DK * 2};
        const uint32_t box[4] = {64, NH, NCB, 1};
        if (!spd_encode_tiled_4d(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(q), dims,
                                 strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    TcParams prm;
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
    prm.MBR = pool->cfg.max_blocks_per_req;
    prm.N_B = pool->cfg.num_blocks;
    prm.S_max = S_max;
    prm.S_fill = S_fill;
    prm.n_units = batch * S_max;
    prm.sorted = (SPD_MLA_SORT && prm.n_units <= SORT_CAP && S_max <= 32) ? 1 : 0;
    prm.out_head_major = out_head_major;
    prm.G = Hq;
    prm.scale_log2 = scale * LOG2E;
    prm.trace = spd_trace(pool);
    prm.tl = reinterpret_cast<long long*>(pool->timeline);
    prm.tl_ctr = pool->timeline_ctr;
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(decode_mla_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_BYTES) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr = true;
    }
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    const cudaError_t le = spd_launch_pdl(decode_mla_tc_kernel, dim3(grid), dim3(NTHREADS), SMEM_BYTES, st,
                                          pool->mla_lo[layer], pool->mla_hi[layer], qmap, prm);
    pool->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
