// prefill_sm100.cu — chunked causal GQA prefill attention on 5th-gen tensor cores
// (tcgen05.mma, accumulators in TMEM, operands staged by TMA), over the paged KV
// pool (P:184 prefill writes K/V; P:229 paged access; P:355 GQA kernels for both
// phases; P:365 chunked prefill).
//
// Tile: 128 rows = the G q heads of kv head g x (128 / G) tokens (row r = token r / G,
// head g*G + r % G), so every K/V tile is staged once for all G heads (GQA packing).
// Work unit: (request i, PAIR of consecutive q tiles A, B, kv head g); A and B share
// every K/V tile.  Units run longest-first (LPT: last pairs first) from a dynamic
// work counter over a persistent grid capped to the prefill SM budget.
//
// Warp roles (384 threads, 1 CTA / SM; setmaxnreg moves registers to the softmax):
//   warp 0      unit fetch, Q_A + Q_B tiles, K tiles (TMA)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, in the order
//               S_A(0) S_B(0) | PV_A(j) S_A(j+1) PV_B(j) S_B(j+1) | ...  so each softmax
//               warpgroup works while the tensor core serves the other tile; each PV runs
//               as two K = 64 halves released separately by the softmax
//               (S = Q K^T: SS, M = N = 128, K = 8 x 16; O += P V: TS, P from TMEM,
//               V MN-major from smem)
//   warp 2      V tiles (TMA)
//   warps 4-7   softmax warpgroup of tile A, warps 8-11 of tile B; one thread per row:
//               tcgen05.ld S, causal mask, online softmax in the log2 domain with packed
//               f32x2 math (exact running max; O rescaled in TMEM when it grows - safe
//               without a wait because S_t(j)'s commit implies PV_t(j-1) completed),
//               P (bf16) written back over S with tcgen05.st; epilogue O / l -> global.
// Prefix kv tiles (keys < P) are gathered from the paged pool as (128 / box_rows) page
// boxes per 64-column half; chunk kv tiles (the request's own new keys) come from
// k_new / v_new (one 32 KiB box per tile).
// TMEM columns: S_A [0,128), S_B [128,256), O_A [256,384), O_B [384,512).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int HD = 128;
constexpr int BM = 128;   // rows per tile
constexpr int BN = 128;   // keys per kv tile
constexpr int NT = 384;
constexpr uint32_t TILE_BYTES = BM * HD * 2;    // 32 KiB
constexpr uint32_t HALF_BYTES = TILE_BYTES / 2; // 16 KiB (64 columns)
constexpr float LOG2E = 1.4426950408889634f;

// The PV MMA of a tile runs in kPvParts K-slices, each released by the softmax as soon as
// its P columns are in TMEM (the first slices overlap the softmax's remaining exps)
#ifndef SPD_PV_PARTS
#define SPD_PV_PARTS 4
#endif
constexpr int kPvParts = SPD_PV_PARTS;
static_assert(kPvParts == 1 || kPvParts == 2 || kPvParts == 4, "PV parts");


struct PUnit {
    // i < 0: no more work.  t0: first chunk row of tile A (tile B starts at t0 + TQ);
    // tv[t]: valid rows (tokens) of tile t; P: cached prefix; np: prefix kv tiles;
    // nkv[t] = np + chunk kv tiles tile t needs (nkv[0] <= nkv[1]); qrow0: global row of
    // chunk row t0; crow0: global row of the request's first chunk row.
    int i, g, t0, P, np, qrow0, crow0, btrow;
    int tv[2], nkv[2];
};

struct PrefillParams {
    const int* cu;          // [n+1]
    const int* req_ids;     // [n]
    const int* prefix;      // [n]
    const int* bt;
    __nv_bfloat16* out;
    int* status;
    unsigned long long* span;  // semipd_set_spans record of this launch (or null)
    unsigned* sched;
    int n, T, Hq, Hkv, G, TQ, pairs_max, n_units, lg_bs, box_rows, MBR, N_B, out_head_major;
    int write_kv;  // 0: the chunk's K/V rows are already in the pool (RoPE pre-pass wrote them)
    // TP head all-gather fused into the epilogue: full tiles take the direct
    // 16-byte-store epilogue and every output vector also goes to each peer's gathered buffer
    // (peer-mapped, offset to this rank's head slice)
    __nv_bfloat16* peers[SEMIPD_MAX_PEERS - 1];
    int n_peers;
    const uint4* k_new;     // chunk K / V rows [T][Hkv][128] (fused pool write, warp 3)
    const uint4* v_new;
    unsigned char* k_pool;  // this layer's K / V pages
    unsigned char* v_pool;
    float scale_log2;
    float scale_log2_pre;  // prefix tiles: FP8 pools stage value(code) of K, so k_scale enters here
    SpdTrace trace;
    long long* tl;  // SPD_TIMELINE builds only: phase clock64 stamps of CTA 0
    int* tl_ctr;
};

#ifdef SPD_TIMELINE
// record slot = kind * 1024 + idx (plain stores, no atomics: keeps the pipeline unperturbed)
#define TL_REC(a, b, c, d, e)                                                              \
    do {                                                                                   \
        if (p.tl && blockIdx.x == 0 && (b) < 1024) {                                       \
            long long* _r = p.tl + 8 * ((a) * 1024 + (b));                                 \
            _r[0] = a; _r[1] = b; _r[2] = c; _r[3] = d; _r[4] = e;                         \
        }                                                                                  \
    } while (0)
#define TL_NOW() clock64()
#define TL_EXTRA(a, b, f, v)                                                               \
    do {                                                                                   \
        if (p.tl && blockIdx.x == 0 && (b) < 1024) p.tl[8 * ((a) * 1024 + (b)) + (f)] = (v); \
    } while (0)
#else
#define TL_EXTRA(a, b, f, v) do { } while (0)
#define TL_REC(a, b, c, d, e) do { } while (0)
#define TL_NOW() 0LL
#endif

struct Smem {
    // operand tiles first (1024-aligned by construction)
    unsigned char q[2][TILE_BYTES];
    unsigned char k[2][TILE_BYTES];
    unsigned char v[2][TILE_BYTES];
    unsigned char ostage[2][HALF_BYTES];  // per q tile: epilogue staging for TMA stores (64 cols)
    uint64_t q_full, q_empty, q_issued;  // q_issued: V loads of a unit queue behind its Q
    uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
    uint64_t s_full[2], p_full[2][kPvParts];  // per q tile; p_full[t][h]: P part h in TMEM
    uint64_t o_full[2], o_empty[2];  // per q tile
    uint64_t ufull[2], uempty[2];
    PUnit units[2];
    uint32_t tmem_base;
};

// Which exp2 pairs of each 32-column S block run on the FMA pipe instead of MUFU (bit i =
// columns 2i, 2i+1).  MUFU.EX2 is 16/clk/SM on B200 (measured, scripts/probe_mufu.cu), so a
// 128 x 128 S tile costs 1024 MUFU cycles, as much as the tile's QK + PV tensor work; moving a
// fraction of the exps to a degree-3 polynomial on the FMA pipe shortens the softmax that sits
// on the per-tile critical path (softmax -> PV -> next S).
#ifndef SPD_POLY_MASK
#define SPD_POLY_MASK 0x1111u
#endif
constexpr uint32_t kPolyMask = SPD_POLY_MASK;

// independent FMNMX3 chains of the row max (latency-bound: 64 three-input maxes per row)
#ifndef SPD_MAX_CHAINS
#define SPD_MAX_CHAINS 4
#endif
constexpr int kMaxChains = SPD_MAX_CHAINS;

// L2 policy of the chunk K/V tile loads (each is re-read by all later q-tile pairs of its
// request and kv head); 0 = evict_normal (evict_last measured no better in the co-run: the
// decode stream is already evict_first)
#ifndef SPD_PRE_L2
#define SPD_PRE_L2 0
#endif
constexpr int kPreL2 = SPD_PRE_L2;

// Epilogue of full tiles: 1 = coalesced st.global from a swizzled smem staging, 0 = TMA store
#ifndef SPD_EPI_DIRECT
#define SPD_EPI_DIRECT 0
#endif
constexpr bool kEpiDirect = SPD_EPI_DIRECT != 0;


// MMA issue from the whole converged warp (elect.sync inside the asm: descriptors stay in
// uniform registers, ~2x the issue rate of a lane-0 branch) or from lane 0
#ifndef SPD_MMA_WARP
#define SPD_MMA_WARP 1
#endif
constexpr bool kMmaWarp = SPD_MMA_WARP != 0;
#if SPD_MMA_WARP
#define MMA_SS umma_ss_warp
#define MMA_TS umma_ts_warp
#define MMA_COMMIT umma_commit_warp
#else
#define MMA_SS umma_ss
#define MMA_TS umma_ts
#define MMA_COMMIT umma_commit
#endif

__device__ __forceinline__ uint64_t kmajor_desc(uint32_t addr) {
    return umma_desc_sw128(addr, 16, 1024);
}

// PEERS: the epilogue also stores every output vector to the peers' gathered buffers (the
// fused TP gather).  A separate instantiation, because compiling the peer stores into the
// one kernel cost the plain path 1-3 % (measured A/B, scripts/gpu_prefill_ab.sh)
template <bool PEERS>
__global__ void __launch_bounds__(NT, 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap qmap,
                      const __grid_constant__ CUtensorMap kmap,
                      const __grid_constant__ CUtensorMap vmap,
                      const __grid_constant__ CUtensorMap kcmap,
                      const __grid_constant__ CUtensorMap vcmap,
                      const __grid_constant__ CUtensorMap omap, PrefillParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    Smem& sm = *reinterpret_cast<Smem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = (int)warp_id();
    const int lane = (int)lane_id();
    const uint64_t kv_pol = l2_policy(kPreL2);  // chunk K/V: re-read by every later q pair

    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_empty, 1);
        mbar_init(&sm.q_issued, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], 1);
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], 1);
            mbar_init(&sm.s_full[s], 1);
            for (int h = 0; h < kPvParts; ++h) mbar_init(&sm.p_full[s][h], 128);
            mbar_init(&sm.o_full[s], 1);
            mbar_init(&sm.o_empty[s], 128);
            mbar_init(&sm.ufull[s], 1);
            mbar_init(&sm.uempty[s], 1 + 8 + 1);  // MMA warp + 8 softmax warps + V producer
        }
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(1, (int)smid(), (int)blockIdx.x, 1 /* kernel kind: tcgen05 prefill */);
        }
    }
#ifdef SPD_TIMELINE
    unsigned long long gt_start = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_start));
    int tl_units = 0;
#endif
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (sched counters, pool)
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = sm.tmem_base;

    if (warp < 4) {
    // ====================== warpgroup 0: TMA producers + MMA issuer ======================
    setmaxnreg_dec<72>();
    if (warp == 0 || warp == 2) {
        // ============================ TMA producers ============================
        const int kv = warp == 2;
        const CUtensorMap* pmap = kv ? &vmap : &kmap;
        const CUtensorMap* cmap = kv ? &vcmap : &kcmap;
        if (lane == 0) {
            if (!kv) tma_prefetch_desc(&qmap);
            tma_prefetch_desc(pmap);
            tma_prefetch_desc(cmap);
        }
        const int oob_z = p.N_B * p.Hkv;
        const int nbox_tile = BN / p.box_rows;  // page boxes per 64-column half of a tile
        const int bs_mask = (1 << p.lg_bs) - 1;
        int kvit = 0, nunit = 0;
        for (;;) {
            const int us = nunit & 1;
            PUnit d;
            d.i = -1;
            if (!kv) {
                int u = 0;
                if (lane == 0) u = (int)atomicAdd(p.sched, 1u);
                u = __shfl_sync(0xffffffffu, u, 0);
                if (u < p.n_units) {
                    const int per_pair = p.n * p.Hkv;
                    const int pair = p.pairs_max - 1 - u / per_pair;  // LPT: last pairs first
                    d.i = (u / p.Hkv) % p.n;
                    d.g = u % p.Hkv;
                    const int c0 = __ldg(p.cu + d.i), c1 = __ldg(p.cu + d.i + 1);
                    const int C = c1 - c0;
                    d.t0 = pair * 2 * p.TQ;
                    if (d.t0 >= C) continue;  // pair past this request's chunk (warp-uniform)
                    d.tv[0] = min(p.TQ, C - d.t0);
                    d.tv[1] = max(0, min(p.TQ, C - d.t0 - p.TQ));
                    d.P = __ldg(p.prefix + d.i);
                    d.np = (d.P + BN - 1) / BN;
                    d.nkv[0] = d.np + (d.t0 + d.tv[0] - 1) / BN + 1;
                    d.nkv[1] = d.tv[1] > 0 ? d.np + (d.t0 + p.TQ + d.tv[1] - 1) / BN + 1 : d.nkv[0];
                    d.qrow0 = c0 + d.t0;
                    d.crow0 = c0;
                    d.btrow = __ldg(p.req_ids + d.i);
                }
                if (lane == 0) {
                    mbar_wait(&sm.uempty[us], ((nunit >> 1) & 1) ^ 1);
                    sm.units[us] = d;
                    mbar_arrive(&sm.ufull[us]);
                }
                __syncwarp();
            } else {
                mbar_wait(&sm.ufull[us], (nunit >> 1) & 1);
                d = sm.units[us];
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.uempty[us]);
            }
            if (d.i < 0) {  // no more units: the next kernel on the stream may be scheduled
                pdl_trigger();
                break;
            }
            if (!kv && lane == 0) {
                // Q tiles A and B (rows = tokens x G heads of kv head g)
                [[maybe_unused]] const long long tq0 = TL_NOW();
                mbar_wait(&sm.q_empty, (nunit & 1) ^ 1);
                TL_REC(30, nunit, tq0, TL_NOW(), 0);
                // one 64 KiB box: (64 cols, G heads, 2 TQ tokens, 2 halves) lands as
                // [half][tile A rows | tile B rows][128 B]
                mbar_arrive_expect_tx(&sm.q_full, 2 * TILE_BYTES);
                tma_load_4d(sm.q[0], &qmap, &sm.q_full, 0, d.g * p.G, d.qrow0, 0);
                mbar_arrive(&sm.q_issued);
            }
            if (kv && lane == 0) mbar_wait(&sm.q_issued, nunit & 1);  // keep V behind this Q
            ++nunit;
            const int* btr = p.bt + (size_t)d.btrow * p.MBR;
            const int last_page = (d.P - 1) >> p.lg_bs;  // prefix pages only
            const int nbox = d.np * nbox_tile;
            auto lookup = [&](int bi) -> int {  // raw block id; -2 = beyond the prefix
                const int page = (bi * p.box_rows) >> p.lg_bs;
                if (bi >= nbox || page > last_page) return -2;
                return page < p.MBR ? __ldg(btr + page) : -1;
            };
            int zc = lookup(lane), zn = lookup(32 + lane);
            const int nkv = d.nkv[1];
            for (int j = 0; j < nkv; ++j, ++kvit) {
                const int st = kvit & 1;
                const uint32_t ph = ((kvit >> 1) & 1) ^ 1;
                uint64_t* emp = kv ? &sm.v_empty[st] : &sm.k_empty[st];
                uint64_t* ful = kv ? &sm.v_full[st] : &sm.k_full[st];
                unsigned char* dst = kv ? sm.v[st] : sm.k[st];
                if (lane == 0) {
                    mbar_wait(emp, ph);
                    mbar_arrive_expect_tx(ful, TILE_BYTES);
                }
                if (j < d.np) {
                    const int bb0 = j * nbox_tile;
                    if (bb0 > 0 && (bb0 & 31) == 0) {
                        zc = zn;
                        zn = lookup(bb0 + 32 + lane);
                    }
                    for (int b = 0; b < nbox_tile; ++b) {
                        const int blk = __shfl_sync(0xffffffffu, zc, (bb0 & 31) + b);
                        if (lane == 0) {
                            int z = oob_z;
                            if (blk >= 0 && blk < p.N_B) z = blk * p.Hkv + d.g;
                            else if (blk != -2 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                            const int r = b * p.box_rows;
                            const int y = (j * BN + r) & bs_mask;
                            tma_load_3d(dst + r * 128, pmap, ful, 0, y, z);
                            tma_load_3d(dst + HALF_BYTES + r * 128, pmap, ful, 64, y, z);
                        }
                    }
                } else if (lane == 0) {
                    // one 32 KiB box (64 cols, 1 head, 128 rows, 2 halves) -> [half][rows][128 B]
                    tma_load_4d_hint(dst, cmap, ful, 0, d.g, d.crow0 + (j - d.np) * BN, 0, kv_pol);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // ================================ MMA issuer ================================
        if (kMmaWarp || lane == 0) {
            const uint32_t idesc_s = umma_idesc_bf16_f32(BM, BN, 0);
            const uint32_t idesc_o = umma_idesc_bf16_f32(BM, HD, 1);
            int kvit = 0, nunit = 0;
            int cnt_a = 0, cnt_b = 0;  // P tiles consumed so far per q tile (p_full phases)
            for (;;) {
                const int us = nunit & 1;
                mbar_wait(&sm.ufull[us], (nunit >> 1) & 1);
                const PUnit d = sm.units[us];
                if (kMmaWarp) __syncwarp();
                if (!kMmaWarp || lane == 0) mbar_arrive(&sm.uempty[us]);
                if (d.i < 0) break;
                [[maybe_unused]] const long long tq1 = TL_NOW();
                mbar_wait(&sm.q_full, nunit & 1);
                TL_REC(31, nunit, tq1, TL_NOW(), d.nkv[1]);
                tc_fence_after();
                const int nA = d.nkv[0], nB = d.nkv[1];
                auto issue_s = [&](int t, int it) {  // S_t = Q_t K^T (K stage of kv tile it)
                    // Q smem: [half][tile A | tile B][128 rows][128 B]; K: [half][128 rows]
                    const uint32_t q_addr = smem_u32(sm.q[0]) + (uint32_t)t * HALF_BYTES;
                    const uint32_t k_addr = smem_u32(sm.k[it & 1]);
                    const uint32_t d_tmem = tmem + (uint32_t)(t * BN);
#if SPD_MMA_WARP
                    // descriptors as (low, high) words: the K16 offsets are 32-bit adds to the low
                    // word on the uniform datapath (umma_ss_warp2)
                    const uint32_t qd = desc_lo(q_addr, 16), kd = desc_lo(k_addr, 16);
#pragma unroll
                    for (int kk = 0; kk < HD / 16; ++kk) {
                        const uint32_t koff = (kk >> 2) * HALF_BYTES + (kk & 3) * 32;
                        const uint32_t qoff = (kk >> 2) * TILE_BYTES + (kk & 3) * 32;
                        umma_ss_warp2(d_tmem, qd + (qoff >> 4), DESC_HI_SBO1K, kd + (koff >> 4), DESC_HI_SBO1K,
                                      idesc_s, kk > 0 ? 1u : 0u);
                    }
#else
#pragma unroll
                    for (int kk = 0; kk < HD / 16; ++kk) {
                        const uint32_t koff = (kk >> 2) * HALF_BYTES + (kk & 3) * 32;
                        const uint32_t qoff = (kk >> 2) * TILE_BYTES + (kk & 3) * 32;
                        MMA_SS(d_tmem, kmajor_desc(q_addr + qoff), kmajor_desc(k_addr + koff),
                                idesc_s, kk > 0 ? 1u : 0u);
                    }
#endif
                    MMA_COMMIT(&sm.s_full[t]);
                };
                auto issue_pv = [&](int t, int& cnt, int it, bool first) {  // O_t += P_t V
                    // in two K = 64 halves: the first starts while the softmax still
                    // computes the exps of keys [64, 128) (p_full[t][0] is armed mid-tile)
                    const uint32_t v_addr = smem_u32(sm.v[it & 1]);
                    const uint32_t p_tmem = tmem + (uint32_t)(t * BN);
                    const uint32_t o_tmem = tmem + 256u + (uint32_t)(t * HD);
#pragma unroll
                    for (int hf = 0; hf < kPvParts; ++hf) {
                        mbar_wait(&sm.p_full[t][hf], cnt & 1);
                        tc_fence_after();
#pragma unroll
                        for (int kk = hf * 8 / kPvParts; kk < (hf + 1) * 8 / kPvParts; ++kk) {
#if SPD_MMA_WARP
                            umma_ts_warp2(o_tmem, p_tmem + (uint32_t)(kk * 8), desc_lo(v_addr, HALF_BYTES) + kk * (2048 >> 4),
                                          DESC_HI_SBO1K, idesc_o, (first && kk == 0) ? 0u : 1u);
#else
                            const uint64_t bdesc = umma_desc_sw128(v_addr + kk * 2048, HALF_BYTES, 1024);
                            MMA_TS(o_tmem, p_tmem + (uint32_t)(kk * 8), bdesc, idesc_o,
                                    (first && kk == 0) ? 0u : 1u);
#endif
                        }
                    }
                    ++cnt;
                };
                auto wait_full = [&](uint64_t* bars, int it) {
                    mbar_wait(&bars[it & 1], (it >> 1) & 1);
                    tc_fence_after();
                };
                const int it0 = kvit;
                // prologue: S_A(0), S_B(0)
                wait_full(sm.k_full, it0);
                issue_s(0, it0);
                issue_s(1, it0);
                MMA_COMMIT(&sm.k_empty[it0 & 1]);
                if (nB == 1) MMA_COMMIT(&sm.q_empty);
                for (int j = 0; j < nB; ++j) {
                    const int it = it0 + j;
                    wait_full(sm.v_full, it);
                    if (j < nA) {
                        if (j == 0) mbar_wait(&sm.o_empty[0], (nunit & 1) ^ 1);
                        issue_pv(0, cnt_a, it, j == 0);
                        if (j == nA - 1) MMA_COMMIT(&sm.o_full[0]);
                    }
                    const bool more = j + 1 < nB;
                    if (more) wait_full(sm.k_full, it + 1);
                    if (j + 1 < nA) issue_s(0, it + 1);
                    if (j == 0) mbar_wait(&sm.o_empty[1], (nunit & 1) ^ 1);
                    issue_pv(1, cnt_b, it, j == 0);
                    MMA_COMMIT(&sm.v_empty[it & 1]);
                    if (j == nB - 1) MMA_COMMIT(&sm.o_full[1]);
                    if (more) {
                        issue_s(1, it + 1);
                        MMA_COMMIT(&sm.k_empty[(it + 1) & 1]);
                        if (j + 1 == nB - 1) MMA_COMMIT(&sm.q_empty);
                    }
                }
                kvit = it0 + nB;
                ++nunit;
#ifdef SPD_TIMELINE
                tl_units += nB;
#endif
            }
        }
    } else {
        // ============ warp 3: the chunk's K/V rows -> pool pages, fused ============
        // Rows are split evenly over the CTAs; the attention itself reads chunk K/V from
        // k_new / v_new and prefix pages written by earlier calls, so nothing in this launch
        // reads what this warp writes (the next kernel on the stream does).
        const int r0 = (int)((long long)p.T * blockIdx.x / gridDim.x);
        const int r1 = p.write_kv ? (int)((long long)p.T * (blockIdx.x + 1) / gridDim.x) : r0;
        if (r0 < r1) {
            int i = 0, hi = p.n - 1;  // last request with cu[i] <= r0
            while (i < hi) {
                const int mid = (i + hi + 1) >> 1;
                if (__ldg(p.cu + mid) <= r0) i = mid; else hi = mid - 1;
            }
            int c_lo = __ldg(p.cu + i), c_hi = __ldg(p.cu + i + 1);
            int pre = __ldg(p.prefix + i);
            const int* btr = p.bt + (size_t)__ldg(p.req_ids + i) * p.MBR;
            const int bs_mask = (1 << p.lg_bs) - 1;
            const int c = lane & 15;         // 16-byte chunk of a 256-byte head row
            for (int row = r0; row < r1; ++row) {
                while (row >= c_hi) {
                    ++i;
                    c_lo = c_hi;
                    c_hi = __ldg(p.cu + i + 1);
                    pre = __ldg(p.prefix + i);
                    btr = p.bt + (size_t)__ldg(p.req_ids + i) * p.MBR;
                }
                const int pos = pre + row - c_lo;
                const int page = pos >> p.lg_bs;
                const int blk = page < p.MBR ? __ldg(btr + page) : -1;
                if (blk < 0 || blk >= p.N_B) {
                    if (lane == 0 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                    continue;
                }
#pragma unroll 1
                for (int g0 = 0; g0 < p.Hkv; g0 += 8) {  // 8 heads per pass, 4 per half-warp
                    uint4 kv[2][4];
#pragma unroll
                    for (int gg = 0; gg < 4; ++gg) {
                        const int g = g0 + (lane >> 4) + 2 * gg;
                        if (g < p.Hkv) {
                            const size_t src = ((size_t)row * p.Hkv + g) * 16 + c;
                            kv[0][gg] = __ldg(p.k_new + src);
                            kv[1][gg] = __ldg(p.v_new + src);
                        }
                    }
#pragma unroll
                    for (int gg = 0; gg < 4; ++gg) {
                        const int g = g0 + (lane >> 4) + 2 * gg;
                        if (g < p.Hkv) {
                            const size_t dst = (((size_t)blk * p.Hkv + g) * (bs_mask + 1) + (pos & bs_mask)) * 16 + c;
                            reinterpret_cast<uint4*>(p.k_pool)[dst] = kv[0][gg];
                            reinterpret_cast<uint4*>(p.v_pool)[dst] = kv[1][gg];
                        }
                    }
                }
            }
        }
    }
    } else {
        // ============================ softmax warpgroups ============================
        setmaxnreg_inc<216>();
        const int t = (warp - 4) >> 2;         // q tile A (0) or B (1)
        const int q4 = warp & 3;               // TMEM lane quarter
        const int r = q4 * 32 + lane;          // tile row
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        const uint32_t s_tmem = tmem + lane_base + (uint32_t)(t * BN);
        const uint32_t o_tmem = tmem + lane_base + 256u + (uint32_t)(t * HD);
        [[maybe_unused]] int tl_tile = 0;  // SPD_TIMELINE record index
        int cnt = 0, nunit = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(&sm.ufull[us], (nunit >> 1) & 1);
            const PUnit d = sm.units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.uempty[us]);
            if (d.i < 0) break;
            const int tok = r / p.G;
            const int trel = d.t0 + t * p.TQ + tok;  // chunk-relative token index of this row
            const int nkv = d.nkv[t];
            float m = -INFINITY;
            uint64_t l2 = f2(0.f, 0.f);
            for (int j = 0; j < nkv; ++j, ++cnt) {
                [[maybe_unused]] const long long ts0 = TL_NOW();
                mbar_wait(&sm.s_full[t], cnt & 1);
                [[maybe_unused]] const long long ts1 = TL_NOW();
                tc_fence_after();
                uint32_t sr[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(s_tmem + c * 32, sr[c]);
                tmem_wait_ld();
                [[maybe_unused]] const long long ts2 = TL_NOW();
                // prefix tile: keys j*BN + c must be < P; chunk tile: chunk-relative key
                // (j - np)*BN + c must be <= this row's token (causal, bottom-right aligned)
                const int lim = j < d.np ? d.P - 1 - j * BN : trel - (j - d.np) * BN;
                if (lim < BN - 1) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (c * 32 + e > lim) sr[c][e] = __float_as_uint(-INFINITY);
                }
                // row max: kMaxChains independent FMNMX3 chains over the 128 columns instead of
                // one 64-deep dependent chain on the softmax critical path
                float mxc[kMaxChains];
#pragma unroll
                for (int k = 0; k < kMaxChains; ++k) mxc[k] = -INFINITY;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const int k = (c * 16 + e / 2) % kMaxChains;
                        mxc[k] = fmax3(mxc[k], __uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1]));
                    }
#pragma unroll
                for (int w = kMaxChains / 2; w >= 1; w /= 2)
#pragma unroll
                    for (int k = 0; k < w; ++k) mxc[k] = fmaxf(mxc[k], mxc[k + w]);
                const float mx = mxc[0];
                const float tsc = j < d.np ? p.scale_log2_pre : p.scale_log2;
                const float mtrue = fmaxf(m, mx * tsc);  // scale > 0: max commutes
                // lazy rescale (R21): the reference max m moves only when the row max
                // exceeds it by > 8 (log2 units), so P <= 2^8 and nearly every tile skips the O
                // round trip through TMEM (the exact-max rescale ran on most tiles: ~10 % of the
                // kernel).  O_t(j-1) is complete when it is rescaled: S_t(j) was issued after
                // PV_t(j-1) and its commit tracks both.
                const bool move = j == 0 || mtrue > m + 8.f;
                if (j > 0 && __any_sync(0xffffffffu, move)) {
                    const float alpha = move ? fast_exp2(m - mtrue) : 1.f;
                    const uint64_t a2 = f2(alpha, alpha);
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(o_tmem + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; e += 2) {
                            float lo, hi;
                            f2_split(fmul2(f2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), a2),
                                     lo, hi);
                            o[e] = __float_as_uint(lo);
                            o[e + 1] = __float_as_uint(hi);
                        }
                        tmem_st32(o_tmem + c * 32, o);
                    }
                    l2 = fmul2(l2, a2);
                }
                if (move) m = mtrue;
                [[maybe_unused]] const long long ts3 = TL_NOW();
                // P = exp2(s * scale - m) (bf16) over the S columns [0, 64); the row sum adds
                // the bf16-rounded P the PV MMA consumes (R21) with mixed-precision FHADD.BF16
                // (one instruction per element, half-register operand), in four chains
                const uint64_t nm2 = f2(-m, -m);
                const uint64_t sc2 = f2(tsc, tsc);
                float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 4; ++c) {  // 32 S columns -> 16 packed P columns
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t x2 = ffma2(f2(__uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1])),
                                                  sc2, nm2);
                        float p0, p1;
                        if ((kPolyMask >> (e >> 1)) & 1u) {
                            f2_split(exp2_poly3(x2), p0, p1);
                        } else {
                            float x0, x1;
                            f2_split(x2, x0, x1);
                            p0 = fast_exp2(x0);
                            p1 = fast_exp2(x1);
                        }
                        const uint32_t pp = pack_bf16(p0, p1);
                        pk[e / 2] = pp;
                        add_bf16x2_f32(ls[2 * (c & 1)], ls[2 * (c & 1) + 1], pp);
                    }
                    tmem_st16(s_tmem + (uint32_t)(c * 16), pk);
                    if ((c + 1) % (4 / kPvParts) == 0) {
                        // release this part of P to the PV MMA
                        tmem_wait_st();
                        tc_fence_before();
                        mbar_arrive(&sm.p_full[t][(c + 1) / (4 / kPvParts) - 1]);
                    }
                }
                l2 = fadd2(l2, f2(ls[0] + ls[2], ls[1] + ls[3]));
                [[maybe_unused]] const long long ts4 = TL_NOW();
                if (lane == 0 && q4 == 0) {
                    TL_REC(t, tl_tile, ts0, ts1, TL_NOW());
                    TL_EXTRA(t, tl_tile, 5, ts2);
                    TL_EXTRA(t, tl_tile, 6, ts3);
                    TL_EXTRA(t, tl_tile, 7, ts4);
                }
                ++tl_tile;
            }
            // ---- epilogue: O / l -> bf16 -> global
            [[maybe_unused]] const long long te0 = TL_NOW();
            mbar_wait(&sm.o_full[t], nunit & 1);
            [[maybe_unused]] const long long te1 = TL_NOW();
            tc_fence_after();
            float la, lb;
            f2_split(l2, la, lb);
            const float inv = 1.f / (la + lb);
            const bool valid = tok < d.tv[t];
            const int hq = d.g * p.G + (r % p.G);
            const int trow = d.qrow0 + t * p.TQ + tok;
            bool o_released = false;
            if (!PEERS && kEpiDirect && d.tv[t] == p.TQ) {
                // full tile: O -> registers (O's TMEM is released to the next unit's PV at
                // once), then per 64-column half: rows -> swizzled smem staging -> coalesced
                // 16-byte global stores, 8 threads per 128-byte row segment (no TMA store: its
                // smem read queued behind the next unit's Q / K / V loads in the TMA unit)
                uint32_t o[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(o_tmem + c * 32, o[c]);
                tmem_wait_ld();
                tc_fence_before();
                mbar_arrive(&sm.o_empty[t]);
                o_released = true;
                unsigned char* stg = sm.ostage[t];
                unsigned char* outb = reinterpret_cast<unsigned char*>(p.out);
                const int lgG = __ffs(p.G) - 1;  // G divides 128: a power of two
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    if (hh) named_bar_sync(2 + t, 128);  // half 0 copied out of the staging
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        const uint32_t* oo = &o[2 * hh + (c8 >> 2)][(c8 & 3) * 8];
                        uint4 v;
                        v.x = pack_bf16(__uint_as_float(oo[0]) * inv, __uint_as_float(oo[1]) * inv);
                        v.y = pack_bf16(__uint_as_float(oo[2]) * inv, __uint_as_float(oo[3]) * inv);
                        v.z = pack_bf16(__uint_as_float(oo[4]) * inv, __uint_as_float(oo[5]) * inv);
                        v.w = pack_bf16(__uint_as_float(oo[6]) * inv, __uint_as_float(oo[7]) * inv);
                        *reinterpret_cast<uint4*>(stg + r * 128 + ((c8 ^ (r & 7)) << 4)) = v;
                    }
                    named_bar_sync(2 + t, 128);
#pragma unroll
                    for (int it = 0; it < 8; ++it) {
                        const int row = it * 16 + (r >> 3), c = r & 7;
                        const uint4 v = *reinterpret_cast<const uint4*>(stg + row * 128 + ((c ^ (row & 7)) << 4));
                        const int rt = d.qrow0 + t * p.TQ + (row >> lgG);
                        const int rh = d.g * p.G + (row & (p.G - 1));
                        const size_t rowoff = p.out_head_major ? (size_t)rh * p.T + rt : (size_t)rt * p.Hq + rh;
                        *reinterpret_cast<uint4*>(outb + rowoff * (HD * 2) + hh * 128 + c * 16) = v;
                    }
                }
            } else if (d.tv[t] == p.TQ) {
                // full tile: rows -> swizzled smem staging -> one TMA store per 64-column half
                // (per-thread 16-byte stores to 256-byte-strided rows were ~4k cycles and held
                // up the next unit's Q load in the SM's memory path)
                const int srow = p.out_head_major ? (r % p.G) * p.TQ + tok : r;
                unsigned char* stg = sm.ostage[t];
                const bool issuer = q4 == 0 && lane == 0;
                [[maybe_unused]] long long tea = 0, teb = 0;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    if (issuer) bulk_wait_group_read0();  // previous store has read the staging
                    named_bar_sync(2 + t, 128);
                    if (hh) teb = TL_NOW();
                    uint32_t o[2][32];
                    tmem_ld32(o_tmem + hh * 64, o[0]);
                    tmem_ld32(o_tmem + hh * 64 + 32, o[1]);
                    tmem_wait_ld();
                    if (!hh) tea = TL_NOW();
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        const uint32_t* oo = &o[c8 >> 2][(c8 & 3) * 8];
                        uint4 v;
                        v.x = pack_bf16(__uint_as_float(oo[0]) * inv, __uint_as_float(oo[1]) * inv);
                        v.y = pack_bf16(__uint_as_float(oo[2]) * inv, __uint_as_float(oo[3]) * inv);
                        v.z = pack_bf16(__uint_as_float(oo[4]) * inv, __uint_as_float(oo[5]) * inv);
                        v.w = pack_bf16(__uint_as_float(oo[6]) * inv, __uint_as_float(oo[7]) * inv);
                        *reinterpret_cast<uint4*>(stg + srow * 128 + ((c8 ^ (srow & 7)) << 4)) = v;
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(2 + t, 128);
                    if (PEERS && p.n_peers > 0) {
                        // fused TP gather (head-major only): the 128 threads copy the staged
                        // half out with 16-byte stores, to the local output and to every peer
                        // (the next half's barrier keeps the staging until all have read it)
                        unsigned char* outb = reinterpret_cast<unsigned char*>(p.out);
#pragma unroll
                        for (int it = 0; it < 8; ++it) {
                            const int row = it * 16 + (r >> 3), c = r & 7;
                            const uint4 v = *reinterpret_cast<const uint4*>(stg + row * 128 + ((c ^ (row & 7)) << 4));
                            const int rt = d.qrow0 + t * p.TQ + row % p.TQ;
                            const int rh = d.g * p.G + row / p.TQ;
                            const size_t bo = ((size_t)rh * p.T + rt) * (HD * 2) + hh * 128 + c * 16;
                            *reinterpret_cast<uint4*>(outb + bo) = v;
#pragma unroll
                            for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
                                if (k < p.n_peers)
                                    *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(p.peers[k]) + bo) = v;
                        }
                    } else if (issuer) {
                        if (p.out_head_major)
                            tma_store_3d(&omap, stg, hh * 64, d.qrow0 + t * p.TQ, d.g * p.G);
                        else
                            tma_store_3d(&omap, stg, hh * 64, d.g * p.G, d.qrow0 + t * p.TQ);
                        bulk_commit_group();
                    }
                }
                if (lane == 0 && q4 == 0) {
                    TL_EXTRA(10 + t, nunit, 5, tea);
                    TL_EXTRA(10 + t, nunit, 6, teb);
                    TL_EXTRA(10 + t, nunit, 7, TL_NOW());
                }
            } else {
                __nv_bfloat16* dst = p.out + (p.out_head_major
                                                  ? ((size_t)hq * p.T + trow) * HD
                                                  : ((size_t)trow * p.Hq + hq) * HD);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t o[32];
                    tmem_ld32(o_tmem + c * 32, o);
                    tmem_wait_ld();
                    if (valid) {
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            uint4 v;
                            v.x = pack_bf16(__uint_as_float(o[e + 0]) * inv, __uint_as_float(o[e + 1]) * inv);
                            v.y = pack_bf16(__uint_as_float(o[e + 2]) * inv, __uint_as_float(o[e + 3]) * inv);
                            v.z = pack_bf16(__uint_as_float(o[e + 4]) * inv, __uint_as_float(o[e + 5]) * inv);
                            v.w = pack_bf16(__uint_as_float(o[e + 6]) * inv, __uint_as_float(o[e + 7]) * inv);
                            *reinterpret_cast<uint4*>(dst + c * 32 + e) = v;
                            if (PEERS) {
#pragma unroll
                                for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
                                    if (k < p.n_peers)
                                        *reinterpret_cast<uint4*>(p.peers[k] + (dst - p.out) + c * 32 + e) = v;
                            }
                        }
                    }
                }
            }
            if (!o_released) {
                tc_fence_before();
                mbar_arrive(&sm.o_empty[t]);
            }
            if (lane == 0 && q4 == 0) TL_REC(10 + t, nunit, te0, te1, TL_NOW());
            ++nunit;
        }
        if (q4 == 0 && lane == 0) bulk_wait_group0();  // all TMA stores of this tile done
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
#ifdef SPD_TIMELINE
    // every CTA: [40, cta, globaltimer start, end, kv-tile pair steps run, smid]
    if (p.tl && warp == 1 && lane == 0 && blockIdx.x < 1024) {
        unsigned long long gt_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_end));
        long long* r = p.tl + 8 * (40 * 1024 + blockIdx.x);
        r[0] = 40; r[1] = blockIdx.x; r[2] = (long long)gt_start; r[3] = (long long)gt_end;
        r[4] = tl_units; r[5] = smid();
    }
#endif
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

bool fast_path_ok(const semipd_pool* pl, int Hq) {
    const auto& c = pl->cfg;
    if (c.dtype == SEMIPD_FP8_E4M3)  // E4M3 pages: the same kernel over bf16 staging pages (R31)
        return !c.kv_shared && c.head_dim_k == HD && c.head_dim_v == HD && Hq % c.num_kv_heads == 0 &&
               Hq / c.num_kv_heads <= 16 && BM % (Hq / c.num_kv_heads) == 0 && c.block_size == 64;
    if (c.dtype != SEMIPD_BF16 || c.kv_shared || c.head_dim_k != HD || c.head_dim_v != HD ||
        !pl->have_maps || Hq % c.num_kv_heads || (c.block_size & (c.block_size - 1)))
        return false;
    const int G = Hq / c.num_kv_heads;
    const int bs = c.block_size;
    return G >= 1 && G <= 16 && BM % G == 0 &&
           (bs == 16 || bs == 32 || bs == 64 || bs == 128);
}

}  // namespace

extern "C" semipd_status semipd_prefill_attn(
    semipd_pool_t pool, int32_t layer, const void* q, const void* k_new, const void* v_new,
    const int32_t* cu_seqlens_q, const int32_t* req_ids, const int32_t* prefix_lens, int32_t n,
    int32_t total_q, int32_t max_chunk_len, int32_t num_q_heads, float softmax_scale, void* out,
    int32_t out_head_major, int32_t sm_budget, int32_t* status_dev, semipd_stream_t s) {
    if (!pool || layer < 0 || layer >= pool->cfg.num_layers || n < 0 || total_q < 0 ||
        max_chunk_len < 0)
        return SEMIPD_ERR_INVALID;
    const auto& c = pool->cfg;
    if (num_q_heads <= 0 || num_q_heads % c.num_kv_heads) return SEMIPD_ERR_INVALID;
    if (sm_budget < -1 || sm_budget > pool->num_sms) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (status_dev && cudaMemsetAsync(status_dev, 0, sizeof(int), st) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    if (n == 0 || total_q == 0) return SEMIPD_OK;
    if (!q || !k_new || (!v_new && !c.kv_shared) || !cu_seqlens_q || !req_ids || !prefix_lens ||
        !out)
        return SEMIPD_ERR_INVALID;
    const int budget = spd_resolve_budget(pool, sm_budget, true);
    if (pool->pre_n_peers > 0 && (!out_head_major || total_q != pool->pre_peer_tokens))
        return SEMIPD_ERR_INVALID;
    if (pool->pre_n_peers > 0 &&
        (!fast_path_ok(pool, num_q_heads) || spd_mla_prefill_ok(pool, num_q_heads)))
        return SEMIPD_ERR_UNSUPPORTED;
    const bool rope = pool->rope_on;
    const bool fp8 = c.dtype == SEMIPD_FP8_E4M3;
    if (fp8) {
        // E4M3 pages (reading R31): quantised K/V write of the chunk, then the call's prefix pages
        // dequantised into the bf16 staging scratch, which the tcgen05 kernel reads as it reads a
        // bf16 pool; the chunk's own keys come from k_new / v_new (bf16) as always
        // (with RoPE set, the rotation of q / k_new in place and the quantised write of the
        // rotated rows are one pass, R28 + R31)
        if (pool->pre_n_peers > 0 || !fast_path_ok(pool, num_q_heads)) return SEMIPD_ERR_UNSUPPORTED;
        if (!pool->have_f8s_maps || n > pool->f8s_cap) return SEMIPD_ERR_INVALID;
        semipd_status r =
            rope ? spd_launch_rope_write(pool, layer, const_cast<void*>(q), const_cast<void*>(k_new),
                                         v_new, cu_seqlens_q, req_ids, prefix_lens, n, total_q,
                                         num_q_heads, status_dev, st)
                 : spd_launch_kv_write_fp8(pool, layer, k_new, v_new, cu_seqlens_q, req_ids,
                                           prefix_lens, n, total_q, status_dev, st);
        if (r == SEMIPD_OK)
            r = spd_launch_dequant_prefix(pool, layer, req_ids, prefix_lens, n, budget, status_dev, st);
        if (r != SEMIPD_OK) return r;
    } else if (rope) {
        // RoPE of q / k_new (in place) at positions prefix + t, fused with the K/V write of the
        // rotated rows (R28): the attention kernels below skip their own write
        semipd_status r = spd_launch_rope_write(pool, layer, const_cast<void*>(q),
                                                const_cast<void*>(k_new), v_new, cu_seqlens_q,
                                                req_ids, prefix_lens, n, total_q, num_q_heads,
                                                status_dev, st);
        if (r != SEMIPD_OK) return r;
    } else if (!fast_path_ok(pool, num_q_heads) || spd_mla_prefill_ok(pool, num_q_heads)) {
        // K/V write into the pool, stream-ordered before attention reads it (these
        // paths read the chunk's own keys from the pool); the tcgen05 path fuses it
        semipd_status r = spd_launch_kv_write(pool, layer, k_new, v_new, cu_seqlens_q, req_ids,
                                              prefix_lens, n, total_q, 0, status_dev, st);
        if (r != SEMIPD_OK) return r;
    }
    if (spd_mla_prefill_ok(pool, num_q_heads))  // absorbed MLA latent cache, 64-token pages (cfg 5)
        return spd_launch_prefill_mla(pool, layer, q, cu_seqlens_q, req_ids, prefix_lens, n, total_q,
                                      max_chunk_len, num_q_heads, softmax_scale, out,
                                      out_head_major, budget, status_dev, st);
    if (!fast_path_ok(pool, num_q_heads))
        return spd_launch_simt_attn(pool, layer, q, cu_seqlens_q, req_ids, prefix_lens, n, total_q,
                                    0, num_q_heads, softmax_scale, out, out_head_major, budget,
                                    status_dev, st);
    // 2. tensor-core attention
    const int G = num_q_heads / c.num_kv_heads;
    const int TQ = BM / G;
    PrefillParams prm;
    prm.cu = cu_seqlens_q;
    prm.req_ids = req_ids;
    prm.prefix = prefix_lens;
    prm.bt = pool->bt;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.n_peers = pool->pre_n_peers;
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k)
        prm.peers[k] = k < pool->pre_n_peers ? static_cast<__nv_bfloat16*>(pool->pre_peers[k]) : nullptr;
    prm.status = status_dev;
    prm.span = spd_next_span(pool);
    prm.sched = &pool->st->sched[0];
    prm.n = n;
    prm.T = total_q;
    prm.write_kv = rope || fp8 ? 0 : 1;
    prm.Hq = num_q_heads;
    prm.Hkv = c.num_kv_heads;
    prm.G = G;
    prm.TQ = TQ;
    prm.pairs_max = (max_chunk_len + 2 * TQ - 1) / (2 * TQ);
    if (prm.pairs_max < 1) return SEMIPD_OK;
    const long long units = (long long)n * prm.pairs_max * c.num_kv_heads;
    if (units > (1LL << 30)) return SEMIPD_ERR_UNSUPPORTED;
    prm.n_units = (int)units;
    prm.lg_bs = __builtin_ctz((unsigned)c.block_size);
    prm.box_rows = pool->box_rows;
    prm.MBR = c.max_blocks_per_req;
    prm.N_B = c.num_blocks;
    prm.out_head_major = out_head_major;
    prm.scale_log2 = softmax_scale * LOG2E;
    prm.scale_log2_pre = fp8 ? prm.scale_log2 * pool->k_scale[layer] : prm.scale_log2;
    const CUtensorMap* pkmap = fp8 ? &pool->f8s_kmap : &pool->kmap[layer];
    const CUtensorMap* pvmap = fp8 ? &pool->f8s_vmap : &pool->vmap[layer];
    if (fp8) {  // prefix pages from the staging scratch: request i of the call -> row i
        spd_fp8_prefill_view(pool, &prm.req_ids, &prm.bt, &prm.N_B);
        prm.box_rows = 64;
    }
    prm.k_new = static_cast<const uint4*>(k_new);
    prm.v_new = static_cast<const uint4*>(v_new);
    prm.k_pool = static_cast<unsigned char*>(pool->k_layer(layer));
    prm.v_pool = static_cast<unsigned char*>(pool->v_layer(layer));
    prm.trace = spd_trace(pool);
    prm.tl = reinterpret_cast<long long*>(pool->timeline);
    prm.tl_ctr = pool->timeline_ctr;
    // Q [T][Hq][128] as (64 cols, Hq heads, T tokens, 2 halves); box (64, G, 2 TQ, 2) = both q
    // tiles of a unit in one 64 KiB TMA (a box costs ~800 cycles of the SM's TMA unit, so one
    // big box instead of four 16 KiB ones)
    CUtensorMap qmap;
    {
        const uint64_t dims[4] = {64, (uint64_t)num_q_heads, (uint64_t)total_q, 2};
        const uint64_t strides[3] = {HD * 2, (uint64_t)num_q_heads * HD * 2, 128};
        const uint32_t box[4] = {64, (uint32_t)G, (uint32_t)(2 * TQ), 2};
        if (!spd_encode_tiled_4d(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(q), dims,
                                 strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    // chunk K / V straight from k_new / v_new as (64 cols, Hkv, T, 2 halves): one 32 KiB box
    // (64, 1, 128 rows, 2) per kv tile lands as [half][128 rows][128 B] (the TMA unit's cost is
    // per box, so one box per tile instead of one per 64-column half)
    CUtensorMap kcmap, vcmap;
    {
        const uint64_t dims[4] = {64, (uint64_t)c.num_kv_heads, (uint64_t)total_q, 2};
        const uint64_t strides[3] = {HD * 2, (uint64_t)c.num_kv_heads * HD * 2, 128};
        const uint32_t box[4] = {64, 1, BN, 2};
        if (!spd_encode_tiled_4d(&kcmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(k_new),
                                 dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B) ||
            !spd_encode_tiled_4d(&vcmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(v_new),
                                 dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    // output map for the epilogue's TMA stores: token-major [T][Hq][128] box (64, G, TQ) or
    // head-major [Hq][T][128] box (64, TQ, G)
    CUtensorMap omap;
    if (!out_head_major) {
        if (!spd_encode_tiled_3d(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, HD, (uint64_t)num_q_heads,
                                 (uint64_t)total_q, HD * 2, (uint64_t)num_q_heads * HD * 2, 64,
                                 (uint32_t)G, (uint32_t)TQ, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    } else {
        if (!spd_encode_tiled_3d(&omap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, out, HD, (uint64_t)total_q,
                                 (uint64_t)num_q_heads, HD * 2, (uint64_t)total_q * HD * 2, 64,
                                 (uint32_t)TQ, (uint32_t)G, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    const size_t smem = sizeof(Smem) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(prefill_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess ||
            cudaFuncSetAttribute(prefill_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr_set = true;
    }
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    const cudaError_t le = prm.n_peers > 0
        ? spd_launch_pdl(prefill_tc_kernel<true>, dim3(grid), dim3(NT), smem, st, qmap, *pkmap, *pvmap, kcmap,
                         vcmap, omap, prm)
        : spd_launch_pdl(prefill_tc_kernel<false>, dim3(grid), dim3(NT), smem, st, qmap, *pkmap, *pvmap, kcmap,
                         vcmap, omap, prm);
    if (le != cudaSuccess) return SEMIPD_ERR_CUDA;
    pool->launches += 1;
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

extern "C" semipd_status semipd_set_prefill_peers(semipd_pool_t pool, void* const* peer_out,
                                                  int32_t n, int32_t tokens) {
    if (!pool || n < 0 || n > SEMIPD_MAX_PEERS - 1 || (n > 0 && (!peer_out || tokens <= 0)))
        return SEMIPD_ERR_INVALID;
    for (int k = 0; k < n; ++k)
        if (!peer_out[k] || reinterpret_cast<uintptr_t>(peer_out[k]) % 16) return SEMIPD_ERR_INVALID;
    for (int k = 0; k < SEMIPD_MAX_PEERS - 1; ++k) pool->pre_peers[k] = k < n ? peer_out[k] : nullptr;
    pool->pre_n_peers = n;
    pool->pre_peer_tokens = n > 0 ? tokens : 0;
    return SEMIPD_OK;
}
