// prefill_mla.cu — absorbed-MLA chunked prefill attention on the 5th-gen tensor cores (cfg 5:
// 16 q heads share ONE latent KV head, dk = 576, dv = 512, V = K[..., :512]; R19).
// Causal, bottom-right aligned (row t of request r sees keys 0 .. P_r + t, R4), keys read
// from the paged latent pool after the chunk's own rows were written there.
//
// Tile: M = 64 rows = 4 consecutive tokens x 16 heads (GQA packing: every K/V page is read
// once per 4 tokens x 16 heads).  With M = 64 a tcgen05 accumulator only occupies TMEM lanes
// 0-15 of each 32-lane quadrant, and a second accumulator can sit at lane base 16
// (scripts/probe_umma_m64.cu), so the 64 x 512 fp32 output fits in 256 columns:
//   S  [64 x 64 keys]  = Q[64 x 576] . K^T       M=64 N=64,  36 x K16, SS  (2 TMEM buffers)
//   O_lo[64 x 256]    += P[64 x 64] . V[:, 0:256]   M=64 N=256, 4 x K16, SS  (lane base 0)
//   O_hi[64 x 256]    += P[64 x 64] . V[:, 256:512] M=64 N=256, 4 x K16, SS  (lane base 16)
// A page (64 keys x 576) lands as two 4-D TMA boxes (column blocks [0,4) and [4,9)) in 40 KiB
// ring slots — the same boxes as the MLA decode kernel; V is read MN-major from them.
//
// Warps: 0 producer (units, TMA), 1 MMA issuer (warp-collective), 2-5 softmax + epilogue.
// Softmax warp w handles token w % 4 of the tile: lanes 0-15 own one head's row each (the
// causal limit is warp-uniform), lanes 16-31 own the O_hi half of the same rows.  Lazy
// rescale (reference max moves only when the running max exceeds it by > 8 in log2 units);
// the denominator sums the bf16-rounded P that the MMA consumes, so both sides of the
// quotient see the same P (R16).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int DK = 576, DV = 512, NH = 16;
constexpr int PAGE = 64;
constexpr int NCB = DK / 64;                            // 9 column blocks
constexpr int CB_LO = 4;
constexpr uint32_t LO_BYTES = CB_LO * PAGE * 128;       // 32 KiB
constexpr uint32_t HI_BYTES = (NCB - CB_LO) * PAGE * 128;  // 40 KiB
constexpr uint32_t SLOT_BYTES = HI_BYTES;
// SPD_MLAP_SWAP = 1: PV as O^T[128 dv x 64 rows] += V^T . P^T per 128-dv block (M = 128: the
//   full tensor rate; 4 accumulators over all 128 TMEM lanes) instead of O_lo / O_hi at
//   M = 64 (half rate); P^T is the K-major P tile the softmax writes anyway.
// SPD_MLAP_RING4 = 1: a 4-slot ring of exactly sized halves (even slots 32 KiB LO boxes, odd
//   slots 40 KiB HI boxes: 2 pages in flight instead of 1.5) and one P buffer.
// Measured (same box, microbench C = 2048, TFLOP/s at 104 / 148 SMs; profiles/r2_mla_prefill_ab.log):
//   SWAP 0 RING4 0: 235 / 309    SWAP 1 RING4 0: 196 / 255
//   SWAP 0 RING4 1: 301 / 389    SWAP 1 RING4 1: 235 / 302
// The ring depth is what limits the pipeline (+28 %); the swapped PV's per-tile four-warp
// agreement on the rescale set and its 16 MMAs per page cost more than its full-rate MMAs gain.
#ifndef SPD_MLAP_SWAP
#define SPD_MLAP_SWAP 0
#endif
#ifndef SPD_MLAP_RING4
#define SPD_MLAP_RING4 1
#endif
constexpr bool SWAP = SPD_MLAP_SWAP != 0;
constexpr int NSLOT = SPD_MLAP_RING4 ? 4 : 3;
constexpr int NPBUF = SPD_MLAP_RING4 ? 1 : 2;
constexpr uint32_t RING_BYTES = SPD_MLAP_RING4 ? 2 * (LO_BYTES + HI_BYTES) : NSLOT * SLOT_BYTES;
__host__ __device__ constexpr uint32_t slot_off(int s) {
    return SPD_MLAP_RING4 ? (uint32_t)(s >> 1) * (LO_BYTES + HI_BYTES) + (uint32_t)(s & 1) * LO_BYTES
                          : (uint32_t)s * SLOT_BYTES;
}
constexpr int TQ = 4;                                   // tokens per unit
constexpr int BM = TQ * NH;                             // 64 rows
constexpr uint32_t Q_BYTES = NCB * BM * 128;            // 72 KiB
constexpr uint32_t P_BYTES = BM * 128;                  // 8 KiB per buffer
constexpr int NTHREADS = 192;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_TH = 8.f;
constexpr uint32_t TM_O = 0, TM_S = 256, TM_COLS = 512;

struct PUnit {
    int i, t0, ntok, P, kend, nt, row0, rid;  // i < 0: done
};

struct PmParams {
    const int* cu;
    const int* req_ids;
    const int* prefix;
    const int* bt;
    __nv_bfloat16* out;  // [T][Hq][512] or [Hq][T][512]
    int* status;
    unsigned long long* span;  // semipd_set_spans record of this launch (or null)
    unsigned* sched;
    int n, T, Hq, maxqb, n_units, MBR, N_B, out_head_major;
    float scale_log2;
    SpdTrace trace;
};

struct Bars {
    uint64_t full[NSLOT], empty[NSLOT], s_full[2], s_empty[2], p_full[2], o_done[2], q_full,
        q_empty, ufull[2], uempty[2];
};

constexpr uint32_t OFF_Q = RING_BYTES;
constexpr uint32_t OFF_P = OFF_Q + Q_BYTES;
constexpr uint32_t OFF_RED = OFF_P + NPBUF * P_BYTES;   // swap: [2][64] alphas, [64] 1/l, flags
constexpr uint32_t OFF_BARS = OFF_RED + (SWAP ? (3 * 64 + 8) * 4 : 0);
constexpr uint32_t OFF_UNITS = OFF_BARS + sizeof(Bars);
constexpr uint32_t OFF_MISC = OFF_UNITS + 2 * sizeof(PUnit);
constexpr uint32_t SMEM_BYTES = 1024 + OFF_MISC + 16;
static_assert(OFF_Q % 1024 == 0 && OFF_P % 1024 == 0, "UMMA operands need 1 KiB alignment");
static_assert(SMEM_BYTES <= 232448, "exceeds the 227 KiB opt-in shared memory");

__global__ void __launch_bounds__(NTHREADS, 1)
    prefill_mla_kernel(const __grid_constant__ CUtensorMap map_lo,
                       const __grid_constant__ CUtensorMap map_hi,
                       const __grid_constant__ CUtensorMap qmap, PmParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    unsigned char* ring = base;
    unsigned char* qs = base + OFF_Q;
    unsigned char* ps = base + OFF_P;
    Bars& bar = *reinterpret_cast<Bars*>(base + OFF_BARS);
    PUnit* units = reinterpret_cast<PUnit*>(base + OFF_UNITS);
    uint32_t* tmem_base = reinterpret_cast<uint32_t*>(base + OFF_MISC);

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
            mbar_init(bar.p_full + i, 4);
            mbar_init(bar.o_done + i, 1);
            mbar_init(bar.ufull + i, 1);
            mbar_init(bar.uempty + i, 5);
        }
        mbar_init(&bar.q_full, 1);
        mbar_init(&bar.q_empty, 1);
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(1, (int)smid(), (int)blockIdx.x, 5 /* kernel kind: MLA prefill */);
        }
    }
    if (warp == 1) tmem_alloc(tmem_base, TM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // PDL: the previous kernel on this stream is complete (workspace counters, pool)
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = *tmem_base;

    if (warp == 0) {
        // =========================== producer ===========================
        if (lane == 0) {
            tma_prefetch_desc(&map_lo);
            tma_prefetch_desc(&map_hi);
            tma_prefetch_desc(&qmap);
        }
        int gh = 0, nunit = 0, nq = 0;
        int u_next = blockIdx.x;
        for (;;) {
            const int u = u_next;
            if (lane == 0) u_next = (int)gridDim.x + (int)atomicAdd(p.sched, 1u);
            u_next = __shfl_sync(0xffffffffu, u_next, 0);
            PUnit d;
            if (u >= p.n_units) {
                d.i = -1;
            } else {
                // longest-first: the last token blocks of every request (most keys) go first
                d.i = u % p.n;
                const int qb = p.maxqb - 1 - u / p.n;
                const int c0 = __ldg(p.cu + d.i), C = __ldg(p.cu + d.i + 1) - c0;
                d.t0 = qb * TQ;
                if (d.t0 >= C) continue;
                d.ntok = min(TQ, C - d.t0);
                d.P = __ldg(p.prefix + d.i);
                d.kend = d.P + d.t0 + d.ntok;
                d.nt = (d.kend + PAGE - 1) / PAGE;
                d.row0 = c0 + d.t0;
                d.rid = __ldg(p.req_ids + d.i);
            }
            const int us = nunit & 1;
            if (lane == 0) {
                mbar_wait(bar.uempty + us, ((nunit >> 1) & 1) ^ 1);
                units[us] = d;
                mbar_arrive(bar.ufull + us);
            }
            __syncwarp();
            ++nunit;
            if (d.i < 0) {  // no more units: the next kernel on the stream may be scheduled
                pdl_trigger();
                break;
            }
            const int* btr = p.bt + (size_t)d.rid * p.MBR;
            int blk_l = -1;
            for (int j = 0; j < d.nt; ++j, gh += 2) {
                if ((j & 31) == 0) {
                    const int pg = j + lane;
                    blk_l = (pg < d.nt && pg < p.MBR) ? __ldg(btr + pg) : -1;
                }
                const int blk = __shfl_sync(0xffffffffu, blk_l, j & 31);
                if (lane == 0) {
                    int z = p.N_B;  // out of range: zero fill
                    if (blk >= 0 && blk < p.N_B) z = blk;
                    else if (p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                    const int s0 = gh % NSLOT, s1 = (gh + 1) % NSLOT;
                    mbar_wait(bar.empty + s0, ((gh / NSLOT) & 1) ^ 1);
                    mbar_arrive_expect_tx(bar.full + s0, LO_BYTES);
                    tma_load_4d(ring + slot_off(s0), &map_lo, bar.full + s0, 0, 0, 0, z);
                    if (j == 0) {
                        // this unit's Q (64 rows): free once the previous unit's last QK is done
                        mbar_wait(&bar.q_empty, (nq & 1) ^ 1);
                        mbar_arrive_expect_tx(&bar.q_full, Q_BYTES);
                        tma_load_4d(qs, &qmap, &bar.q_full, 0, 0, d.row0, 0);
                    }
                    mbar_wait(bar.empty + s1, (((gh + 1) / NSLOT) & 1) ^ 1);
                    mbar_arrive_expect_tx(bar.full + s1, HI_BYTES);
                    tma_load_4d(ring + slot_off(s1), &map_hi, bar.full + s1, 0, 0, CB_LO, z);
                }
                __syncwarp();
            }
            ++nq;
        }
    } else if (warp == 1) {
        // =========================== MMA issuer (warp-collective) ===========================
        constexpr uint32_t ID_QK = umma_idesc_bf16_f32_ab(BM, PAGE, 0, 0);
        constexpr uint32_t ID_PV = SWAP ? umma_idesc_bf16_f32_ab(128, BM, 1, 0)
                                        : umma_idesc_bf16_f32_ab(BM, 256, 0, 1);
        const uint32_t ring_a = smem_u32(ring);
        const uint32_t dq0 = desc_lo(smem_u32(qs), 16);  // (low, high) descriptor words (umma_ss_warp2)
        constexpr uint32_t DH = DESC_HI_SBO1K;
        const uint32_t dp0 = desc_lo(smem_u32(ps), 16);
        auto probe = [&](const uint64_t* b, uint32_t par) {
            bool r = false;
            if (lane == 0) r = mbar_test_wait(b, par);
            return __shfl_sync(0xffffffffu, r ? 1 : 0, 0) != 0;
        };
        int gh = 0, gt = 0, nunit = 0, nq = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(bar.ufull + us, (nunit >> 1) & 1);
            const PUnit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(bar.uempty + us);
            ++nunit;
            if (d.i < 0) break;
            bool q_ok = false, qk_lo = false;
            int nqk = 0, npv = 0;
            while (npv < d.nt) {
                const int tp = gt + npv, pb = tp & 1;
                if (npv < nqk && probe(bar.p_full + pb, (tp >> 1) & 1)) {
                    const int h0 = gh + 2 * npv;
                    const int s0 = h0 % NSLOT, s1 = (h0 + 1) % NSLOT;
                    tc_fence_after();
                    const uint32_t dpa = dp0 + (uint32_t)((pb % NPBUF) * (P_BYTES / 16));
                    if constexpr (SWAP) {
                        // O^T[dv block m] += V^T[128 dv x 64 keys] . P^T: V^T MN-major straight
                        // from the page boxes (LBO 8 KiB between 64-column blocks, SBO 1 KiB
                        // between 8-key groups); blocks 0, 1 in the first box, 2, 3 in the second
                        const uint32_t lo = ring_a + slot_off(s0), hi = ring_a + slot_off(s1);
#pragma unroll
                        for (int m = 0; m < DV / 128; ++m) {
                            const uint32_t a0 = m < 2 ? lo + m * (2 * PAGE * 128)
                                                      : hi + (2 * m - CB_LO) * (PAGE * 128);
                            const uint32_t da = desc_lo(a0, PAGE * 128);
#pragma unroll
                            for (int ks = 0; ks < PAGE / 16; ++ks)
                                umma_ss_warp2(tmem + TM_O + m * BM, da + (uint32_t)(ks * 128), DH,
                                             dpa + (uint32_t)(ks * 2), DH, ID_PV, (npv > 0 || ks > 0) ? 1u : 0u);
                            if (m == 1) umma_commit_warp(bar.empty + s0);
                        }
                    } else {
                        // V^T blocks: dv [0,256) = column blocks 0-3 (first box), [256,512) = 4-7
                        const uint32_t dvlo = desc_lo(ring_a + slot_off(s0), PAGE * 128);
                        const uint32_t dvhi = desc_lo(ring_a + slot_off(s1), PAGE * 128);
#pragma unroll
                        for (int ks = 0; ks < PAGE / 16; ++ks)
                            umma_ss_warp2(tmem + TM_O, dpa + (uint32_t)(ks * 2), DH, dvlo + (uint32_t)(ks * 128), DH,
                                         ID_PV, (npv > 0 || ks > 0) ? 1u : 0u);
                        umma_commit_warp(bar.empty + s0);
#pragma unroll
                        for (int ks = 0; ks < PAGE / 16; ++ks)
                            umma_ss_warp2(tmem + TM_O + (16u << 16), dpa + (uint32_t)(ks * 2), DH,
                                         dvhi + (uint32_t)(ks * 128), DH, ID_PV, (npv > 0 || ks > 0) ? 1u : 0u);
                    }
                    umma_commit_warp(bar.o_done + pb);
                    umma_commit_warp(bar.empty + s1);
                    ++npv;
                    continue;
                }
                if (nqk < d.nt) {
                    const int t = gt + nqk, sb = t & 1, h0 = gh + 2 * nqk;
                    const int s0 = h0 % NSLOT, s1 = (h0 + 1) % NSLOT;
                    if (!q_ok) q_ok = probe(&bar.q_full, nq & 1);
                    if (q_ok && !qk_lo && probe(bar.s_empty + sb, ((t >> 1) & 1) ^ 1) &&
                        probe(bar.full + s0, (h0 / NSLOT) & 1)) {
                        tc_fence_after();
                        const uint32_t dk = desc_lo(ring_a + slot_off(s0), 16);
#pragma unroll
                        for (int k = 0; k < CB_LO * 4; ++k) {
                            const int cb = k >> 2;
                            umma_ss_warp2(tmem + TM_S + sb * PAGE,
                                         dq0 + (uint32_t)(cb * (BM * 128 / 16) + (k & 3) * 2), DH,
                                         dk + (uint32_t)(cb * (PAGE * 128 / 16) + (k & 3) * 2), DH, ID_QK,
                                         k > 0);
                        }
                        qk_lo = true;
                        continue;
                    }
                    if (qk_lo && probe(bar.full + s1, ((h0 + 1) / NSLOT) & 1)) {
                        tc_fence_after();
                        const uint32_t dk = desc_lo(ring_a + slot_off(s1), 16);
#pragma unroll
                        for (int k = CB_LO * 4; k < DK / 16; ++k) {
                            const int cb = k >> 2;
                            umma_ss_warp2(tmem + TM_S + sb * PAGE,
                                         dq0 + (uint32_t)(cb * (BM * 128 / 16) + (k & 3) * 2), DH,
                                         dk + (uint32_t)((cb - CB_LO) * (PAGE * 128 / 16) + (k & 3) * 2), DH,
                                         ID_QK, 1u);
                        }
                        umma_commit_warp(bar.s_full + sb);
                        if (nqk == d.nt - 1) umma_commit_warp(&bar.q_empty);
                        qk_lo = false;
                        ++nqk;
                        continue;
                    }
                }
                __nanosleep(32);
            }
            ++nq;
            gt += d.nt;
            gh += 2 * d.nt;
        }
    } else {
        // =========================== softmax + epilogue ===========================
        const int qd = warp & 3;  // TMEM lane quadrant = token of the tile
        const uint32_t lane_base = (uint32_t)(qd * 32) << 16;
        const bool lo = lane < 16;
        const int h = lane & 15;  // head of this lane's row
        const int row = qd * 16 + h;
        float* red = reinterpret_cast<float*>(base + OFF_RED);  // swap: [2][64] alpha, [64] 1/l
        int* rflag = reinterpret_cast<int*>(red + 3 * BM);       // swap: [2][4] rescale flags
        int gt = 0, nunit = 0;
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(bar.ufull + us, (nunit >> 1) & 1);
            const PUnit d = units[us];
            __syncwarp();
            if (lane == 0) mbar_arrive(bar.uempty + us);
            ++nunit;
            if (d.i < 0) break;
            const int klim = d.P + d.t0 + qd + 1;  // keys [0, klim) visible to this token
            float mref = -INFINITY;                 // reference max of P / O (log2 domain)
            float lsum = 0.f;
            for (int j = 0; j < d.nt; ++j) {
                const int t = gt + j, sb = t & 1;
                mbar_wait(bar.s_full + sb, (t >> 1) & 1);
                tc_fence_after();
                uint32_t sr[2][32];
                tmem_ld32(tmem + lane_base + TM_S + sb * PAGE, sr[0]);
                tmem_ld32(tmem + lane_base + TM_S + sb * PAGE + 32, sr[1]);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar.s_empty + sb);
                const int k0 = j * PAGE;
                float mt = -INFINITY;
#pragma unroll
                for (int c = 0; c < PAGE; ++c) {
                    float x = __uint_as_float(sr[c >> 5][c & 31]) * p.scale_log2;
                    x = (k0 + c < klim) ? x : -INFINITY;
                    sr[c >> 5][c & 31] = __float_as_uint(x);
                    mt = fmaxf(mt, x);
                }
                // lazy rescale: move the reference only when the max grew by > RESCALE_TH
                const bool move = lo && (mt > mref + RESCALE_TH || j == 0);
                const float mnew = move ? fmaxf(mt, mref) : mref;
                const float alpha = (move && j > 0) ? fast_exp2(mref - mnew) : 1.f;
                mref = mnew;
                lsum *= alpha;
                bool any_rescale = __any_sync(0xffffffffu, move && j > 0);
                if constexpr (SWAP) {
                    // O^T holds every row in a column across all 128 lanes: the four warps
                    // agree on this tile's rescale set through smem (double-buffered by tile)
                    float* alph = red + sb * BM;
                    if (lo) alph[row] = alpha;
                    if (lane == 0) rflag[sb * 4 + qd] = any_rescale ? 1 : 0;
                    named_bar_sync(1, 128);
                    any_rescale = (rflag[sb * 4 + 0] | rflag[sb * 4 + 1] | rflag[sb * 4 + 2] |
                                   rflag[sb * 4 + 3]) != 0;
                }
                // the P buffer is free once the PV that last read it completed (NPBUF = 2:
                // PV(t-2), NPBUF = 1: PV(t-1)); O may be rescaled only after PV(t-1) completed
                if (any_rescale && j > 0) {
                    mbar_wait(bar.o_done + ((t - 1) & 1), ((t - 1) >> 1) & 1);
                } else if (t >= NPBUF) {
                    mbar_wait(bar.o_done + ((t - NPBUF) & 1), ((t - NPBUF) >> 1) & 1);
                }
                tc_fence_after();
                if (any_rescale && j > 0) {
                    if constexpr (SWAP) {
                        // column r of every O^T block scales by alpha[r]
                        const float* alph = red + sb * BM;
#pragma unroll 1
                        for (int m = 0; m < DV / 128; ++m) {
#pragma unroll 1
                            for (int cc = 0; cc < BM; cc += 32) {
                                const uint32_t oa = tmem + lane_base + TM_O + m * BM + cc;
                                uint32_t o[32];
                                tmem_ld32(oa, o);
                                tmem_wait_ld();
#pragma unroll
                                for (int e = 0; e < 32; ++e)
                                    o[e] = __float_as_uint(__uint_as_float(o[e]) * alph[cc + e]);
                                tmem_st32(oa, o);
                            }
                        }
                    } else {
                        // lanes 0-15: O_lo of row (qd, h); lanes 16-31: O_hi of the same row
                        const float a = __shfl_sync(0xffffffffu, alpha, h);
                        const uint32_t ob = tmem + lane_base + TM_O;
#pragma unroll 1
                        for (int cc = 0; cc < 256; cc += 32) {
                            uint32_t o[32];
                            tmem_ld32(ob + cc, o);
                            tmem_wait_ld();
#pragma unroll
                            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * a);
                            tmem_st32(ob + cc, o);
                        }
                    }
                    tmem_wait_st();
                }
                // P row (64 keys, bf16) -> P buffer, K-major 128-B swizzle (the A operand of
                // P.V, or the B operand P^T of the swapped V^T.P^T); lsum from the rounded values
                if (lo) {
                    unsigned char* prow = ps + (sb % NPBUF) * P_BYTES + row * 128;
                    const int sw = row & 7;
#pragma unroll
                    for (int c8 = 0; c8 < 8; ++c8) {
                        uint32_t w[4];
#pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            const int c = c8 * 8 + 2 * e;
                            const __nv_bfloat16 b0 = __float2bfloat16_rn(
                                fast_exp2(__uint_as_float(sr[c >> 5][c & 31]) - mref));
                            const __nv_bfloat16 b1 = __float2bfloat16_rn(
                                fast_exp2(__uint_as_float(sr[(c + 1) >> 5][(c + 1) & 31]) - mref));
                            lsum += __bfloat162float(b0) + __bfloat162float(b1);
                            w[e] = (uint32_t)__bfloat16_as_ushort(b0) |
                                   ((uint32_t)__bfloat16_as_ushort(b1) << 16);
                        }
                        *reinterpret_cast<uint4*>(prow + ((c8 ^ sw) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar.p_full + sb);
            }
            gt += d.nt;
            // ---- epilogue: O / l -> bf16
            mbar_wait(bar.o_done + ((gt - 1) & 1), ((gt - 1) >> 1) & 1);
            tc_fence_after();
            if constexpr (SWAP) {
                // thread = dv index (block m, quadrant qd, lane) of all 64 rows: lane pairs
                // exchange so each lane stores bf16x2 of every other row
                float* rl = red + 2 * BM;
                if (lo) rl[row] = __frcp_rn(lsum);
                named_bar_sync(1, 128);
                const bool odd = lane & 1;
#pragma unroll 1
                for (int m = 0; m < DV / 128; ++m) {
                    const int dve = m * 128 + qd * 32 + (lane & ~1);
#pragma unroll 1
                    for (int cc = 0; cc < BM; cc += 32) {
                        uint32_t o[32];
                        tmem_ld32(tmem + lane_base + TM_O + m * BM + cc, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int r = cc + e;
                            const float v = __uint_as_float(o[e]) * rl[r];
                            const float other = __shfl_xor_sync(0xffffffffu, v, 1);
                            const int tk = r >> 4, hh = r & 15;
                            if (((r & 1) != 0) == odd && tk < d.ntok && hh < p.Hq) {
                                const size_t tok = (size_t)d.row0 + tk;
                                __nv_bfloat16* op = p.out + (p.out_head_major ? ((size_t)hh * p.T + tok) * DV
                                                                              : (tok * p.Hq + hh) * DV) + dve;
                                *reinterpret_cast<uint32_t*>(op) = odd ? pack_bf16(other, v) : pack_bf16(v, other);
                            }
                        }
                    }
                }
                // rl / alpha / flags are rewritten by the next unit
                named_bar_sync(1, 128);
            } else {
                // lanes 0-15: dv [0,256), lanes 16-31: [256,512)
                const float rl = __frcp_rn(__shfl_sync(0xffffffffu, lsum, h));
                const bool store = qd < d.ntok && h < p.Hq;
                const size_t tok = (size_t)d.row0 + qd;
                __nv_bfloat16* orow = p.out + (p.out_head_major ? ((size_t)h * p.T + tok) * DV
                                                                : (tok * p.Hq + h) * DV) +
                                      (lo ? 0 : 256);
                const uint32_t ob = tmem + lane_base + TM_O;
#pragma unroll 1
                for (int cc = 0; cc < 256; cc += 32) {
                    uint32_t o[32];
                    tmem_ld32(ob + cc, o);
                    tmem_wait_ld();
                    if (store) {
#pragma unroll
                        for (int e8 = 0; e8 < 4; ++e8) {
                            uint4 v;
                            v.x = pack_bf16(__uint_as_float(o[e8 * 8 + 0]) * rl, __uint_as_float(o[e8 * 8 + 1]) * rl);
                            v.y = pack_bf16(__uint_as_float(o[e8 * 8 + 2]) * rl, __uint_as_float(o[e8 * 8 + 3]) * rl);
                            v.z = pack_bf16(__uint_as_float(o[e8 * 8 + 4]) * rl, __uint_as_float(o[e8 * 8 + 5]) * rl);
                            v.w = pack_bf16(__uint_as_float(o[e8 * 8 + 6]) * rl, __uint_as_float(o[e8 * 8 + 7]) * rl);
                            *reinterpret_cast<uint4*>(orow + cc + e8 * 8) = v;
                        }
                    }
                }
            }
            tc_fence_before();
        }
    }
    tc_fence_before();
    __syncthreads();
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

bool spd_mla_prefill_ok(const semipd_pool* p, int Hq) {
    const auto& c = p->cfg;
    return c.dtype == SEMIPD_BF16 && c.kv_shared && c.num_kv_heads == 1 && c.head_dim_k == DK &&
           c.head_dim_v == DV && Hq <= NH && c.block_size == PAGE && p->have_mla_tc_maps;
}

semipd_status spd_launch_prefill_mla(semipd_pool_t pool, int layer, const void* q,
                                     const int* cu_seqlens, const int* req_ids,
                                     const int* prefix_lens, int n, int total_q, int max_chunk_len,
                                     int Hq, float scale, void* out, int out_head_major,
                                     int budget, int* status_dev, cudaStream_t st) {
    if ((reinterpret_cast<uintptr_t>(q) & 15) != 0) return SEMIPD_ERR_INVALID;
    // Q [T][Hq][576] as (64 cols, Hq heads, T tokens, 9 column blocks); box (64, 16, 4, 9)
    // lands [cb][token][head][128 B] = K-major rows t * 16 + h; heads >= Hq and tokens >= T
    // are zero-filled
    CUtensorMap qmap;
    {
        const uint64_t dims[4] = {64, (uint64_t)Hq, (uint64_t)total_q, NCB};
        const uint64_t strides[3] = {DK * 2, (uint64_t)Hq * DK * 2, 128};
        const uint32_t box[4] = {64, NH, TQ, NCB};
        if (!spd_encode_tiled_4d(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(q), dims,
                                 strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    PmParams prm;
    prm.cu = cu_seqlens;
    prm.req_ids = req_ids;
    prm.prefix = prefix_lens;
    prm.bt = pool->bt;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.status = status_dev;
    prm.span = spd_next_span(pool);
    prm.sched = &pool->st->sched[0];
    prm.n = n;
    prm.T = total_q;
    prm.Hq = Hq;
    prm.maxqb = (max_chunk_len + TQ - 1) / TQ;
    if (prm.maxqb < 1) return SEMIPD_OK;
    const long long units = (long long)n * prm.maxqb;
    if (units > (1LL << 30)) return SEMIPD_ERR_UNSUPPORTED;
    prm.n_units = (int)units;
    prm.MBR = pool->cfg.max_blocks_per_req;
    prm.N_B = pool->cfg.num_blocks;
    prm.out_head_major = out_head_major;
    prm.scale_log2 = scale * LOG2E;
    prm.trace = spd_trace(pool);
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(prefill_mla_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_BYTES) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr = true;
    }
    int grid = budget > 0 ? budget : prm.n_units;
    if (grid > prm.n_units) grid = prm.n_units;
    const cudaError_t le = spd_launch_pdl(prefill_mla_kernel, dim3(grid), dim3(NTHREADS), SMEM_BYTES, st,
                                          pool->mla_lo[layer], pool->mla_hi[layer], qmap, prm);
    pool->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
