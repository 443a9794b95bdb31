// prefill_mla_exp.cu — expanded-form MLA chunked prefill (R32).
//
// The absorbed form (prefill_mla.cu) attends over the 576-wide latent directly: 2 x (576 + 512)
// flops per (query, key, head).  The expanded form first projects every key's cached latent
// c_j (512) to per-head keys and values with the model's up-projections,
//   k_nope[j][h] = bf16(W_UK[h] c_j) (128),  v[j][h] = bf16(W_UV[h] c_j) (128),
// keys [k_nope | k_pe_j] (192, the rope part k_pe_j = latent columns 512..575 is shared by all
// heads), then runs causal MHA per head: 2 x (192 + 128) flops per (query, key, head) plus
// 2 x 512 x 2 x 128 per (key, head) for the projection — 3.4x fewer flops than the absorbed
// form for a chunk without prefix.  The latent pool stays the cache (the chunk's latent
// rows are written first; P:229 paged access); the expanded K / V are per-call activations.
//
// Three launches on the caller's stream:
//   1. mla_exp_prep_kernel (CUDA cores, HBM-bound): the chunk's latent rows -> pool pages
//      (bit copies), every key's k_pe -> a contiguous [rows][64] buffer, the call's row
//      offsets (each request's keys padded to 128-row tiles) -> the workspace header.
//   2. mla_exp_gemm_kernel (tcgen05): [keys x 512] x [512 x 2 H 128] up-projection.  A = latent
//      rows gathered from the paged pool by TMA (one box per page per 64-column k-stage), B =
//      W_UK / W_UV rows (K-major), D = 128 x 256 fp32 tiles in TMEM (two buffers: the epilogue
//      of tile n overlaps the mainloop of tile n + 1), epilogue -> bf16 RNE -> K_exp / V_exp
//      [rows][H][128].  Rows past a request's keys are written as zeros (finite P V inputs).
//   3. mla_exp_attn_kernel (tcgen05): the GQA prefill kernel's structure (prefill_sm100.cu) at
//      G = 1 with dqk = 192: unit = (request, pair of 128-row q tiles, head), S = Q K^T over
//      12 K16 steps, O += P V; Q pair in one 96 KiB TMA box, K (3 x 64-column slots: two
//      k_nope halves + k_pe) and V (2 slots) through one ring of eight 16 KiB slots, so the
//      96 KiB Q pair and 1.6 kv tiles fit in 224 KiB.  Softmax as in the GQA kernel (exact
//      causal limit, lazy rescale R21, bf16 P summed as consumed).  Epilogue: 16-byte stores
//      of each thread's 256-byte output row.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

using namespace spd;

constexpr int XDN = 128;            // k_nope / q_nope per head
constexpr int XDR = 64;             // rope part
constexpr int XDC = 512;            // latent (W_UK / W_UV input) width
constexpr int XDV = 128;            // v per head
constexpr int XDL = XDC + XDR;      // 576: latent pool row
constexpr int XBM = 128;            // q rows per tile, keys per kv tile, key rows per GEMM tile
constexpr int XMAXN = 1024;         // requests per call
constexpr float XLOG2E = 1.4426950408889634f;

// ------------------------------------------------------------------ kv split of long units
// SPD_X_SPLIT_MIN = k (a compile switch, OFF by default): a unit (request, pair of q tiles, head)
// whose tile B needs >= k kv tiles runs as two parts over kv tiles [0, h) and [h, nB), h = nB / 2,
// on two CTAs; the part that finishes first stores its unnormalised O rows with (m, l), the
// second merges them with its own in TMEM (x_split_epilogue; weights and sum formed without
// contraction, so bitwise independent of which part came first).  The rule depends on shapes
// only (R26).  Parity-green (tests/test_gpu_mla_expanded.py, 30/30 at k = 10), but measured
// slower (profiles/r2_mla_expanded_split_ab.log, C = 2048): splitting alone shortens the
// critical path (-18 % at 148 SMs, P = 0, with the merge stubbed out), but the merge handshake
// (partial store, release / acquire flag, partial load) stalls both parts' pipelines: +17 % at
// 148 SMs and +52 % at 44 SMs with it.
#ifndef SPD_X_SPLIT_MIN
#define SPD_X_SPLIT_MIN 1000000
#endif
constexpr int XSPLIT_MIN = SPD_X_SPLIT_MIN;
constexpr bool kXSplit = XSPLIT_MIN < 1000000;
#ifndef SPD_X_RESCALE16
#define SPD_X_RESCALE16 1
#endif
constexpr int XPROW = XDV + 4;  // floats per stored partial row: O[128], m, l, pad
__host__ __device__ __forceinline__ int x_pair_nkv(int P, int C, int pair) {  // kv tiles of tile B
    const int last = min(C, (pair + 1) * 2 * XBM);  // chunk rows of the pair's end
    return (P + last - 1) / XBM + 1;
}
__host__ __device__ __forceinline__ int x_split_pairs(int P, int C) {  // pairs that split
    const int pairs = (C + 2 * XBM - 1) / (2 * XBM);
    int k = 0;
    for (int pr = 0; pr < pairs; ++pr) k += x_pair_nkv(P, C, pr) >= XSPLIT_MIN;
    return k;
}
__host__ __device__ __forceinline__ int x_first_split_pair(int P, int C) {
    const int pairs = (C + 2 * XBM - 1) / (2 * XBM);
    int pr = 0;
    while (pr < pairs && x_pair_nkv(P, C, pr) < XSPLIT_MIN) ++pr;
    return pr;
}

// ------------------------------------------------------------------ workspace
// [hdr: int mtoff[n + 1] (128-row tile offset of each request's keys), int sbase[n + 1] (split
// pair offset)] [K_exp rows x H x 128] [V_exp rows x H x 128] [Kpe rows x 64] [Lat rows x 512]
// [split counters: slots x 2 tiles x (role counter, flag) int] [partials: slots x 2 tiles x 128 rows
// x XPROW fp32 (the first part's rows)],
// rows = max_total_keys + 128 n (per-request padding), slots = (max_total_keys / 256 + n) x H
// (a split pair has >= 1 chunk row per 256, so the call has at most total_q / 256 + n of them)
size_t x_hdr_bytes(int n) { return spd_al256(sizeof(int) * 2 * (size_t)(n + 1)); }
size_t x_rows(int n, int max_keys) { return (size_t)max_keys + (size_t)XBM * (size_t)n; }
size_t x_slots(int n, int max_keys, int H) {
    return kXSplit ? ((size_t)max_keys / (2 * XBM) + (size_t)n) * (size_t)H : 0;
}
size_t x_cnt_bytes(size_t slots) { return spd_al256(slots * 2 * 2 * sizeof(int)); }
size_t x_part_bytes(size_t slots) { return spd_al256(slots * 2 * XBM * XPROW * sizeof(float)); }
size_t x_ws_bytes(int n, int max_keys, int H) {
    const size_t r = x_rows(n, max_keys), sl = x_slots(n, max_keys, H);
    return x_hdr_bytes(n) + spd_al256(r * H * XDN * 2) + spd_al256(r * H * XDV * 2) + spd_al256(r * XDR * 2) +
           spd_al256(r * XDC * 2) + x_cnt_bytes(sl) + x_part_bytes(sl);
}

// s_off[i] = sum_{i' < i} val(i') (exclusive scan over the block; every thread takes a
// contiguous range of requests)
template <typename V>
__device__ void x_scan(V val, int n, int* s_off, int* s_warp) {
    const int T = blockDim.x, tid = threadIdx.x;
    const int per = (n + T - 1) / T;
    const int a = min(n, tid * per), b = min(n, a + per);
    int sum = 0;
    for (int i = a; i < b; ++i) sum += val(i);
    const int lane = tid & 31, w = tid >> 5;
    int inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) s_warp[w] = inc;
    __syncthreads();
    if (tid == 0) {
        int acc = 0;
        for (int k = 0; k < T / 32; ++k) {
            const int v = s_warp[k];
            s_warp[k] = acc;
            acc += v;
        }
    }
    __syncthreads();
    int run = s_warp[w] + inc - sum;  // exclusive prefix of this thread's range
    if (tid == 0) s_off[0] = 0;
    for (int i = a; i < b; ++i) {
        run += val(i);
        s_off[i + 1] = run;
    }
    __syncthreads();
}

// largest i in [0, n) with off[i] <= x (off non-decreasing, off[0] = 0)
template <typename F>
__device__ __forceinline__ int x_find(F off, int n, int x) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off(mid) <= x) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// ------------------------------------------------------------------ 1. prep
struct XPrep {
    const int* cu;
    const int* req_ids;
    const int* prefix;
    const int* bt;
    const uint4* kv_new;     // [T][576] bf16
    unsigned char* pool;     // this layer's latent pages [N_B][bs][576]
    uint4* kpe;              // [rows][64] bf16
    uint4* lat;              // [rows][512] bf16: every key's latent c_j, contiguous (GEMM A)
    int* hdr;
    int* status;
    int n, lg_bs, MBR, N_B, H;
    int T;               // total_q: chunk rows of kv_new
    long long rows_cap;  // workspace rows (max_total_keys + 128 n)
    long long slots_cap; // split slots of the workspace
    int* cnt;            // split counters / flags [slots][2][2]
    unsigned long long* span;
};

__global__ void __launch_bounds__(1024) mla_exp_prep_kernel(XPrep p) {
    // per-request metadata in smem (every CTA loads and scans it; n <= 1024 requests): chunk
    // offsets, prefixes and block-table rows first (coalesced), then the tile-offset scan
    __shared__ int s_off[XMAXN + 1];
    __shared__ int s_cu[XMAXN + 1];
    __shared__ int s_P[XMAXN];
    __shared__ int s_rid[XMAXN];
    __shared__ int s_warp[32];
    pdl_wait();  // PDL: the previous kernel on this stream (it may read this workspace) is complete
    if (threadIdx.x == 0) span_begin(p.span);
    for (int i = threadIdx.x; i <= p.n; i += blockDim.x) {
        s_cu[i] = __ldg(p.cu + i);
        if (i < p.n) {
            s_P[i] = __ldg(p.prefix + i);
            s_rid[i] = __ldg(p.req_ids + i);
        }
    }
    __syncthreads();
    long long n_slots = 0;
    if constexpr (kXSplit) {  // split-pair offsets first (s_off is reused for the tile offsets)
        x_scan([&](int i) { return x_split_pairs(s_P[i], s_cu[i + 1] - s_cu[i]); }, p.n, s_off, s_warp);
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i <= p.n; i += blockDim.x) p.hdr[p.n + 1 + i] = s_off[i];
        n_slots = (long long)s_off[p.n] * p.H;
        __syncthreads();
    } else if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i <= p.n; i += blockDim.x) p.hdr[p.n + 1 + i] = 0;
    }
    x_scan([&](int i) { return (s_P[i] + s_cu[i + 1] - s_cu[i] + XBM - 1) / XBM; }, p.n, s_off, s_warp);
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i <= p.n; i += blockDim.x) p.hdr[i] = s_off[i];
    const int R = s_off[p.n] * XBM;
    if (R > p.rows_cap || n_slots > p.slots_cap) {  // max_total_keys was too small: write nothing
        if (threadIdx.x == 0) {
            if (p.status) atomicMax(p.status, SEMIPD_ERR_INVALID);
            span_end(p.span);
        }
        return;
    }
    const int bs_mask = (1 << p.lg_bs) - 1;
    constexpr int RU = XDL * 2 / 16;  // 72 uint4 per latent row
    constexpr int PU = XDR * 2 / 16;  // 8 uint4 of k_pe
    const int lane = threadIdx.x & 31;
    const int nw = gridDim.x * (blockDim.x >> 5);
    const uint4 zero = make_uint4(0u, 0u, 0u, 0u);
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < 4 * n_slots;
         k += (long long)gridDim.x * blockDim.x)
        p.cnt[k] = 0;  // this call's split counters / flags
    // one warp per padded key row, two rows in flight per warp: the chunk's latent rows go to the
    // pool; every key's latent to Lat (the GEMM's contiguous A) and its k_pe to Kpe
    // (chunk keys from kv_new, prefix keys from the pool, padding / bad-block rows zero)
    constexpr int LU = XDC * 2 / 16;  // 64 uint4 of c_j
    for (int g0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); g0 < R; g0 += 2 * nw) {
        uint4 v[2][3];
        uint4* prow[2];
        int kind[2];  // -1: beyond R, 0: padding / bad block, 1: chunk row, 2: prefix row
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int g = g0 + u * nw;
            kind[u] = g < R ? 0 : -1;
            prow[u] = nullptr;
            if (g >= R) continue;
            const int i = x_find([&](int q) { return s_off[q]; }, p.n, g / XBM);
            const int j = g - s_off[i] * XBM;
            const int P = s_P[i], c0 = s_cu[i], nk = P + s_cu[i + 1] - c0;
            if (j >= nk) continue;
            const int page = j >> p.lg_bs;
            const int blk = page < p.MBR ? __ldg(p.bt + (size_t)s_rid[i] * p.MBR + page) : -1;
            if (blk < 0 || blk >= p.N_B) {
                if (lane == 0 && p.status) atomicMax(p.status, SEMIPD_ERR_BAD_BLOCK);
                continue;
            }
            if (j >= P && c0 + j - P >= p.T) {  // cu_seqlens_q beyond the host's total_q
                if (lane == 0 && p.status) atomicMax(p.status, SEMIPD_ERR_INVALID);
                continue;
            }
            prow[u] = reinterpret_cast<uint4*>(p.pool + ((size_t)blk * (bs_mask + 1) + (j & bs_mask)) * (XDL * 2));
            const uint4* src = j >= P ? p.kv_new + (size_t)(c0 + j - P) * RU : prow[u];
            kind[u] = j >= P ? 1 : 2;
#pragma unroll
            for (int r3 = 0; r3 < 3; ++r3)
                if (lane + 32 * r3 < RU) v[u][r3] = j >= P ? __ldg(src + lane + 32 * r3) : src[lane + 32 * r3];
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (kind[u] < 0) continue;
            const size_t g = (size_t)g0 + u * nw;
            uint4* ld = p.lat + g * LU;
            uint4* kd = p.kpe + g * PU;
#pragma unroll
            for (int r3 = 0; r3 < 3; ++r3) {
                const int c = lane + 32 * r3;
                if (c < RU) {
                    const uint4 x = kind[u] > 0 ? v[u][r3] : zero;
                    if (kind[u] == 1) prow[u][c] = x;
                    if (c < LU) ld[c] = x;
                    else kd[c - LU] = x;
                }
            }
        }
    }
    pdl_trigger();
    __syncthreads();
    if (threadIdx.x == 0) span_end(p.span);
}

// ------------------------------------------------------------------ 2. up-projection GEMM
constexpr int GCB = 2;                        // 64-column blocks per stage
constexpr int GST = 2;                        // stages in flight
constexpr uint32_t GA = XBM * 128 * GCB;      // A stage: 128 rows x 128 cols (32 KiB, one box)
constexpr uint32_t GB = 256 * 128 * GCB;      // B stage: 256 rows x 128 cols (64 KiB, one box)
constexpr int GNT = 192;

struct GSmem {
    unsigned char a[GST][GA];
    unsigned char b[GST][GB];
    uint64_t full[GST], empty[GST], accf[2], acce[2];
    uint32_t tmem_base;
};

struct XGemm {
    const int* cu;
    const int* req_ids;
    const int* prefix;
    const int* bt;
    const int* hdr;
    __nv_bfloat16* kexp;
    __nv_bfloat16* vexp;
    int* status;
    unsigned long long* span;
    int n, H, lg_bs, box_rows, MBR, N_B;
    long long rows_cap;
};

__device__ __forceinline__ uint64_t xk_desc(uint32_t addr) { return umma_desc_sw128(addr, 16, 1024); }

__global__ void __launch_bounds__(GNT, 1)
    mla_exp_gemm_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap ukmap,
                        const __grid_constant__ CUtensorMap uvmap, XGemm p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    GSmem& sm = *reinterpret_cast<GSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = (int)warp_id(), lane = (int)lane_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < GST; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.accf[s], 1);
            mbar_init(&sm.acce[s], 128);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // PDL: the prep kernel (Lat, hdr) is complete
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = sm.tmem_base;
    const int MT = __ldg(p.hdr + p.n);
    const int NTN = p.H;  // n tiles of 256 columns: H / 2 head pairs of K_nope, then of V
    // rows beyond the workspace: INVALID was set by the prep kernel; no tiles
    const int total = (long long)MT * XBM > p.rows_cap ? 0 : MT * NTN;
    auto off = [&](int k) { return __ldg(p.hdr + k); };

    if (warp == 0) {
        // ================================ TMA producer ================================
        if (lane == 0) {
            tma_prefetch_desc(&amap);
            tma_prefetch_desc(&ukmap);
            tma_prefetch_desc(&uvmap);
        }
        int sc = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
            const int mt = tile / NTN, nt = tile % NTN;
            const CUtensorMap* bm = nt < NTN / 2 ? &ukmap : &uvmap;
            const int brow = (nt % (NTN / 2)) * 256;
            for (int ks = 0; ks < XDC / (64 * GCB); ++ks, ++sc) {
                const int s = sc % GST;
                if (lane == 0) {
                    mbar_wait(&sm.empty[s], ((sc / GST) & 1) ^ 1);
                    mbar_arrive_expect_tx(&sm.full[s], GA + GB);
                    // (64 cols, rows, column blocks) boxes land as [block][rows][128 B]
                    tma_load_3d(sm.a[s], &amap, &sm.full[s], 0, mt * XBM, ks * GCB);
                    tma_load_3d(sm.b[s], bm, &sm.full[s], 0, brow, ks * GCB);
                }
                __syncwarp();
            }
        }
        pdl_trigger();  // every tile's loads issued: the attention kernel may be scheduled
    } else if (warp == 1) {
        // ================================ MMA issuer ================================
        const uint32_t idesc = umma_idesc_bf16_f32(XBM, 256, 0);
        int sc = 0, lt = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++lt) {
            const int ab = lt & 1;
            mbar_wait(&sm.acce[ab], ((lt >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)(ab * 256);
            for (int ks = 0; ks < XDC / (64 * GCB); ++ks, ++sc) {
                const int s = sc % GST;
                mbar_wait(&sm.full[s], (sc / GST) & 1);
                tc_fence_after();
                const uint64_t da = xk_desc(smem_u32(sm.a[s])), db = xk_desc(smem_u32(sm.b[s]));
#pragma unroll
                for (int kk = 0; kk < 4 * GCB; ++kk) {
                    const int cb = kk >> 2;
                    umma_ss_warp(d, da + (uint64_t)((cb * XBM * 128 + (kk & 3) * 32) >> 4),
                                 db + (uint64_t)((cb * 256 * 128 + (kk & 3) * 32) >> 4), idesc,
                                 (ks | kk) ? 1u : 0u);
                }
                umma_commit_warp(&sm.empty[s]);
            }
            umma_commit_warp(&sm.accf[ab]);
        }
    } else {
        // ============ epilogue (warps 2-5): fp32 TMEM -> bf16 (RNE) -> K_exp / V_exp ============
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        int lt = 0;
        for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++lt) {
            const int ab = lt & 1;
            const int mt = tile / NTN, nt = tile % NTN;
            const int i = x_find(off, p.n, mt);
            const int kbase = (mt - off(i)) * XBM;
            const int nk = __ldg(p.prefix + i) + __ldg(p.cu + i + 1) - __ldg(p.cu + i);
            const bool valid = kbase + r < nk;
            const size_t row = (size_t)mt * XBM + r;
            __nv_bfloat16* base = nt < NTN / 2 ? p.kexp : p.vexp;
            const int h0 = (nt % (NTN / 2)) * 2;
            mbar_wait(&sm.accf[ab], (lt >> 1) & 1);
            tc_fence_after();
#pragma unroll 2
            for (int c = 0; c < 8; ++c) {
                uint32_t v[32];
                tmem_ld32(tmem + lane_base + (uint32_t)(ab * 256 + c * 32), v);
                tmem_wait_ld();
                uint4* dst = reinterpret_cast<uint4*>(base + (row * p.H + h0 + (c >> 2)) * XDN + (c & 3) * 32);
#pragma unroll
                for (int e = 0; e < 32; e += 8) {
                    uint4 o = make_uint4(0u, 0u, 0u, 0u);
                    if (valid) {
                        o.x = pack_bf16(__uint_as_float(v[e + 0]), __uint_as_float(v[e + 1]));
                        o.y = pack_bf16(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                        o.z = pack_bf16(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
                        o.w = pack_bf16(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
                    }
                    dst[e / 8] = o;
                }
            }
            tc_fence_before();
            mbar_arrive(&sm.acce[ab]);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
    if (threadIdx.x == 0) span_end(p.span);
}

// ------------------------------------------------------------------ 2'. up-projection GEMM, A in TMEM
// The same product with the latent tile held in TMEM (the MMA's A operand, K packed two bf16 per
// column: cols [0, 256)) and only W streamed through shared memory, so each SM ingests 128 B of
// operands per 128 x 128 x 16 MMA (64 cycles) instead of the SS form's 48 KiB per 512 cycles.
// Work item = (128-key m-tile, XG consecutive 128-column n-tiles = XG heads of K or V); the
// epilogue warps stage the item's A rows (global -> registers -> tcgen05.st) and then drain the
// double-buffered 128-column accumulators (cols [256, 512)); while an item's n-tiles run they
// already hold the first half of the next item's rows in registers.
// SPD_X_GEMM_TA = 1 selects this kernel.  Parity-green (33/33) but measured SLOWER than the SS
// GEMM at every budget (C = 2048, P = 0: 241 / 365 / 655 vs 283 / 414 / 740 TFLOP/s at 44 / 74 /
// 148 SMs; profiles/r2_mla_expanded_gemm_ta_ab.log): the A staging between items (a global load
// round trip and 8 TMEM stores per thread, the MMA idle meanwhile) and the N = 128 tiles cost more
// than the halved operand traffic gains.  Default 0.
#ifndef SPD_X_GEMM_TA
#define SPD_X_GEMM_TA 0
#endif
constexpr bool kXGemmTA = SPD_X_GEMM_TA != 0;
constexpr int XG = 4;                         // n-tiles (heads) per work item
constexpr int TCB = 2;                        // 64-column blocks per B stage
constexpr int TST = 6;                        // B stages in flight
constexpr uint32_t TB = 128 * 128 * TCB;      // B stage: 128 rows x 128 cols (32 KiB, one box)

struct TSmem {
    unsigned char b[TST][TB];
    uint64_t full[TST], empty[TST], dfull[2], dempty[2], a_full, a_free;
    uint32_t tmem_base;
};

__global__ void __launch_bounds__(GNT, 1)
    mla_exp_gemm_ta_kernel(const __grid_constant__ CUtensorMap ukmap, const __grid_constant__ CUtensorMap uvmap,
                           const uint4* __restrict__ lat, XGemm p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    TSmem& sm = *reinterpret_cast<TSmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = (int)warp_id(), lane = (int)lane_id();
    if (threadIdx.x == 0) {
        for (int s = 0; s < TST; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.dfull[s], 1);
            mbar_init(&sm.dempty[s], 128);
        }
        mbar_init(&sm.a_full, 128);
        mbar_init(&sm.a_free, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = sm.tmem_base;
    const int MT = __ldg(p.hdr + p.n);
    const int NG = 2 * p.H / XG;  // items per m-tile
    const int total = (long long)MT * XBM > p.rows_cap ? 0 : MT * NG;
    constexpr int KS = XDC / (64 * TCB);  // B stages per n-tile

    if (warp == 0) {
        // ================================ TMA producer (W rows) ================================
        if (lane == 0) {
            tma_prefetch_desc(&ukmap);
            tma_prefetch_desc(&uvmap);
        }
        int sc = 0;
        for (int it = blockIdx.x; it < total; it += gridDim.x) {
            const int g = it % NG;
            for (int j = 0; j < XG; ++j) {
                const int nt = g * XG + j;  // < H: K head nt; else V head nt - H
                const CUtensorMap* bm = nt < p.H ? &ukmap : &uvmap;
                const int brow = (nt < p.H ? nt : nt - p.H) * XDN;
                for (int ks = 0; ks < KS; ++ks, ++sc) {
                    const int s = sc % TST;
                    if (lane == 0) {
                        mbar_wait(&sm.empty[s], ((sc / TST) & 1) ^ 1);
                        mbar_arrive_expect_tx(&sm.full[s], TB);
                        tma_load_3d(sm.b[s], bm, &sm.full[s], 0, brow, ks * TCB);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // ================================ MMA issuer (A from TMEM) ================================
        const uint32_t idesc = umma_idesc_bf16_f32(XBM, XDN, 0);
        int sc = 0, dt = 0, li = 0;
        for (int it = blockIdx.x; it < total; it += gridDim.x, ++li) {
            mbar_wait(&sm.a_full, li & 1);
            tc_fence_after();
            for (int j = 0; j < XG; ++j, ++dt) {
                const int db = dt & 1;
                mbar_wait(&sm.dempty[db], ((dt >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + 256u + (uint32_t)(db * XDN);
                for (int ks = 0; ks < KS; ++ks, ++sc) {
                    const int s = sc % TST;
                    mbar_wait(&sm.full[s], (sc / TST) & 1);
                    tc_fence_after();
                    const uint32_t bl = desc_lo(smem_u32(sm.b[s]), 16);
#pragma unroll
                    for (int kk = 0; kk < 4 * TCB; ++kk)
                        umma_ts_warp2(d, tmem + (uint32_t)(ks * 64 + kk * 8),
                                      bl + (uint32_t)(((kk >> 2) * 128 * 128 + (kk & 3) * 32) >> 4), DESC_HI_SBO1K,
                                      idesc, (ks | kk) ? 1u : 0u);
                    umma_commit_warp(&sm.empty[s]);
                }
                umma_commit_warp(&sm.dfull[db]);
            }
            umma_commit_warp(&sm.a_free);  // every MMA of the item done: A may be replaced
        }
    } else {
        // ===== warps 2-5: stage A rows into TMEM, drain the accumulators (fp32 -> bf16 RNE) =====
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        constexpr int LU = XDC * 2 / 16;  // 64 uint4 per latent row
        uint4 nxt[LU / 2];                // first half of the next item's row
        auto load_half = [&](int it, int h, uint4 (&v)[LU / 2]) {
            const uint4* src = lat + ((size_t)(it / NG) * XBM + r) * LU + h * (LU / 2);
#pragma unroll
            for (int c = 0; c < LU / 2; ++c) v[c] = __ldg(src + c);
        };
        auto store_half = [&](int h, const uint4 (&v)[LU / 2]) {  // 32 uint4 = 128 columns
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t w[32];
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    w[4 * e + 0] = v[c * 8 + e].x;
                    w[4 * e + 1] = v[c * 8 + e].y;
                    w[4 * e + 2] = v[c * 8 + e].z;
                    w[4 * e + 3] = v[c * 8 + e].w;
                }
                tmem_st32(tmem + lane_base + (uint32_t)(h * 128 + c * 32), w);
            }
        };
        // A of item `it` into TMEM: the prefetched first half + the second half loaded now
        auto stage = [&](int it) {
            uint4 h1[LU / 2];
            load_half(it, 1, h1);
            store_half(0, nxt);
            store_half(1, h1);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&sm.a_full);
            if (it + (int)gridDim.x < total) load_half(it + gridDim.x, 0, nxt);
        };
        int dt = 0;
        if (blockIdx.x < total) {
            load_half(blockIdx.x, 0, nxt);
            stage(blockIdx.x);
        }
        for (int it = blockIdx.x; it < total; it += gridDim.x) {
            const int mt = it / NG, g = it % NG;
            const int i = x_find([&](int k) { return __ldg(p.hdr + k); }, p.n, mt);
            const int kbase = (mt - __ldg(p.hdr + i)) * XBM;
            const int nk = __ldg(p.prefix + i) + __ldg(p.cu + i + 1) - __ldg(p.cu + i);
            const bool valid = kbase + r < nk;
            const size_t row = (size_t)mt * XBM + r;
            for (int j = 0; j < XG; ++j, ++dt) {
                const int db = dt & 1;
                const int nt = g * XG + j;
                __nv_bfloat16* base = nt < p.H ? p.kexp : p.vexp;
                const int h = nt < p.H ? nt : nt - p.H;
                mbar_wait(&sm.dfull[db], (dt >> 1) & 1);
                tc_fence_after();
                if (j == XG - 1 && it + (int)gridDim.x < total) {
                    // the item's last accumulator is complete, so are all its MMAs: the next
                    // item's A goes in first (the MMA warp restarts on the other accumulator)
                    mbar_wait(&sm.a_free, ((dt / XG) & 1));
                    stage(it + gridDim.x);
                }
                uint4* dst = reinterpret_cast<uint4*>(base + (row * p.H + h) * XDN);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t v[32];
                    tmem_ld32(tmem + lane_base + (uint32_t)(256 + db * XDN + c * 32), v);
                    tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 32; e += 8) {
                        uint4 o = make_uint4(0u, 0u, 0u, 0u);
                        if (valid) {
                            o.x = pack_bf16(__uint_as_float(v[e + 0]), __uint_as_float(v[e + 1]));
                            o.y = pack_bf16(__uint_as_float(v[e + 2]), __uint_as_float(v[e + 3]));
                            o.z = pack_bf16(__uint_as_float(v[e + 4]), __uint_as_float(v[e + 5]));
                            o.w = pack_bf16(__uint_as_float(v[e + 6]), __uint_as_float(v[e + 7]));
                        }
                        dst[c * 4 + e / 8] = o;
                    }
                }
                tc_fence_before();
                mbar_arrive(&sm.dempty[db]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
    if (threadIdx.x == 0) span_end(p.span);
}

// ------------------------------------------------------------------ 3. attention
constexpr int ANT = 384;
constexpr int NSLOT = 8;
constexpr uint32_t SLOT = XBM * 128;          // 16 KiB: 128 rows x 64 columns
constexpr uint32_t QCH = 2 * SLOT;            // one 64-column chunk of the Q pair (tiles A, B)
constexpr int kXPvParts = 4;
// exp2 pairs of each 32-column S block on the FMA pipe (bit i = columns 2i, 2i + 1), as the GQA
// prefill kernel's SPD_POLY_MASK
#ifndef SPD_X_POLY
#define SPD_X_POLY 0x1111u
#endif

struct XUnit {
    int i, h, t0, P, qrow0, krow0;
    int tv[2], nkv[2];  // nkv[t]: one past the last kv tile of tile t in this part
    int kv0;            // first kv tile of this part
    int slot;           // split slot (-1: unsplit unit)
    int part;
    int single;         // 1: tile A alone (a q tile of a split row); tile B idle
};

struct ASmem {
    unsigned char q[3][QCH];                  // [chunk][tile A rows | tile B rows][128 B]
    unsigned char ring[NSLOT][SLOT];
    uint64_t q_full, q_empty;
    uint64_t full[NSLOT], empty[NSLOT];
    uint64_t s_full[2], p_full[2][kXPvParts];
    uint64_t o_full[2], o_empty[2];
    uint64_t ufull[2], uempty[2];
    XUnit units[2];
    int role[2];  // per softmax warpgroup: the split counter's old value
    uint32_t tmem_base;
};

struct XAttn {
    const int* cu;
    const int* prefix;
    const int* hdr;
    __nv_bfloat16* out;
    int* status;
    unsigned long long* span;
    unsigned* sched;
    int single_rows;  // the longest `single_rows` pair rows run as two single-tile units each
    float* part;  // split partials [slots][2 tiles][128 rows][XPROW]
    int* cnt;     // split counters [slots][2 tiles][role counter, flag]
    int n, T, H, pairs_max, n_units;
    float scale_log2;
    SpdTrace trace;
};

// Epilogue of one split part.  The warpgroup's thread 0 takes a role from the slot's counter:
// the part that arrives first stores its unnormalised O rows (relative to 2^m) with (m, l) to
// rows[r] and raises the slot's flag (release); the second waits for the flag (acquire), reads
// those rows and merges them with its own O (still in TMEM).  Both weights and the sum are
// formed without contraction, so the result does not depend on which part came first.  TMEM's
// O is released (o_empty) as soon as this warpgroup has read it.
__device__ __forceinline__ void x_split_epilogue(float* rows, int* ctr, int* role, uint64_t* o_empty,
                                                 uint32_t o_tmem, int r, int t, float m, float l, bool valid,
                                                 uint4* dst) {
    if (r == 0) *role = atomicAdd(ctr, 1);
    named_bar_sync(2 + t, 128);
    const int rl = *role;
    float4* row = reinterpret_cast<float4*>(rows + (size_t)r * XPROW);
    if (rl == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tmem_ld32(o_tmem + c * 32, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; e += 4)
                row[c * 8 + e / 4] = make_float4(__uint_as_float(o[e]), __uint_as_float(o[e + 1]),
                                                 __uint_as_float(o[e + 2]), __uint_as_float(o[e + 3]));
        }
        tc_fence_before();
        mbar_arrive(o_empty);
        row[XDV / 4] = make_float4(m, l, 0.f, 0.f);
        named_bar_sync(2 + t, 128);
        if (r == 0) {
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(ctr + 1), "r"(1) : "memory");
        }
        return;
    }
    if (r == 0) {
        int f = 0;
        do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(ctr + 1) : "memory");
            if (!f) __nanosleep(64);
        } while (!f);
    }
    named_bar_sync(2 + t, 128);
    const float4 ml = __ldcg(row + XDV / 4);
    const float mm = fmaxf(ml.x, m);
    const float fo = fast_exp2(ml.x - mm), fm = fast_exp2(m - mm);
    const float inv = 1.f / __fadd_rn(__fmul_rn(ml.y, fo), __fmul_rn(l, fm));
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        float4 ot[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) ot[k] = __ldcg(row + c * 8 + k);
        uint32_t o[32];
        tmem_ld32(o_tmem + c * 32, o);
        tmem_wait_ld();
        if (c == 3) {
            tc_fence_before();
            mbar_arrive(o_empty);
        }
        auto mg = [&](float mine, float other) {
            return __fmul_rn(__fadd_rn(__fmul_rn(mine, fm), __fmul_rn(other, fo)), inv);
        };
        if (valid) {
#pragma unroll
            for (int k = 0; k < 8; k += 2) {
                const float* a = reinterpret_cast<const float*>(&ot[k]);
                uint4 v;
                v.x = pack_bf16(mg(__uint_as_float(o[4 * k + 0]), a[0]), mg(__uint_as_float(o[4 * k + 1]), a[1]));
                v.y = pack_bf16(mg(__uint_as_float(o[4 * k + 2]), a[2]), mg(__uint_as_float(o[4 * k + 3]), a[3]));
                v.z = pack_bf16(mg(__uint_as_float(o[4 * k + 4]), a[4]), mg(__uint_as_float(o[4 * k + 5]), a[5]));
                v.w = pack_bf16(mg(__uint_as_float(o[4 * k + 6]), a[6]), mg(__uint_as_float(o[4 * k + 7]), a[7]));
                dst[c * 4 + k / 2] = v;
            }
        }
    }
    if (r == 0) {  // ready for the next call
        ctr[0] = 0;
        ctr[1] = 0;
    }
}

__global__ void __launch_bounds__(ANT, 1)
    mla_exp_attn_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kxmap,
                        const __grid_constant__ CUtensorMap vxmap, const __grid_constant__ CUtensorMap pemap,
                        XAttn p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    ASmem& sm = *reinterpret_cast<ASmem*>(smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u));
    const int warp = (int)warp_id(), lane = (int)lane_id();
    if (threadIdx.x == 0) {
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_empty, 1);
        for (int s = 0; s < NSLOT; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.s_full[s], 1);
            for (int h = 0; h < kXPvParts; ++h) mbar_init(&sm.p_full[s][h], 128);
            mbar_init(&sm.o_full[s], 1);
            mbar_init(&sm.o_empty[s], 128);
            mbar_init(&sm.ufull[s], 1);
            mbar_init(&sm.uempty[s], 1 + 8);  // MMA warp + 8 softmax warps
        }
        fence_mbar_init();
        if (p.trace.buf) {
            int slot = atomicAdd(p.trace.ctr, 1);
            if (slot < p.trace.cap)
                reinterpret_cast<int4*>(p.trace.buf)[slot] =
                    make_int4(1, (int)smid(), (int)blockIdx.x, 10 /* kernel kind: expanded MLA prefill */);
        }
    }
    if (warp == 1) tmem_alloc(&sm.tmem_base, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // PDL: the GEMM (K_exp, V_exp) and prep (Kpe, hdr) are complete
    if (threadIdx.x == 0) span_begin(p.span);
    const uint32_t tmem = sm.tmem_base;

    if (warp < 4) {
        setmaxnreg_dec<72>();
        if (warp == 0) {
            // ====================== producer: units, Q pair, K / V slots ======================
            if (lane == 0) {
                tma_prefetch_desc(&qmap);
                tma_prefetch_desc(&kxmap);
                tma_prefetch_desc(&vxmap);
                tma_prefetch_desc(&pemap);
            }
            int sc = 0, nunit = 0;
            for (;;) {
                const int us = nunit & 1;
                XUnit d;
                d.i = -1;
                int u = 0;
                if (lane == 0) u = (int)atomicAdd(p.sched, 1u);
                u = __shfl_sync(0xffffffffu, u, 0);
                if (u < p.n_units) {
                    // u -> (slot v = (pair, part), request, head); LPT: last pairs first
                    const int per_pair = p.n * p.H;
                    // units: first the q tiles of the `single_rows` longest pair rows as single-
                    // tile units (last tile first), then the remaining pair rows (last first)
                    const int ns = 2 * p.single_rows * per_pair;
                    const bool single = u < ns;
                    const int uu = single ? u : u - ns;
                    const int v = uu / per_pair;
                    const int pair = single ? p.pairs_max - 1 - (v >> 1)
                                            : p.pairs_max - 1 - p.single_rows - (kXSplit ? v >> 1 : v);
                    const int part = kXSplit && !single ? v & 1 : 0;
                    d.i = (uu / p.H) % p.n;
                    d.h = uu % p.H;
                    const int c0 = __ldg(p.cu + d.i), C = __ldg(p.cu + d.i + 1) - c0;
                    d.t0 = single ? (2 * pair + 1 - (v & 1)) * XBM : pair * 2 * XBM;
                    if (d.t0 >= C) continue;  // tile / pair past this request's chunk (warp-uniform)
                    d.single = single;
                    d.tv[0] = min(XBM, C - d.t0);
                    d.tv[1] = single ? 0 : max(0, min(XBM, C - d.t0 - XBM));
                    d.P = __ldg(p.prefix + d.i);
                    const int nA = (d.P + d.t0 + d.tv[0] - 1) / XBM + 1;
                    const int nB = d.tv[1] > 0 ? (d.P + d.t0 + XBM + d.tv[1] - 1) / XBM + 1 : nA;
                    const bool split = !single && x_pair_nkv(d.P, C, pair) >= XSPLIT_MIN;
                    if (!split && part) continue;
                    d.part = part;
                    if (split) {  // nB >= 10 and nA >= nB - 1: both tiles keep >= 1 kv tile per part
                        const int hk = nB / 2;
                        d.kv0 = part ? hk : 0;
                        d.nkv[0] = part ? nA : hk;
                        d.nkv[1] = part ? nB : hk;
                        const int sb = __ldg(p.hdr + p.n + 1 + d.i) + pair - x_first_split_pair(d.P, C);
                        d.slot = sb * p.H + d.h;
                    } else {
                        d.kv0 = 0;
                        d.nkv[0] = nA;
                        d.nkv[1] = nB;
                        d.slot = -1;
                    }
                    d.qrow0 = c0 + d.t0;
                    d.krow0 = __ldg(p.hdr + d.i) * XBM;
                }
                if (lane == 0) {
                    mbar_wait(&sm.uempty[us], ((nunit >> 1) & 1) ^ 1);
                    sm.units[us] = d;
                    mbar_arrive(&sm.ufull[us]);
                }
                __syncwarp();
                if (d.i < 0) {  // no more units: the next kernel on the stream may be scheduled
                    pdl_trigger();
                    break;
                }
                if (lane == 0) {
                    mbar_wait(&sm.q_empty, (nunit & 1) ^ 1);
                    // (64 cols, head h, 256 tokens, 3 chunks) -> [chunk][A rows | B rows][128 B]
                    mbar_arrive_expect_tx(&sm.q_full, 3 * QCH);
                    tma_load_4d(sm.q[0], &qmap, &sm.q_full, 0, d.h, d.qrow0, 0);
                }
                ++nunit;
                for (int j = d.kv0; j < d.nkv[1]; ++j) {
                    const int krow = d.krow0 + j * XBM;
                    // kv tile j = K slots (k_nope cols 0-63, 64-127, k_pe) then V slots (0-63, 64-127)
#pragma unroll 1
                    for (int c = 0; c < 5; ++c, ++sc) {
                        if (lane == 0) {
                            const int s = sc % NSLOT;
                            mbar_wait(&sm.empty[s], ((sc / NSLOT) & 1) ^ 1);
                            mbar_arrive_expect_tx(&sm.full[s], SLOT);
                            if (c < 2)
                                tma_load_3d(sm.ring[s], &kxmap, &sm.full[s], c * 64, d.h, krow);
                            else if (c == 2)
                                tma_load_3d(sm.ring[s], &pemap, &sm.full[s], 0, krow, 0);
                            else
                                tma_load_3d(sm.ring[s], &vxmap, &sm.full[s], (c - 3) * 64, d.h, krow);
                        }
                    }
                    __syncwarp();
                }
            }
        } else if (warp == 1) {
            // ================================ MMA issuer ================================
            const uint32_t idesc_s = umma_idesc_bf16_f32(XBM, XBM, 0);
            const uint32_t idesc_o = umma_idesc_bf16_f32(XBM, XDV, 1);
            const uint32_t idesc_o64 = umma_idesc_bf16_f32(XBM, 64, 1);
            int sc = 0, nunit = 0, cnt_a = 0, cnt_b = 0;
            int npair = 0;  // pair units so far: the phase of tile B's o_empty (single units skip B)
            auto wait_slot = [&](int c) { mbar_wait(&sm.full[c & (NSLOT - 1)], (c / NSLOT) & 1); };
            auto release = [&](int c0, int k) {
                for (int e = 0; e < k; ++e) umma_commit_warp(&sm.empty[(c0 + e) & (NSLOT - 1)]);
            };
            for (;;) {
                const int us = nunit & 1;
                mbar_wait(&sm.ufull[us], (nunit >> 1) & 1);
                const XUnit d = sm.units[us];
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.uempty[us]);
                if (d.i < 0) break;
                mbar_wait(&sm.q_full, nunit & 1);
                tc_fence_after();
                const int nA = d.nkv[0], nB = d.nkv[1];
                const uint32_t q_base = smem_u32(sm.q[0]);
                const uint32_t ring_a = smem_u32(sm.ring[0]);
                // smem descriptors as (low, high) words: low = start >> 4 | LBO >> 4 << 16 (the K16
                // steps add 16-byte offsets to it), high = SBO 1 KiB, version 1, 128-byte swizzle
                constexpr uint32_t DHI = (1024u >> 4) | (1u << 14) | (2u << 29);
                auto dlo = [](uint32_t addr, uint32_t lbo) { return (addr >> 4) | ((lbo >> 4) << 16); };
                auto issue_s = [&](int t, int kc) {  // S_t = Q_t [k_nope | k_pe]^T, 12 x K16
                    const uint32_t qd = dlo(q_base + t * SLOT, 16);
                    uint32_t kd[3];
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) kd[ch] = dlo(ring_a + ((kc + ch) & (NSLOT - 1)) * SLOT, 16);
#pragma unroll
                    for (int kk = 0; kk < 12; ++kk) {
                        const int ch = kk >> 2;
                        umma_ss_warp2(tmem + (uint32_t)(t * XBM), qd + ((ch * QCH + (kk & 3) * 32) >> 4), DHI,
                                      kd[ch] + (((kk & 3) * 32) >> 4), DHI, idesc_s, kk > 0 ? 1u : 0u);
                    }
                    umma_commit_warp(&sm.s_full[t]);
                };
                auto issue_pv = [&](int t, int& cnt, int vc, bool first) {  // O_t += P_t V
                    const int s0 = vc & (NSLOT - 1), s1 = (vc + 1) & (NSLOT - 1);
                    const uint32_t vd0 = dlo(ring_a + s0 * SLOT, SLOT), vd1 = dlo(ring_a + s1 * SLOT, SLOT);
                    const uint32_t p_tmem = tmem + (uint32_t)(t * XBM);
                    const uint32_t o_tmem = tmem + 256u + (uint32_t)(t * XDV);
                    if (s1 == s0 + 1) {  // adjacent slots: one N = 128 MMA per K16 (LBO = slot pitch)
#pragma unroll
                        for (int hf = 0; hf < kXPvParts; ++hf) {
                            mbar_wait(&sm.p_full[t][hf], cnt & 1);
                            tc_fence_after();
#pragma unroll
                            for (int kk = hf * 8 / kXPvParts; kk < (hf + 1) * 8 / kXPvParts; ++kk)
                                umma_ts_warp2(o_tmem, p_tmem + (uint32_t)(kk * 8), vd0 + kk * (2048 >> 4), DHI,
                                              idesc_o, (first && kk == 0) ? 0u : 1u);
                        }
                    } else {  // ring wrap: the two 64-column halves as N = 64 MMAs
#pragma unroll
                        for (int hf = 0; hf < kXPvParts; ++hf) {
                            mbar_wait(&sm.p_full[t][hf], cnt & 1);
                            tc_fence_after();
#pragma unroll
                            for (int kk = hf * 8 / kXPvParts; kk < (hf + 1) * 8 / kXPvParts; ++kk) {
                                const uint32_t acc = (first && kk == 0) ? 0u : 1u;
                                umma_ts_warp2(o_tmem, p_tmem + (uint32_t)(kk * 8), vd0 + kk * (2048 >> 4), DHI,
                                              idesc_o64, acc);
                                umma_ts_warp2(o_tmem + 64u, p_tmem + (uint32_t)(kk * 8), vd1 + kk * (2048 >> 4), DHI,
                                              idesc_o64, acc);
                            }
                        }
                    }
                    ++cnt;
                };
                const int c0 = sc, j0 = d.kv0;
                if (d.single) {  // tile A alone: S(j) -> softmax -> PV(j) -> S(j + 1)
                    for (int e = 0; e < 3; ++e) wait_slot(c0 + e);
                    tc_fence_after();
                    issue_s(0, c0);
                    release(c0, 3);
                    if (nA == 1) umma_commit_warp(&sm.q_empty);
                    for (int j = 0; j < nA; ++j) {
                        const int vc = c0 + 5 * j + 3;
                        wait_slot(vc);
                        wait_slot(vc + 1);
                        tc_fence_after();
                        if (j == 0) mbar_wait(&sm.o_empty[0], (nunit & 1) ^ 1);
                        issue_pv(0, cnt_a, vc, j == 0);
                        release(vc, 2);
                        if (j == nA - 1) {
                            umma_commit_warp(&sm.o_full[0]);
                        } else {
                            const int kn = c0 + 5 * (j + 1);
                            for (int e = 0; e < 3; ++e) wait_slot(kn + e);
                            tc_fence_after();
                            issue_s(0, kn);
                            release(kn, 3);
                            if (j + 1 == nA - 1) umma_commit_warp(&sm.q_empty);
                        }
                    }
                    sc = c0 + 5 * nA;
                    ++nunit;
                    continue;
                }
                for (int e = 0; e < 3; ++e) wait_slot(c0 + e);
                tc_fence_after();
                issue_s(0, c0);
                issue_s(1, c0);
                release(c0, 3);
                if (nB - j0 == 1) umma_commit_warp(&sm.q_empty);
                for (int j = j0; j < nB; ++j) {
                    const int vc = c0 + 5 * (j - j0) + 3;
                    wait_slot(vc);
                    wait_slot(vc + 1);
                    tc_fence_after();
                    if (j < nA) {
                        if (j == j0) mbar_wait(&sm.o_empty[0], (nunit & 1) ^ 1);
                        issue_pv(0, cnt_a, vc, j == j0);
                        if (j == nA - 1) umma_commit_warp(&sm.o_full[0]);
                    }
                    const bool more = j + 1 < nB;
                    const int kn = c0 + 5 * (j + 1 - j0);
                    if (more) {
                        for (int e = 0; e < 3; ++e) wait_slot(kn + e);
                        tc_fence_after();
                    }
                    if (j + 1 < nA) issue_s(0, kn);
                    if (j == j0) mbar_wait(&sm.o_empty[1], (npair & 1) ^ 1);
                    issue_pv(1, cnt_b, vc, j == j0);
                    release(vc, 2);
                    if (j == nB - 1) umma_commit_warp(&sm.o_full[1]);
                    if (more) {
                        issue_s(1, kn);
                        release(kn, 3);
                        if (j + 1 == nB - 1) umma_commit_warp(&sm.q_empty);
                    }
                }
                sc = c0 + 5 * (nB - j0);
                ++npair;
                ++nunit;
            }
        }
        // warps 2, 3: no role
    } else {
        // ============================ softmax warpgroups ============================
        setmaxnreg_inc<216>();
        const int t = (warp - 4) >> 2;  // q tile A (0) or B (1)
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
        const uint32_t s_tmem = tmem + lane_base + (uint32_t)(t * XBM);
        const uint32_t o_tmem = tmem + lane_base + 256u + (uint32_t)(t * XDV);
        const float tsc = p.scale_log2;
        int cnt = 0, nunit = 0;
        int nown = 0;  // units this warpgroup computed (tile B skips single units): o_full phase
        for (;;) {
            const int us = nunit & 1;
            mbar_wait(&sm.ufull[us], (nunit >> 1) & 1);
            // the loop's fields now; the epilogue's are re-read from smem after the loop (fewer
            // registers live across it) and the unit slot is released after that read
            const XUnit& du = sm.units[us];
            if (du.i < 0) {
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.uempty[us]);
                break;
            }
            if (t == 1 && du.single) {  // a single-tile unit: tile B has no work
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.uempty[us]);
                ++nunit;
                continue;
            }
            const int kv0 = du.kv0, dP = du.P;
            const int trel = du.t0 + t * XBM + r;  // chunk-relative token of this row
            const int nkv = du.nkv[t];
            float m = -INFINITY;
            uint64_t l2 = f2(0.f, 0.f);
            for (int j = kv0; j < nkv; ++j, ++cnt) {
                mbar_wait(&sm.s_full[t], cnt & 1);
                tc_fence_after();
                uint32_t sr[4][32];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld32(s_tmem + c * 32, sr[c]);
                tmem_wait_ld();
                // causal, bottom-right aligned: key j * 128 + c <= P + trel
                const int lim = dP + trel - j * XBM;
                if (lim < XBM - 1) {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int e = 0; e < 32; ++e)
                            if (c * 32 + e > lim) sr[c][e] = __float_as_uint(-INFINITY);
                }
                float mxc[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const int k = (c * 16 + e / 2) % 4;
                        mxc[k] = fmax3(mxc[k], __uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1]));
                    }
                const float mx = fmaxf(fmaxf(mxc[0], mxc[1]), fmaxf(mxc[2], mxc[3]));
                const float mtrue = fmaxf(m, mx * tsc);
                // lazy rescale (R21): the reference max moves only when exceeded by > 8 (log2)
                const bool move = j == kv0 || mtrue > m + 8.f;
                if (j > kv0 && __any_sync(0xffffffffu, move)) {
                    const float alpha = move ? fast_exp2(m - mtrue) : 1.f;
                    const uint64_t a2 = f2(alpha, alpha);
#if SPD_X_RESCALE16
#pragma unroll 1
                    for (int c = 0; c < 8; ++c) {  // 16 columns at a time (registers: S is live)
                        uint32_t o[16];
                        tmem_ld16(o_tmem + c * 16, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; e += 2) {
                            float lo, hi;
                            f2_split(fmul2(f2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), a2), lo, hi);
                            o[e] = __float_as_uint(lo);
                            o[e + 1] = __float_as_uint(hi);
                        }
                        tmem_st16(o_tmem + c * 16, o);
                    }
#else
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint32_t o[32];
                        tmem_ld32(o_tmem + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 32; e += 2) {
                            float lo, hi;
                            f2_split(fmul2(f2(__uint_as_float(o[e]), __uint_as_float(o[e + 1])), a2), lo, hi);
                            o[e] = __float_as_uint(lo);
                            o[e + 1] = __float_as_uint(hi);
                        }
                        tmem_st32(o_tmem + c * 32, o);
                    }
#endif
                    l2 = fmul2(l2, a2);
                }
                if (move) m = mtrue;
                const uint64_t nm2 = f2(-m, -m);
                const uint64_t sc2 = f2(tsc, tsc);
                float ls[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    uint32_t pk[16];
#pragma unroll
                    for (int e = 0; e < 32; e += 2) {
                        const uint64_t x2 = ffma2(f2(__uint_as_float(sr[c][e]), __uint_as_float(sr[c][e + 1])), sc2, nm2);
                        float p0, p1;
                        if ((SPD_X_POLY >> (e >> 1)) & 1u) {
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
                    tmem_wait_st();
                    tc_fence_before();
                    mbar_arrive(&sm.p_full[t][c]);
                }
                l2 = fadd2(l2, f2(ls[0] + ls[2], ls[1] + ls[3]));
            }
            // ---- epilogue: O / l -> bf16 -> out [T][H][128] (each thread its 256-byte row)
            mbar_wait(&sm.o_full[t], nown & 1);
            ++nown;
            tc_fence_after();
            XUnit d;
            d.tv[t] = du.tv[t];
            d.qrow0 = du.qrow0;
            d.h = du.h;
            d.slot = du.slot;
            d.part = du.part;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.uempty[us]);
            float la, lb;
            f2_split(l2, la, lb);
            // rows past total_q (a cu_seqlens_q[n] larger than the host's total_q) are not stored
            const bool valid = r < d.tv[t] && d.qrow0 + t * XBM + r < p.T;
            uint4* dst = reinterpret_cast<uint4*>(p.out + ((size_t)(d.qrow0 + t * XBM + r) * p.H + d.h) * XDV);
            if (d.slot < 0) {
                const float inv = 1.f / (la + lb);
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
                            dst[c * 4 + e / 8] = v;
                        }
                    }
                }
            } else {
                x_split_epilogue(p.part + (size_t)(d.slot * 2 + t) * XBM * XPROW, p.cnt + (d.slot * 2 + t) * 2,
                                 &sm.role[t], &sm.o_empty[t], o_tmem, r, t, m, la + lb, valid, dst);
            }
            if (d.slot < 0) {
                tc_fence_before();
                mbar_arrive(&sm.o_empty[t]);
            }
            ++nunit;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
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

// SPD_X_SINGLE: the host picks how many of the longest pair rows run as single-tile units, by a
// makespan model in pair-step units (a pair row r costs 2 r + 2 steps, a lone tile k costs
// SPD_X_SINGLE_COST x (k + 1): one tile's chain without a partner to overlap), minimising
// max(longest unit, total work / grid); a chunk without prefix is assumed.
// Measured (profiles/r2_mla_expanded_single_ab.log): a lone tile's kv step takes about as long
// as a pair step (the S -> softmax -> P V -> S chain is the same; pairing only fills the tensor
// pipe's idle time with the other tile), so single-tile rows shorten the critical path only when
// nothing else is running: -19 % at 148 SMs for a chunk without prefix, +10-15 % at 89-118 SMs and
// +46 % at 148 SMs with a 4096-token prefix (the model's cost 0.7 is wrong; ~1.1 would never
// split).  Default 0.
#ifndef SPD_X_SINGLE
#define SPD_X_SINGLE 0
#endif
#ifndef SPD_X_SINGLE_COST
#define SPD_X_SINGLE_COST 0.7
#endif
constexpr bool kXSingle = SPD_X_SINGLE != 0;
int x_single_rows(int pairs_max, int units_per_row, int grid) {
    int best_ks = 0;
    double best = 1e300;
    for (int ks = 0; ks <= pairs_max; ++ks) {
        double total = 0.0, crit = 0.0;
        for (int r = 0; r < pairs_max; ++r) {
            if (r >= pairs_max - ks) {
                for (int k = 2 * r; k <= 2 * r + 1; ++k) {
                    const double c = SPD_X_SINGLE_COST * (k + 1);
                    total += c * units_per_row;
                    crit = c > crit ? c : crit;
                }
            } else {
                const double c = 2.0 * r + 2.0;
                total += c * units_per_row;
                crit = c > crit ? c : crit;
            }
        }
        const double mk = crit > total / grid ? crit : total / grid;
        if (mk < best - 1e-9) {
            best = mk;
            best_ks = ks;
        }
    }
    return best_ks;
}

bool x_pool_ok(const semipd_pool* pl) {
    const auto& c = pl->cfg;
    const int bs = c.block_size;
    return c.dtype == SEMIPD_BF16 && c.kv_shared && c.num_kv_heads == 1 && c.head_dim_k == XDL &&
           pl->have_maps && (bs == 16 || bs == 32 || bs == 64 || bs == 128) && pl->box_rows == bs;
}

}  // namespace

extern "C" size_t semipd_prefill_mla_expanded_workspace_bytes(semipd_pool_t pool, int32_t max_reqs,
                                                              int32_t max_total_keys, int32_t num_heads) {
    if (!pool || !x_pool_ok(pool) || max_reqs <= 0 || max_reqs > XMAXN || max_total_keys < 0 ||
        num_heads <= 0 || num_heads % 2 || num_heads > 128)
        return 0;
    return x_ws_bytes(max_reqs, max_total_keys, num_heads);
}

extern "C" semipd_status semipd_prefill_mla_expanded(
    semipd_pool_t pool, int32_t layer, const void* q, const void* kv_new, const void* w_uk,
    const void* w_uv, const int32_t* cu_seqlens_q, const int32_t* req_ids, const int32_t* prefix_lens,
    int32_t n, int32_t total_q, int32_t max_chunk_len, int32_t max_total_keys, int32_t num_heads,
    float softmax_scale, void* out, void* workspace, size_t ws_bytes, int32_t sm_budget,
    int32_t* status_dev, semipd_stream_t s) {
    if (!pool || layer < 0 || layer >= pool->cfg.num_layers || n < 0 || n > XMAXN || total_q < 0 ||
        max_chunk_len < 0 || max_total_keys < 0)
        return SEMIPD_ERR_INVALID;
    if (num_heads <= 0 || num_heads % 2 || num_heads > 128) return SEMIPD_ERR_INVALID;
    if (sm_budget < -1 || sm_budget > pool->num_sms) return SEMIPD_ERR_INVALID;
    if (!x_pool_ok(pool)) return SEMIPD_ERR_UNSUPPORTED;
    if (pool->pre_n_peers > 0) return SEMIPD_ERR_UNSUPPORTED;
    // RoPE (semipd_set_rope) on the decoupled columns only: k_pe = latent columns [512, 576)
    // carry the rotation, q_pe = q columns [128, 192) the same frequencies (MLA's decoupled RoPE)
    const int rope_qoff = pool->rope_on ? XDN + (pool->rope.rot_offset - XDC) : 0;
    if (pool->rope_on && pool->rope.rot_offset < XDC) return SEMIPD_ERR_UNSUPPORTED;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (status_dev && cudaMemsetAsync(status_dev, 0, sizeof(int), st) != cudaSuccess) return SEMIPD_ERR_CUDA;
    if (n == 0 || total_q == 0) return SEMIPD_OK;
    if (!q || !kv_new || !w_uk || !w_uv || !cu_seqlens_q || !req_ids || !prefix_lens || !out || !workspace)
        return SEMIPD_ERR_INVALID;
    if (reinterpret_cast<uintptr_t>(workspace) % 256 || ws_bytes < x_ws_bytes(n, max_total_keys, num_heads))
        return SEMIPD_ERR_INVALID;
    const auto& c = pool->cfg;
    const int H = num_heads;
    int budget = spd_resolve_budget(pool, sm_budget, true);
    const size_t rows = x_rows(n, max_total_keys);
    unsigned char* wb = static_cast<unsigned char*>(workspace);
    int* hdr = reinterpret_cast<int*>(wb);
    __nv_bfloat16* kexp = reinterpret_cast<__nv_bfloat16*>(wb + x_hdr_bytes(n));
    __nv_bfloat16* vexp = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<unsigned char*>(kexp) +
                                                           spd_al256(rows * H * XDN * 2));
    __nv_bfloat16* kpe = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<unsigned char*>(vexp) +
                                                          spd_al256(rows * H * XDV * 2));
    const size_t slots = x_slots(n, max_total_keys, H);
    __nv_bfloat16* lat = reinterpret_cast<__nv_bfloat16*>(reinterpret_cast<unsigned char*>(kpe) +
                                                          spd_al256(rows * XDR * 2));
    int* cnt = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(lat) + spd_al256(rows * XDC * 2));
    float* part = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(cnt) + x_cnt_bytes(slots));
    const int lg_bs = __builtin_ctz((unsigned)c.block_size);

    // 0. with RoPE set: q_pe and the chunk's k_pe rotated in place at prefix + t (R4, R28); the
    //    prep below then writes the rotated latent rows into the pool and Kpe
    if (pool->rope_on) {
        const semipd_status r = spd_launch_rope_write_ex(
            pool, layer, const_cast<void*>(q), XDN + XDR, rope_qoff, const_cast<void*>(kv_new), nullptr,
            cu_seqlens_q, req_ids, prefix_lens, n, total_q, H, 0, status_dev, st);
        if (r != SEMIPD_OK) return r;
    }
    // 1. prep: chunk latent rows -> pool, k_pe -> Kpe, row offsets -> hdr
    XPrep pp;
    pp.cu = cu_seqlens_q;
    pp.req_ids = req_ids;
    pp.prefix = prefix_lens;
    pp.bt = pool->bt;
    pp.kv_new = static_cast<const uint4*>(kv_new);
    pp.pool = static_cast<unsigned char*>(pool->k_layer(layer));
    pp.kpe = reinterpret_cast<uint4*>(kpe);
    pp.lat = reinterpret_cast<uint4*>(lat);
    pp.hdr = hdr;
    pp.status = status_dev;
    pp.n = n;
    pp.lg_bs = lg_bs;
    pp.MBR = c.max_blocks_per_req;
    pp.N_B = c.num_blocks;
    pp.rows_cap = (long long)rows;
    pp.slots_cap = (long long)slots;
    pp.cnt = cnt;
    pp.H = H;
    pp.T = total_q;
    pp.span = spd_next_span(pool);
    const int max_mt = (int)((rows + XBM - 1) / XBM);
    int gprep = budget > 0 ? budget : pool->num_sms;
    const int prep_need = (int)((rows + 63) / 64);  // 32 warps x 2 rows per CTA and step
    if (gprep > prep_need) gprep = prep_need;
    if (spd_launch_pdl(mla_exp_prep_kernel, dim3(gprep), dim3(1024), 0, st, pp) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    pool->launches += 1;
    if (cudaGetLastError() != cudaSuccess) return SEMIPD_ERR_CUDA;

    // 2. up-projection GEMM
    // (64 cols, rows, 8 column blocks) views: one box = 128-column stage of 128 latent rows
    // (A, 32 KiB) / 256 weight rows (B, 64 KiB), landing as [block][rows][128 B]
    CUtensorMap amap, ukmap, uvmap;
    {
        const uint32_t abox[3] = {64, XBM, GCB}, bbox[3] = {64, 256, GCB};
        const uint64_t adims[3] = {64, rows, XDC / 64}, astr[2] = {XDC * 2, 128};
        const uint64_t bdims[3] = {64, (uint64_t)H * XDN, XDC / 64}, bstr[2] = {XDC * 2, 128};
        if (!spd_encode_tiled_3d(&amap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, lat, adims[0], adims[1], adims[2],
                                 astr[0], astr[1], abox[0], abox[1], abox[2], CU_TENSOR_MAP_SWIZZLE_128B) ||
            !spd_encode_tiled_3d(&ukmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(w_uk), bdims[0],
                                 bdims[1], bdims[2], bstr[0], bstr[1], bbox[0], bbox[1], bbox[2],
                                 CU_TENSOR_MAP_SWIZZLE_128B) ||
            !spd_encode_tiled_3d(&uvmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(w_uv), bdims[0],
                                 bdims[1], bdims[2], bstr[0], bstr[1], bbox[0], bbox[1], bbox[2],
                                 CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    XGemm gp;
    gp.cu = cu_seqlens_q;
    gp.req_ids = req_ids;
    gp.prefix = prefix_lens;
    gp.bt = pool->bt;
    gp.hdr = hdr;
    gp.kexp = kexp;
    gp.vexp = vexp;
    gp.status = status_dev;
    gp.span = spd_next_span(pool);
    gp.n = n;
    gp.H = H;
    gp.lg_bs = lg_bs;
    gp.box_rows = pool->box_rows;
    gp.MBR = c.max_blocks_per_req;
    gp.N_B = c.num_blocks;
    gp.rows_cap = (long long)rows;
    const size_t gsm = sizeof(GSmem) + 1024;
    const size_t tsm = sizeof(TSmem) + 1024;
    const size_t asm_ = sizeof(ASmem) + 1024;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(mla_exp_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gsm) !=
                cudaSuccess ||
            cudaFuncSetAttribute(mla_exp_gemm_ta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm) !=
                cudaSuccess ||
            cudaFuncSetAttribute(mla_exp_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)asm_) !=
                cudaSuccess)
            return SEMIPD_ERR_CUDA;
        attr_set = true;
    }
    if (kXGemmTA) {
        // W views for the A-in-TMEM GEMM: one box = 128 rows (one head) x 128 columns
        CUtensorMap tuk, tuv;
        const uint32_t tbox[3] = {64, XDN, TCB};
        const uint64_t bdims[3] = {64, (uint64_t)H * XDN, XDC / 64}, bstr[2] = {XDC * 2, 128};
        if (!spd_encode_tiled_3d(&tuk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(w_uk), bdims[0],
                                 bdims[1], bdims[2], bstr[0], bstr[1], tbox[0], tbox[1], tbox[2],
                                 CU_TENSOR_MAP_SWIZZLE_128B) ||
            !spd_encode_tiled_3d(&tuv, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(w_uv), bdims[0],
                                 bdims[1], bdims[2], bstr[0], bstr[1], tbox[0], tbox[1], tbox[2],
                                 CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
        const long long items = (long long)max_mt * (2 * H / XG);
        int tgrid = budget > 0 ? budget : (int)(items < (1 << 30) ? items : (1 << 30));
        if (tgrid > items) tgrid = (int)items;
        if (spd_launch_pdl(mla_exp_gemm_ta_kernel, dim3(tgrid), dim3(GNT), tsm, st, tuk, tuv,
                           reinterpret_cast<const uint4*>(lat), gp) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
    } else {
        const long long gtiles = (long long)max_mt * H;
        int ggrid = budget > 0 ? budget : (int)(gtiles < (1 << 30) ? gtiles : (1 << 30));
        if (ggrid > gtiles) ggrid = (int)gtiles;
        if (spd_launch_pdl(mla_exp_gemm_kernel, dim3(ggrid), dim3(GNT), gsm, st, amap, ukmap, uvmap, gp) !=
            cudaSuccess)
            return SEMIPD_ERR_CUDA;
    }
    pool->launches += 1;
    if (cudaGetLastError() != cudaSuccess) return SEMIPD_ERR_CUDA;

    // 3. attention
    XAttn ap;
    ap.cu = cu_seqlens_q;
    ap.prefix = prefix_lens;
    ap.hdr = hdr;
    ap.out = static_cast<__nv_bfloat16*>(out);
    ap.status = status_dev;
    ap.span = spd_next_span(pool);
    ap.sched = &pool->st->sched[0];
    ap.n = n;
    ap.T = total_q;
    ap.H = H;
    ap.pairs_max = (max_chunk_len + 2 * XBM - 1) / (2 * XBM);
    if (ap.pairs_max < 1) return SEMIPD_OK;
    // single-tile rows: when the grid is wide enough that the longest pair rows would set the
    // kernel's critical path, their two q tiles run as separate units (R26 holds: a tile's
    // arithmetic does not depend on being paired; only the K / V loads were shared)
    const int grid0 = budget > 0 ? budget : 1 << 30;
    ap.single_rows = kXSingle ? x_single_rows(ap.pairs_max, n * H, grid0) : 0;
    const long long units = (long long)n * H * (2 * ap.single_rows + (long long)(ap.pairs_max - ap.single_rows) *
                                                                           (kXSplit ? 2 : 1));
    if (units > (1LL << 30)) return SEMIPD_ERR_UNSUPPORTED;
    ap.n_units = (int)units;
    ap.scale_log2 = softmax_scale * XLOG2E;
    ap.part = part;
    ap.cnt = cnt;
    ap.trace = spd_trace(pool);
    CUtensorMap qmap, kxmap, vxmap, pemap;
    {
        const uint64_t dims[4] = {64, (uint64_t)H, (uint64_t)total_q, 3};
        const uint64_t strides[3] = {(XDN + XDR) * 2, (uint64_t)H * (XDN + XDR) * 2, 128};
        const uint32_t box[4] = {64, 1, 2 * XBM, 3};
        if (!spd_encode_tiled_4d(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, const_cast<void*>(q), dims, strides, box,
                                 CU_TENSOR_MAP_SWIZZLE_128B))
            return SEMIPD_ERR_CUDA;
    }
    if (!spd_encode_tiled_3d(&kxmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kexp, XDN, (uint64_t)H, rows, XDN * 2,
                             (uint64_t)H * XDN * 2, 64, 1, XBM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !spd_encode_tiled_3d(&vxmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, vexp, XDV, (uint64_t)H, rows, XDV * 2,
                             (uint64_t)H * XDV * 2, 64, 1, XBM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !spd_encode_tiled_3d(&pemap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, kpe, XDR, rows, 1, XDR * 2,
                             rows * XDR * 2, 64, XBM, 1, CU_TENSOR_MAP_SWIZZLE_128B))
        return SEMIPD_ERR_CUDA;
    int grid = budget > 0 ? budget : ap.n_units;
    if (grid > ap.n_units) grid = ap.n_units;
    if (spd_launch_pdl(mla_exp_attn_kernel, dim3(grid), dim3(ANT), asm_, st, qmap, kxmap, vxmap, pemap, ap) !=
        cudaSuccess)
        return SEMIPD_ERR_CUDA;
    pool->launches += 1;
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
