// common.cuh — sm_100a device helpers (inline PTX): mbarrier, TMA, tcgen05/TMEM,
// ldmatrix / mma.sync, proxy fences.  Part of the CUDA path only (no oracle code).
#pragma once
#include <cuda.h>
#include <cuda_fp8.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define SPD_DEV __device__ __forceinline__

namespace spd {

SPD_DEV uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
SPD_DEV uint32_t lane_id() { return threadIdx.x & 31u; }
SPD_DEV uint32_t warp_id() { return __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0); }
SPD_DEV uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

SPD_DEV unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// ------------------------------------------------------------------ launch spans
// Device-side launch timing (semipd_set_spans): every CTA's thread 0 calls span_begin at
// entry and span_end after the CTA's final __syncthreads.  Record (8 x u64, zero-initialised):
//   [0] ~min(start)  [1] max(end)  [2] sum of durations (ns)  [3] launches
//   [4] CTAs done in the running launch  [5] last start  [6] last end
// The CTA that finishes last folds the launch into [2] / [3], keeps [5] / [6] and resets
// [0], [1], [4], so a launch captured in a CUDA graph accumulates over its replays.
SPD_DEV void span_begin(unsigned long long* rec) {
    if (rec) atomicMax(rec + 0, ~globaltimer_ns());
}
SPD_DEV void span_end(unsigned long long* rec) {
    if (!rec) return;
    atomicMax(rec + 1, globaltimer_ns());
    __threadfence();
    if (atomicAdd(rec + 4, 1ull) == gridDim.x - 1) {
        __threadfence();
        volatile unsigned long long* v = rec;
        const unsigned long long t0 = ~v[0], t1 = v[1];
        rec[2] += t1 - t0;
        rec[3] += 1;
        rec[5] = t0;
        rec[6] = t1;
        rec[0] = 0;
        rec[1] = 0;
        rec[4] = 0;
        __threadfence();
    }
}

// ------------------------------------------------------------------ cp.async (LDGSTS)
// 16-byte global -> shared copy through L2 (.cg) with an L2 policy; src_bytes = 0 zero-fills
SPD_DEV void cp_async16_hint(uint32_t dst, const void* src, uint32_t src_bytes, uint64_t pol) {
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst),
                 "l"(src), "r"(src_bytes), "l"(pol)
                 : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed (no pending-count
// increment: the barrier's expected count includes this arrival)
SPD_DEV void cp_async_mbar_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// ------------------------------------------------------------------ mbarrier
SPD_DEV void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
SPD_DEV void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SPD_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
SPD_DEV void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SPD_DEV bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
// non-blocking probe of a phase (for a thread that polls several barriers)
SPD_DEV bool mbar_test_wait(const uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
SPD_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}

// ------------------------------------------------------------------ TMA
SPD_DEV void tma_prefetch_desc(const CUtensorMap* m) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
// 3-D tiled load, completes `bytes` on bar (expect_tx armed separately).
SPD_DEV void tma_load_3d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
SPD_DEV void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z,
                         int w) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
        : "memory");
}
// L2 eviction-priority policies for TMA loads (createpolicy): the decode KV stream is read
// once per step and should not push out the prefill's reused chunk K/V tiles in the co-run
SPD_DEV uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SPD_DEV uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SPD_DEV uint64_t l2_policy_evict_normal() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// 0 = evict_normal, 1 = evict_first, 2 = evict_last
SPD_DEV uint64_t l2_policy(int kind) {
    return kind == 1 ? l2_policy_evict_first() : kind == 2 ? l2_policy_evict_last() : l2_policy_evict_normal();
}
SPD_DEV void tma_load_3d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z,
                              uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "l"(policy)
        : "memory");
}
SPD_DEV void tma_load_4d_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z,
                              int w, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w),
        "l"(policy)
        : "memory");
}
// L2 prefetch of one 4-D box (no shared memory, no barrier: fire and forget)
SPD_DEV void tma_prefetch_l2_4d(const CUtensorMap* m, int x, int y, int z, int w) {
    asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(x), "r"(y), "r"(z), "r"(w)
                 : "memory");
}
// smem -> global tensor store (bulk async group), and the group completion waits
SPD_DEV void tma_store_3d(const CUtensorMap* m, const void* src, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(m),
        "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
SPD_DEV void bulk_commit_group() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SPD_DEV void bulk_wait_group_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SPD_DEV void bulk_wait_group0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy global writes -> later async-proxy (TMA) reads
SPD_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SPD_DEV void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------------ tcgen05 / TMEM
SPD_DEV void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
SPD_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
                 : "memory");
}
SPD_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SPD_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// D[tmem] (+)= A[smem desc] * B[smem desc]
SPD_DEV void umma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                     uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]
SPD_DEV void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                     uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
// Warp-collective forms: the whole (converged) warp executes the call with warp-uniform
// operands and elect.sync picks one issuing lane inside the asm.  The descriptors then stay
// in uniform registers — about 2x the issue rate of a lane-0-only branch for small MMAs
// (scripts/probe_umma_rate.cu: 25.6 vs 50 cycles per M64 N16 K16 SS MMA).
SPD_DEV void umma_ss_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                          uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
SPD_DEV void umma_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                          uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accum)
        : "memory");
}
// The two 32-bit words of umma_desc_sw128(addr, lbo, 1024): low = start >> 4 | LBO >> 4 << 16,
// high = SBO (1 KiB) >> 4 | version 1 | 128-byte swizzle.
constexpr uint32_t DESC_HI_SBO1K = (1024u >> 4) | (1u << 14) | (2u << 29);
SPD_DEV uint32_t desc_lo(uint32_t smem_addr, uint32_t lbo_bytes) {
    return ((smem_addr >> 4) & 0x3FFFu) | (((lbo_bytes >> 4) & 0x3FFFu) << 16);
}
// Same, with each smem descriptor passed as two 32-bit words (low: start address and LBO
// fields, high: SBO / version / layout): callers add 16-byte offsets to the low word with 32-bit
// arithmetic and keep the constant high word in one register (no 64-bit adds per MMA).
SPD_DEV void umma_ss_warp2(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t b_lo, uint32_t b_hi,
                           uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\tsetp.ne.b32 p, %6, 0;\n\t"
        "mov.b64 da, {%1, %2};\n\tmov.b64 db, {%3, %4};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %5, p;\n\t}" ::"r"(d_tmem),
        "r"(a_lo), "r"(a_hi), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accum)
        : "memory");
}
SPD_DEV void umma_ts_warp2(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi, uint32_t idesc,
                           uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b64 db;\n\tsetp.ne.b32 p, %5, 0;\n\t"
        "mov.b64 db, {%2, %3};\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], db, %4, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accum)
        : "memory");
}
SPD_DEV void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            smem_u32(bar))
        : "memory");
}
// arrive(one) on bar when all previously issued tcgen05.mma of this thread complete
SPD_DEV void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns
SPD_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
SPD_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15])
        : "memory");
}
// warp-wide float max (sm_100a CREDUX); result uniform across the warp
SPD_DEV float redux_max_f32(float v) {
    float r;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(v));
    return r;
}
SPD_DEV void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
SPD_DEV void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns: thread i gets lane (base_lane + i), cols c..c+31
SPD_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}
SPD_DEV void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}

// UMMA shared-memory descriptor (sm_100 "version 1"), 128-byte swizzle.
//   start address >> 4 in [0,14); LBO >> 4 in [16,30); SBO >> 4 in [32,46);
//   version = 1 in [46,48); base offset 0; layout type SWIZZLE_128B = 2 in [61,64).
SPD_DEV uint64_t umma_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;
    return d;
}
// Instruction descriptor, kind::f16: bf16 x bf16 -> f32, M x N, K-major A,
// B K-major (b_mn_major = 0) or MN-major (1).
__host__ __device__ constexpr uint32_t umma_idesc_bf16_f32(uint32_t M, uint32_t N,
                                                           uint32_t b_mn_major) {
    return (1u << 4)                  // D format f32
           | (1u << 7)                // A bf16
           | (1u << 10)               // B bf16
           | (0u << 15)               // A K-major
           | (b_mn_major << 16)       // B major
           | ((N >> 3) << 17)         // N / 8
           | ((M >> 4) << 24);        // M / 16
}
// same, with the A operand's major-ness selectable (a_mn_major = 1: M contiguous in smem)
__host__ __device__ constexpr uint32_t umma_idesc_bf16_f32_ab(uint32_t M, uint32_t N,
                                                              uint32_t a_mn_major,
                                                              uint32_t b_mn_major) {
    return umma_idesc_bf16_f32(M, N, b_mn_major) | (a_mn_major << 15);
}

// ------------------------------------------------------------------ legacy warp MMA
SPD_DEV void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
SPD_DEV void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// transpose of an 8x8 b16 matrix held in mma fragment layout (row t/4, cols 2(t%4)..+1)
SPD_DEV uint32_t movmatrix_t(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}
SPD_DEV void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                            uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
SPD_DEV uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
SPD_DEV float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// ------------------------------------------------------------------ packed fp32x2 (sm_100)
SPD_DEV uint64_t f2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
SPD_DEV void f2_split(uint64_t v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
SPD_DEV uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
SPD_DEV uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
SPD_DEV uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("mul.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
SPD_DEV float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// 2^x for a pair on the FMA pipe (no MUFU): x = n + f with n = rint(x), f in [-1/2, 1/2]
// (magic-number rounding), 2^f by a degree-4 polynomial (Taylor degree 5: rel. error ~3e-6, far below the
// bf16 rounding of P), 2^n by adding n to the exponent bits.  x is clamped at -125, so
// masked (-inf) inputs give ~2^-125 (3e-38) instead of 0.
SPD_DEV uint64_t exp2_poly2(uint64_t x2) {
    const float kMagic = 12582912.0f;  // 1.5 * 2^23
    float x0, x1;
    f2_split(x2, x0, x1);
    x0 = fmaxf(x0, -125.0f);
    x1 = fmaxf(x1, -125.0f);
    const uint64_t t = fadd2(f2(x0, x1), f2(kMagic, kMagic));
    const uint64_t r = fadd2(t, f2(-kMagic, -kMagic));
    float r0, r1, t0, t1;
    f2_split(r, r0, r1);
    f2_split(t, t0, t1);
    const uint64_t f = fadd2(f2(x0, x1), f2(-r0, -r1));
    uint64_t p = f2(1.3333558146e-3f, 1.3333558146e-3f);
    p = ffma2(p, f, f2(9.6181291076e-3f, 9.6181291076e-3f));
    p = ffma2(p, f, f2(5.5504108665e-2f, 5.5504108665e-2f));
    p = ffma2(p, f, f2(2.4022650696e-1f, 2.4022650696e-1f));
    p = ffma2(p, f, f2(6.9314718056e-1f, 6.9314718056e-1f));
    p = ffma2(p, f, f2(1.0f, 1.0f));
    float p0, p1;
    f2_split(p, p0, p1);
    const int n0 = __float_as_int(t0) - 0x4B400000, n1 = __float_as_int(t1) - 0x4B400000;
    return f2(__int_as_float(__float_as_int(p0) + (n0 << 23)),
              __int_as_float(__float_as_int(p1) + (n1 << 23)));
}

template <uint32_t N>
SPD_DEV void setmaxnreg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <uint32_t N>
SPD_DEV void setmaxnreg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

// 2^x for a pair on the FMA pipe: x = j + f with j = rint(x) (magic-number rounding, exact for
// |x| < 2^22), f in [-1/2, 1/2]; 2^f by a degree-3 relative-minimax polynomial (max rel. error
// 7.5e-5, below the bf16 rounding of P, 2^-9); 2^j added into the exponent bits.  x is clamped
// at -125 so the exponent add cannot underflow: masked (-inf) scores give ~2^-125 instead of 0.
SPD_DEV uint64_t exp2_poly3(uint64_t x2) {
    constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
    float x0, x1;
    f2_split(x2, x0, x1);
    const uint64_t xc = f2(fmaxf(x0, -125.f), fmaxf(x1, -125.f));
    const uint64_t t = fadd2(xc, f2(kMagic, kMagic));                      // M + j
    const uint64_t nj = ffma2(t, f2(-1.f, -1.f), f2(kMagic, kMagic));      // -j (exact)
    const uint64_t fr = fadd2(xc, nj);                                     // f
    uint64_t q = ffma2(f2(0.05517049f, 0.05517049f), fr, f2(0.24260938f, 0.24260938f));
    q = ffma2(q, fr, f2(0.69326103f, 0.69326103f));
    q = ffma2(q, fr, f2(0.99992818f, 0.99992818f));
    float q0, q1, t0, t1;
    f2_split(q, q0, q1);
    f2_split(t, t0, t1);
    // bits(M + j) = 0x4B400000 + j and 0x4B400000 << 23 == 0 (mod 2^32): (bits << 23) = j << 23
    return f2(__uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23)),
              __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23)));
}

// a += float(lo half of pp), b += float(hi half): add.f32.bf16 is one FHADD.BF16 per element
// with a half-register operand (no unpacking)
SPD_DEV void add_bf16x2_f32(float& a, float& b, uint32_t pp) {
    asm("{\n\t.reg .b16 lo, hi;\n\tmov.b32 {lo, hi}, %2;\n\t"
        "add.rn.f32.bf16 %0, lo, %0;\n\tadd.rn.f32.bf16 %1, hi, %1;\n\t}"
        : "+f"(a), "+f"(b)
        : "r"(pp));
}

// Programmatic dependent launch (the attention kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, internal.h spd_launch_pdl): a kernel may
// start while the previous kernel on its stream drains; pdl_wait() blocks until that kernel has
// completed and its memory is visible, so it comes before any dependent global access.
// pdl_trigger() lets the next kernel's CTAs be scheduled once every CTA of this grid has issued
// it (or exited).
SPD_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SPD_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// named barrier among `nthreads` threads (id 1..15; 0 is __syncthreads)
SPD_DEV void named_bar_sync(uint32_t id, uint32_t nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// E4M3 pages (reading R31) write rule: code = E4M3_rne_satfinite(fl32(x / s)) of two floats;
// lo -> low byte (fp8.cu's quantised writes and the fused RoPE write in rope.cu)
SPD_DEV uint32_t quant2(float lo, float hi, float s) {
    const float2 v = make_float2(__fdiv_rn(lo, s), __fdiv_rn(hi, s));
    return (uint32_t)__nv_cvt_float2_to_fp8x2(v, __NV_SATFINITE, __NV_E4M3);
}

// 8 bf16 (one uint4) -> 8 codes (one uint2), element order kept
SPD_DEV uint2 quant8(uint4 x, float s) {
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t b[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        b[i] = quant2(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u), s);
    return make_uint2(b[0] | (b[1] << 16), b[2] | (b[3] << 16));
}

}  // namespace spd
