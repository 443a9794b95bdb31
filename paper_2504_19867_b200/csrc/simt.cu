// simt.cu — K/V write kernel (K/V "written into the KV cache") and the
// generic CUDA-core attention kernel used for shapes without a tensor-core path
// (fp32 pools: cfg 1 needs 1e-4, which tcgen05 kind::tf32 cannot give; other head
// dims).  Both run under the same persistent SM budget as the fast kernels.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T>
__device__ __forceinline__ T from_f(float x);
template <>
__device__ __forceinline__ float from_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

struct RowMap {
    const int* cu;     // mode 0: cu_seqlens [n+1]; mode 1: nullptr (row b <-> request b)
    const int* req;    // block-table row per request
    const int* pos0;   // mode 0: prefix_lens; mode 1: ctx_lens
    int n;
};

// row -> (request index, absolute position of the row's token)
__device__ __forceinline__ void map_row(const RowMap& m, int row, int& i, int& pos) {
    if (m.cu == nullptr) {
        i = row;
        pos = __ldg(m.pos0 + row);
        return;
    }
    int lo = 0, hi = m.n - 1;  // last i with cu[i] <= row
    while (lo < hi) {
        int mid = (lo + hi + 1) >> 1;
        if (__ldg(m.cu + mid) <= row) lo = mid; else hi = mid - 1;
    }
    i = lo;
    pos = __ldg(m.pos0 + lo) + (row - __ldg(m.cu + lo));
}

__device__ __forceinline__ void set_status(int* status, int v) {
    if (status) atomicMax(status, v);
}

// one warp per (row, kv head) pair, 16-byte vector copies; bit-exact
constexpr int kKvWarps = 8;
__global__ void __launch_bounds__(kKvWarps * 32)
    kv_write_kernel(RowMap m, int rows, const uint4* __restrict__ k_new,
                    const uint4* __restrict__ v_new, unsigned char* k_pool,
                    unsigned char* v_pool, const int* __restrict__ bt, int MBR, int N_B, int Hkv,
                    int bs, int k_vec, int v_vec, int* status) {
    // PDL: the previous kernel is complete; the attention kernel that follows may launch now
    // (its own griddepcontrol.wait holds its reads of these rows until this kernel completes)
    spd::pdl_wait();
    spd::pdl_trigger();
    const int lane = threadIdx.x & 31;
    const long long total = (long long)rows * Hkv;
    for (long long u = (long long)blockIdx.x * kKvWarps + (threadIdx.x >> 5); u < total;
         u += (long long)gridDim.x * kKvWarps) {
        const int row = (int)(u / Hkv), g = (int)(u % Hkv);
        int i, pos;
        map_row(m, row, i, pos);
        const int page = pos / bs;
        const int blk = page < MBR ? __ldg(bt + (size_t)__ldg(m.req + i) * MBR + page) : -1;
        if (blk < 0 || blk >= N_B) {
            if (lane == 0) set_status(status, SEMIPD_ERR_BAD_BLOCK);
            continue;
        }
        const size_t slot = ((size_t)blk * Hkv + g) * bs + (pos % bs);
        uint4* kd = reinterpret_cast<uint4*>(k_pool) + slot * k_vec;
        const uint4* ks = k_new + ((size_t)row * Hkv + g) * k_vec;
        for (int c = lane; c < k_vec; c += 32) kd[c] = __ldg(ks + c);
        if (v_pool) {
            uint4* vd = reinterpret_cast<uint4*>(v_pool) + slot * v_vec;
            const uint4* vs = v_new + ((size_t)row * Hkv + g) * v_vec;
            for (int c = lane; c < v_vec; c += 32) vd[c] = __ldg(vs + c);
        }
    }
}

constexpr int kSimtThreads = 128;
constexpr int kMaxDvPerThread = 8;  // dv <= 1024

template <typename T>
__global__ void __launch_bounds__(kSimtThreads)
    simt_attn_kernel(RowMap m, int rows, int Hq, int Hkv, int dk, int dv, int bs, int MBR,
                     int N_B, const T* __restrict__ q, const T* __restrict__ k_pool,
                     const T* __restrict__ v_pool, int v_row_stride, const int* __restrict__ bt,
                     float scale, T* __restrict__ out, int out_head_major, int* status,
                     SpdTrace trace, int phase) {
    extern __shared__ float smem[];
    float* sq = smem;                    // [dk]
    float* sp = sq + dk;                 // [128]
    int* sblk = reinterpret_cast<int*>(sp + kSimtThreads);  // [128]
    float* red = reinterpret_cast<float*>(sblk + kSimtThreads);  // [32]
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int G = Hq / Hkv;
    if (trace.buf && tid == 0) {
        int slot = atomicAdd(trace.ctr, 1);
        if (slot < trace.cap) {
            int4 rec = make_int4(phase, (int)spd::smid(), (int)blockIdx.x, 0 /* kernel kind: simt */);
            reinterpret_cast<int4*>(trace.buf)[slot] = rec;
        }
    }
    for (long long u = blockIdx.x; u < (long long)rows * Hq; u += gridDim.x) {
        const int row = (int)(u / Hq), h = (int)(u % Hq), g = h / G;
        int i, pos;
        map_row(m, row, i, pos);
        const int* btr = bt + (size_t)__ldg(m.req + i) * MBR;
        const int n_keys = pos + 1;
        for (int c = tid; c < dk; c += kSimtThreads)
            sq[c] = to_f(q[((size_t)row * Hq + h) * dk + c]);
        float acc[kMaxDvPerThread];
#pragma unroll
        for (int r = 0; r < kMaxDvPerThread; ++r) acc[r] = 0.f;
        float mrun = -INFINITY, lrun = 0.f;
        __syncthreads();
        for (int tile = 0; tile < n_keys; tile += kSimtThreads) {
            const int j = tile + tid;
            float s = -INFINITY;
            int blk = -1;
            if (j < n_keys) {
                const int page = j / bs;
                blk = page < MBR ? __ldg(btr + page) : -1;
                if (blk < 0 || blk >= N_B) {
                    set_status(status, SEMIPD_ERR_BAD_BLOCK);
                    blk = -1;
                } else {
                    const T* kr = k_pool + (((size_t)blk * Hkv + g) * bs + (j % bs)) * dk;
                    float dot = 0.f;
                    for (int c = 0; c < dk; ++c) dot = fmaf(sq[c], to_f(kr[c]), dot);
                    s = dot * scale;
                }
            }
            // block max
            float mx = s;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            if (lane == 0) red[w] = mx;
            __syncthreads();
            mx = red[0];
            for (int k = 1; k < kSimtThreads / 32; ++k) mx = fmaxf(mx, red[k]);
            __syncthreads();
            const float mnew = fmaxf(mrun, mx);
            const float alpha = mrun == -INFINITY ? 0.f : expf(mrun - mnew);
            const float p = (s == -INFINITY) ? 0.f : expf(s - mnew);
            sp[tid] = p;
            sblk[tid] = blk;
            float ps = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
            if (lane == 0) red[w] = ps;
            __syncthreads();
            float tot = 0.f;
            for (int k = 0; k < kSimtThreads / 32; ++k) tot += red[k];
            lrun = lrun * alpha + tot;
            mrun = mnew;
            const int nk = min(kSimtThreads, n_keys - tile);
#pragma unroll
            for (int r = 0; r < kMaxDvPerThread; ++r) {
                const int c = tid + r * kSimtThreads;
                if (c < dv) {
                    float a = acc[r] * alpha;
                    for (int jj = 0; jj < nk; ++jj) {
                        const int b2 = sblk[jj];
                        if (b2 < 0) continue;
                        const int jk = tile + jj;
                        const T* vr = v_pool + (((size_t)b2 * Hkv + g) * bs + (jk % bs)) * v_row_stride;
                        a = fmaf(sp[jj], to_f(vr[c]), a);
                    }
                    acc[r] = a;
                }
            }
            __syncthreads();
        }
        const float inv = 1.f / lrun;
#pragma unroll
        for (int r = 0; r < kMaxDvPerThread; ++r) {
            const int c = tid + r * kSimtThreads;
            if (c < dv) {
                const size_t o = out_head_major ? (((size_t)h * rows + row) * dv + c)
                                                : (((size_t)row * Hq + h) * dv + c);
                out[o] = from_f<T>(acc[r] * inv);
            }
        }
        __syncthreads();
    }
}

}  // namespace

semipd_status spd_launch_kv_write(semipd_pool_t p, int layer, const void* k_new, const void* v_new,
                                  const int* cu_seqlens, const int* req_ids, const int* pos0,
                                  int n, int total_rows, int mode, int* status_dev,
                                  cudaStream_t s) {
    if (total_rows <= 0) return SEMIPD_OK;
    if (p->cfg.dtype == SEMIPD_FP8_E4M3) {  // quantised write (reading R31), prefill rows only
        if (mode != 0) return SEMIPD_ERR_UNSUPPORTED;
        return spd_launch_kv_write_fp8(p, layer, k_new, v_new, cu_seqlens, req_ids, pos0, n,
                                       total_rows, status_dev, s);
    }
    RowMap m{mode == 0 ? cu_seqlens : nullptr, req_ids, pos0, n};
    const auto& c = p->cfg;
    const int k_vec = (int)(c.head_dim_k * p->esize / 16);
    const int v_vec = (int)(c.head_dim_v * p->esize / 16);
    const long long units = (long long)total_rows * c.num_kv_heads;
    long long grid = (units + kKvWarps - 1) / kKvWarps;
    if (grid > 16LL * p->num_sms) grid = 16LL * p->num_sms;
    unsigned char* vpool = c.kv_shared ? nullptr : static_cast<unsigned char*>(p->v_layer(layer));
    const cudaError_t le = spd_launch_pdl(kv_write_kernel, dim3((unsigned)grid), dim3(kKvWarps * 32), 0, s,
                                          m, total_rows, static_cast<const uint4*>(k_new),
                                        static_cast<const uint4*>(v_new),
                                        static_cast<unsigned char*>(p->k_layer(layer)), vpool,
                                        p->bt, c.max_blocks_per_req, c.num_blocks,
                                        c.num_kv_heads, c.block_size, k_vec, v_vec, status_dev);
    p->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

semipd_status spd_launch_simt_attn(semipd_pool_t p, int layer, const void* q, const int* cu_seqlens,
                                   const int* req_ids, const int* pos0, int n, int total_rows,
                                   int mode, int Hq, float scale, void* out, int out_head_major,
                                   int budget, int* status_dev, cudaStream_t s) {
    const auto& c = p->cfg;
    if (c.head_dim_v > kSimtThreads * kMaxDvPerThread) return SEMIPD_ERR_UNSUPPORTED;
    if (total_rows <= 0) return SEMIPD_OK;
    RowMap m{mode == 0 ? cu_seqlens : nullptr, req_ids, pos0, n};
    const long long units = (long long)total_rows * Hq;
    long long grid = budget > 0 ? budget : units;
    if (grid > units) grid = units;
    if (grid > (1LL << 30)) grid = 1LL << 30;
    const size_t smem = sizeof(float) * (c.head_dim_k + kSimtThreads + 32) + sizeof(int) * kSimtThreads;
    const int v_stride = c.kv_shared ? c.head_dim_k : c.head_dim_v;
    const SpdTrace tr = spd_trace(p);
    const int phase = mode == 0 ? 1 : 2;
    if (c.dtype == SEMIPD_FP32) {
        simt_attn_kernel<float><<<(unsigned)grid, kSimtThreads, smem, s>>>(
            m, total_rows, Hq, c.num_kv_heads, c.head_dim_k, c.head_dim_v, c.block_size,
            c.max_blocks_per_req, c.num_blocks, static_cast<const float*>(q),
            static_cast<const float*>(p->k_layer(layer)), static_cast<const float*>(p->v_layer(layer)),
            v_stride, p->bt, scale, static_cast<float*>(out), out_head_major, status_dev, tr, phase);
    } else {
        simt_attn_kernel<__nv_bfloat16><<<(unsigned)grid, kSimtThreads, smem, s>>>(
            m, total_rows, Hq, c.num_kv_heads, c.head_dim_k, c.head_dim_v, c.block_size,
            c.max_blocks_per_req, c.num_blocks, static_cast<const __nv_bfloat16*>(q),
            static_cast<const __nv_bfloat16*>(p->k_layer(layer)),
            static_cast<const __nv_bfloat16*>(p->v_layer(layer)), v_stride, p->bt, scale,
            static_cast<__nv_bfloat16*>(out), out_head_major, status_dev, tr, phase);
    }
    p->launches += 1;
    return cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}
