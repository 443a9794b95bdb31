// alloc.cu — the unified memory manager's atomic block allocator (§4.4,
// fig:atomic): "querying the memory utilization ..., getting the blocks ..., and
// updating the memory utilization" run as ONE critical section under a device
// lock ("the memory utilization is locked until the update step finishes").
// A single CTA holds the lock; its 256 threads do the pops/pushes in parallel.
// Contract: SPEC S:234-251; sequential semantics = oracle/semipd_oracle.c (the
// two share no code); linearisation order is recorded in the op log.
#include <cuda/atomic>
#include <cuda_runtime.h>

#include "common.cuh"
#include "internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxN = 1024;  // requests per call

enum : int { kOpAlloc = 1, kOpFree = 2 };

struct AllocArgs {
    SpdDevState* st;
    int* free_stack;
    int* nblk;
    int* bt;
    int* oplog;
    long long oplog_cap;
    int N_B, R, MBR;
};

__device__ void lock_acquire(SpdDevState* st) {
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> lk(st->lock);
    unsigned ns = 32;
    while (lk.exchange(1u, cuda::memory_order_acquire) != 0u) {
        __nanosleep(ns);
        if (ns < 2048) ns <<= 1;
    }
}
__device__ void lock_release(SpdDevState* st) {
    __threadfence();
    cuda::atomic_ref<unsigned int, cuda::thread_scope_device> lk(st->lock);
    lk.store(0u, cuda::memory_order_release);
}

// block-wide exclusive scan of one value per thread; returns the block total in *total
__device__ int block_exclusive_scan(int v, int* scratch, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = lane < kThreads / 32 ? scratch[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < kThreads / 32) scratch[lane] = s;  // inclusive warp totals
    }
    __syncthreads();
    const int warp_off = w > 0 ? scratch[w - 1] : 0;
    *total = scratch[kThreads / 32 - 1];
    __syncthreads();
    return warp_off + x - v;
}

// item owning flattened index idx: last i with prefix[i] <= idx (prefix is non-decreasing)
__device__ __forceinline__ int owner(const int* prefix, int n, int idx) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (prefix[mid] <= idx) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ void log_op(const AllocArgs& a, int kind, int n, int status, const int* ids,
                       const int* counts, unsigned long long seq) {
    // all threads participate; thread 0 owns the header
    const long long words = 4 + (long long)n * (kind == kOpAlloc ? 2 : 1);
    __shared__ long long s_off;
    if (threadIdx.x == 0) {
        long long off = a.st->oplog_len;
        if (a.oplog == nullptr || off + words > a.oplog_cap) {
            a.st->oplog_dropped += 1;
            s_off = -1;
        } else {
            a.st->oplog_len = off + words;
            s_off = off;
            a.oplog[off + 0] = (int)seq;
            a.oplog[off + 1] = kind;
            a.oplog[off + 2] = n;
            a.oplog[off + 3] = status;
        }
    }
    __syncthreads();
    const long long off = s_off;
    if (off >= 0) {
        for (int i = threadIdx.x; i < n; i += kThreads) {
            a.oplog[off + 4 + i] = __ldg(ids + i);
            if (kind == kOpAlloc) a.oplog[off + 4 + n + i] = __ldg(counts + i);
        }
    }
}

__global__ void __launch_bounds__(kThreads) alloc_kernel(AllocArgs a, const int* __restrict__ ids,
                                                         const int* __restrict__ counts, int n,
                                                         int* status_dev) {
    __shared__ int s_base[kMaxN];   // first table slot of item i in its row
    __shared__ int s_prefix[kMaxN]; // blocks popped before item i (argument order)
    __shared__ int scratch[32];
    __shared__ int s_flag, s_top;
    __shared__ unsigned long long s_seq;
    const int tid = threadIdx.x;
    // PDL: everything before this call on the stream is complete; the next kernel may launch
    // now (its own griddepcontrol.wait holds it until this one has completed)
    spd::pdl_wait();
    spd::pdl_trigger();
    if (tid == 0) {
        lock_acquire(a.st);
        s_top = __ldcg(&a.st->top);
        s_seq = __ldcg(&a.st->op_seq);
        s_flag = SEMIPD_OK;
    }
    __syncthreads();
    const int top = s_top;
    // ---- query: validate + total
    int total = 0;
    for (int c0 = 0; c0 < n; c0 += kThreads) {
        const int i = c0 + tid;
        int cnt = 0;
        if (i < n) {
            const int id = __ldg(ids + i);
            cnt = __ldg(counts + i);
            if (id < 0 || id >= a.R || cnt < 1) atomicMax(&s_flag, SEMIPD_ERR_INVALID);
        }
        int chunk_total;
        const int ex = block_exclusive_scan(cnt, scratch, &chunk_total);
        if (i < n) s_prefix[i] = total + ex;
        total += chunk_total;
    }
    __syncthreads();
    int status = s_flag;
    if (status == SEMIPD_OK && total > top) status = SEMIPD_ERR_OOM;
    if (status == SEMIPD_OK) {
        for (int i = tid; i < n; i += kThreads) {
            const int id = __ldg(ids + i);
            int before = 0, all = 0;
            for (int k = 0; k < n; ++k) {
                if (__ldg(ids + k) == id) {
                    const int c = __ldg(counts + k);
                    all += c;
                    if (k < i) before += c;
                }
            }
            const int cur = __ldcg(a.nblk + id);
            s_base[i] = cur + before;
            if ((long long)cur + all > a.MBR) atomicMax(&s_flag, SEMIPD_ERR_TABLE_FULL);
        }
        __syncthreads();
        if (s_flag != SEMIPD_OK) status = s_flag;
    }
    // ---- get + update
    if (status == SEMIPD_OK) {
        // the idx-th popped block (argument order) goes to item i = owner(idx)
        for (int idx = tid; idx < total; idx += kThreads) {
            const int i = owner(s_prefix, n, idx);
            const int id = __ldg(ids + i);
            a.bt[(size_t)id * a.MBR + s_base[i] + (idx - s_prefix[i])] =
                __ldcg(a.free_stack + (top - 1 - idx));
        }
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) {
            const int id = __ldg(ids + i);
            bool first = true;
            int all = 0;
            for (int k = 0; k < n; ++k)
                if (__ldg(ids + k) == id) {
                    if (k < i) first = false;
                    all += __ldg(counts + k);
                }
            if (first) a.nblk[id] = __ldcg(a.nblk + id) + all;
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (status == SEMIPD_OK) {
            a.st->top = top - total;
            if (top - total < __ldcg(&a.st->min_free)) a.st->min_free = top - total;
        }
        a.st->op_seq = s_seq + 1ull;
    }
    log_op(a, kOpAlloc, n, status, ids, counts, s_seq);
    __syncthreads();
    if (tid == 0) {
        lock_release(a.st);
        if (status_dev) *status_dev = status;
    }
}

__global__ void __launch_bounds__(kThreads) free_kernel(AllocArgs a, const int* __restrict__ ids,
                                                        int n, int* status_dev) {
    __shared__ int s_prefix[kMaxN];
    __shared__ int scratch[32];
    __shared__ int s_flag, s_top;
    __shared__ unsigned long long s_seq;
    const int tid = threadIdx.x;
    // PDL: everything before this call on the stream is complete; the next kernel may launch
    // now (its own griddepcontrol.wait holds it until this one has completed)
    spd::pdl_wait();
    spd::pdl_trigger();
    if (tid == 0) {
        lock_acquire(a.st);
        s_top = __ldcg(&a.st->top);
        s_seq = __ldcg(&a.st->op_seq);
        s_flag = SEMIPD_OK;
    }
    __syncthreads();
    const int top = s_top;
    for (int i = tid; i < n; i += kThreads) {
        const int id = __ldg(ids + i);
        if (id < 0 || id >= a.R) atomicMax(&s_flag, SEMIPD_ERR_INVALID);
    }
    __syncthreads();
    int status = s_flag;
    if (status == SEMIPD_OK) {
        for (int i = tid; i < n; i += kThreads) {
            const int id = __ldg(ids + i);
            bool bad = __ldcg(a.nblk + id) == 0;
            for (int k = 0; k < i && !bad; ++k) bad = __ldg(ids + k) == id;
            if (bad) atomicMax(&s_flag, SEMIPD_ERR_UNKNOWN_REQ);
        }
        __syncthreads();
        status = s_flag;
    }
    int total = 0;
    if (status == SEMIPD_OK) {
        for (int c0 = 0; c0 < n; c0 += kThreads) {
            const int i = c0 + tid;
            const int cnt = i < n ? __ldcg(a.nblk + __ldg(ids + i)) : 0;
            int chunk_total;
            const int ex = block_exclusive_scan(cnt, scratch, &chunk_total);
            if (i < n) s_prefix[i] = total + ex;
            total += chunk_total;
        }
        __syncthreads();
        // push blocks in (argument, table) order: slot top + idx
        for (int idx = tid; idx < total; idx += kThreads) {
            const int i = owner(s_prefix, n, idx);
            int* row = a.bt + (size_t)__ldg(ids + i) * a.MBR;
            const int j = idx - s_prefix[i];
            a.free_stack[top + idx] = __ldcg(row + j);
            row[j] = -1;
        }
        __syncthreads();
        for (int i = tid; i < n; i += kThreads) a.nblk[__ldg(ids + i)] = 0;
    }
    __syncthreads();
    if (tid == 0) {
        if (status == SEMIPD_OK) a.st->top = top + total;
        a.st->op_seq = s_seq + 1ull;
    }
    log_op(a, kOpFree, n, status, ids, nullptr, s_seq);
    __syncthreads();
    if (tid == 0) {
        lock_release(a.st);
        if (status_dev) *status_dev = status;
    }
}

AllocArgs args_of(semipd_pool_t p) {
    AllocArgs a;
    a.st = p->st;
    a.free_stack = p->free_stack;
    a.nblk = p->nblk;
    a.bt = p->bt;
    a.oplog = p->cfg.oplog_words > 0 ? p->oplog : nullptr;
    a.oplog_cap = p->cfg.oplog_words;
    a.N_B = p->cfg.num_blocks;
    a.R = p->cfg.max_reqs;
    a.MBR = p->cfg.max_blocks_per_req;
    return a;
}

}  // namespace

extern "C" {

semipd_status semipd_alloc_blocks(semipd_pool_t pool, const int32_t* req_ids,
                                  const int32_t* n_blocks, int32_t n, int32_t* status_dev,
                                  semipd_stream_t s) {
    if (!pool || n < 0 || n > kMaxN) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (n == 0) {
        if (status_dev && cudaMemsetAsync(status_dev, 0, sizeof(int), st) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        return SEMIPD_OK;
    }
    if (!req_ids || !n_blocks) return SEMIPD_ERR_INVALID;
    const cudaError_t le = spd_launch_pdl(alloc_kernel, dim3(1), dim3(kThreads), 0, st, args_of(pool),
                                          req_ids, n_blocks, n, status_dev);
    pool->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

semipd_status semipd_free_blocks(semipd_pool_t pool, const int32_t* req_ids, int32_t n,
                                 int32_t* status_dev, semipd_stream_t s) {
    if (!pool || n < 0 || n > kMaxN) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (n == 0) {
        if (status_dev && cudaMemsetAsync(status_dev, 0, sizeof(int), st) != cudaSuccess)
            return SEMIPD_ERR_CUDA;
        return SEMIPD_OK;
    }
    if (!req_ids) return SEMIPD_ERR_INVALID;
    const cudaError_t le = spd_launch_pdl(free_kernel, dim3(1), dim3(kThreads), 0, st, args_of(pool),
                                          req_ids, n, status_dev);
    pool->launches += 1;
    return le == cudaSuccess && cudaGetLastError() == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

}  // extern "C"
