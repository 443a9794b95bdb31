// peer.cu — head-output all-gather over peer memory with no SMs (§8(e)).
//
// TP by KV head (§4.5: the prefill workers form one group, the decode workers another)
// leaves one exchange step: every rank's head-major shard [Hq/TP, T, dv] must reach every
// other rank's gathered buffer [Hq, T, dv].  NCCL's all-gather does that with CTAs taken from
// the phase's SM partition.  Here the copy engines do it instead:
//   1. entry handshake: tell every peer "my previous reads of the gathered buffer are done"
//      and wait for the same from all of them, so a push cannot overwrite data a peer is
//      still reading;
//   2. push the local shard into each peer's gathered buffer (cudaMemcpyAsync on IPC-mapped
//      pointers: copy-engine DMA over NVLink, no kernel);
//   3. set slot `rank` of each peer's flag array (a stream write-value op, which fences the
//      stream's prior writes first);
//   4. wait until every peer's slot of the own flag array is set, and reset it (wait-value
//      and write-value ops; 3 and 4 go out as ONE cuStreamBatchMemOp).
// Steps 3-4 are stream memory operations executed by the GPU front end: the gather occupies
// no SM of either partition.  Everything is stream-ordered on the caller's stream.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "internal.h"

namespace {

typedef CUresult (*PFN_batch)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

PFN_batch g_batch = nullptr;

bool load_stream_memops() {
    // the _v2 stream memory operations (CUDA >= 11.7) are enabled by default; the v1 ones
    // need a driver module option, so ask for the CUDA 12.0 ABI explicitly (thread-safe once)
    static const bool ok = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", &p, 12000, cudaEnableDefault,
                                             &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            g_batch = reinterpret_cast<PFN_batch>(p);
        return g_batch != nullptr;
    }();
    return ok;
}

semipd_status fail(const char* what, int code) {
    std::fprintf(stderr, "semipd_peer_gather: %s failed (%d)\n", what, code);
    return SEMIPD_ERR_CUDA;
}

// One batched stream-memory-operation call per handshake (measured on this B200: one write /
// wait call costs ~2 us of submission, a batch ~0.6 us per op): set this rank's slot in every
// peer's flag array (writes fence the stream's prior writes, so copies / kernel stores land
// first), then wait for and reset each own slot.  base_slot: 0 = "landed", world = "ready".
semipd_status handshake(CUstream cs, uint32_t* const* peer_flags, uint32_t* my_flags, int world,
                        int rank, int base_slot) {
    auto dp = [](const uint32_t* p) { return reinterpret_cast<CUdeviceptr>(p); };
    CUstreamBatchMemOpParams ops[3 * SEMIPD_MAX_PEERS];
    std::memset(ops, 0, sizeof(ops));
    int n = 0;
    for (int k = 0; k < world; ++k) {
        if (k == rank) continue;
        ops[n].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
        ops[n].writeValue.address = dp(peer_flags[k] + base_slot + rank);
        ops[n].writeValue.value = 1u;
        ++n;
    }
    for (int k = 0; k < world; ++k) {
        if (k == rank) continue;
        ops[n].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[n].waitValue.address = dp(my_flags + base_slot + k);
        ops[n].waitValue.value = 1u;
        ops[n].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
        ++n;
        ops[n].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
        ops[n].writeValue.address = dp(my_flags + base_slot + k);
        ops[n].writeValue.value = 0u;
        ++n;
    }
    if (n == 0) return SEMIPD_OK;
    const CUresult r = g_batch(cs, (unsigned)n, ops, 0);
    return r == CUDA_SUCCESS ? SEMIPD_OK : fail("batched flag operations", (int)r);
}

}  // namespace

extern "C" {

semipd_status semipd_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
    if (!dev_ptr || !handle_out || bytes == 0) return SEMIPD_ERR_INVALID;
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return SEMIPD_ERR_CUDA;
    cudaIpcMemHandle_t h;
    // cudaMemset is asynchronous to the host: finish the zeroing before the handle leaves
    // this call, or a late memset could erase a peer's first ready / landed flag
    if (cudaMemset(p, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess ||
        cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return SEMIPD_ERR_CUDA;
    }
    static_assert(sizeof(h) == SEMIPD_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &h, sizeof(h));
    *dev_ptr = p;
    return SEMIPD_OK;
}

semipd_status semipd_ipc_free(void* dev_ptr) {
    if (!dev_ptr) return SEMIPD_ERR_INVALID;
    return cudaFree(dev_ptr) == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

semipd_status semipd_ipc_open(const void* handle, void** dev_ptr) {
    if (!handle || !dev_ptr) return SEMIPD_ERR_INVALID;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return SEMIPD_ERR_CUDA;
    }
    *dev_ptr = p;
    return SEMIPD_OK;
}

semipd_status semipd_ipc_close(void* dev_ptr) {
    if (!dev_ptr) return SEMIPD_ERR_INVALID;
    return cudaIpcCloseMemHandle(dev_ptr) == cudaSuccess ? SEMIPD_OK : SEMIPD_ERR_CUDA;
}

semipd_status semipd_peer_gather(const void* src, size_t bytes, void* const* dsts,
                                 uint32_t* const* peer_flags, uint32_t* my_flags, int32_t world,
                                 int32_t rank, semipd_stream_t s) {
    if (world < 1 || world > SEMIPD_MAX_PEERS || rank < 0 || rank >= world || !dsts ||
        !peer_flags || !my_flags || (bytes > 0 && !src))
        return SEMIPD_ERR_INVALID;
    for (int k = 0; k < world; ++k)
        if (!dsts[k] || !peer_flags[k]) return SEMIPD_ERR_INVALID;
    if (!load_stream_memops()) return SEMIPD_ERR_UNSUPPORTED;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    CUstream cs = reinterpret_cast<CUstream>(st);
    // Flags are binary semaphores (values 0 / 1): a waiter resets its own slot after the wait,
    // so the operations carry no per-call value and a captured CUDA graph replays correctly.
    // Slots [world, 2 world) = "ready", [0, world) = "landed".  The ready handshake orders a
    // peer's next "landed" write after this rank's reset of the previous one (and vice versa).
    if (semipd_status e = handshake(cs, peer_flags, my_flags, world, rank, world); e != SEMIPD_OK)
        return e;
    if (bytes > 0) {
        // push to the peers in ring order starting after this rank, so the ranks' first copies
        // target different destinations
        for (int i = 0; i < world; ++i) {
            const int k = (rank + 1 + i) % world;
            if (dsts[k] == src) continue;
            const cudaError_t e = cudaMemcpyAsync(dsts[k], src, bytes, cudaMemcpyDefault, st);
            if (e != cudaSuccess) {
                cudaGetLastError();
                return fail("peer copy", (int)e);
            }
        }
    }
    if (semipd_status e = handshake(cs, peer_flags, my_flags, world, rank, 0); e != SEMIPD_OK)
        return e;
    return SEMIPD_OK;
}

semipd_status semipd_peer_handshake(uint32_t* const* peer_flags, uint32_t* my_flags,
                                    int32_t world, int32_t rank, int32_t which, semipd_stream_t s) {
    if (world < 1 || world > SEMIPD_MAX_PEERS || rank < 0 || rank >= world || !peer_flags ||
        !my_flags || (which != 0 && which != 1))
        return SEMIPD_ERR_INVALID;
    for (int k = 0; k < world; ++k)
        if (!peer_flags[k]) return SEMIPD_ERR_INVALID;
    if (!load_stream_memops()) return SEMIPD_ERR_UNSUPPORTED;
    return handshake(reinterpret_cast<CUstream>(s), peer_flags, my_flags, world, rank,
                     which == 0 ? world : 0);
}

}  // extern "C"
