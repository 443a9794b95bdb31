/*
 * semipd.h — C ABI of libsemipd.so, the B200 (sm_100a) hot path of semi-PD
 * (arXiv 2504.19867): prefill and decode attention co-running on disjoint SM
 * partitions of one GPU over ONE unified paged KV-cache pool.
 *
 * Paper passages (PAPER.md line, section):
 *   P:184 §4.2  prefill writes the request's K/V "into the KV cache"; decode
 *               updates it "at each decode iteration"; a request moves from the
 *               prefill worker's queue to the decode worker's after prefill.
 *   P:195 §4.3  "(x, y) ... the percentage of the total SMs dispatched to the
 *               prefill and decode processes".
 *   P:209-216   resident holder of weights + KV, delayed and asynchronous switching;
 *               x + y > 100 is allowed ("compete for the resources").
 *   P:229 §4.4  paged KV "accessed through the block table index"; allocation
 *               (query -> get -> update) is atomic: "the memory utilization is
 *               locked until the update step finishes".
 *   P:355 §6    GQA attention kernels for both phases.
 * SPEC.md (allocator contract): S:234-262.
 *
 * Conventions (all functions):
 *   - Pointers are DEVICE pointers unless documented "host".  All device work is
 *     stream-ordered on the given stream (a cudaStream_t passed as void*; NULL =
 *     legacy default stream).  No call allocates device memory: the caller owns
 *     the pool backing memory, all I/O tensors and workspaces (PyTorch allocates
 *     them in the Python binding) and must keep them alive while in use.
 *   - Host argument errors return SEMIPD_ERR_INVALID / SEMIPD_ERR_UNSUPPORTED
 *     synchronously and launch nothing.  Device-side outcomes (OOM, unknown free,
 *     table full, bad block) are written to *status_dev (int32, may be NULL) on
 *     the stream; the call itself returns SEMIPD_OK once launched.
 *   - n == 0 / batch == 0 / empty chunk is a no-op returning SEMIPD_OK.
 *   - Element dtype of every activation tensor equals the pool dtype (bf16 for FP8 pools).
 *   - One in-flight prefill call and one in-flight decode call per pool (one
 *     prefill worker stream and one decode worker stream); allocator calls
 *     may come from any number of streams / host threads (linearizable).
 */
#ifndef SEMIPD_H
#define SEMIPD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct semipd_pool* semipd_pool_t; /* opaque; owned by the library */
typedef void* semipd_stream_t;             /* cudaStream_t */

typedef enum {
    SEMIPD_OK = 0,
    SEMIPD_ERR_INVALID = 1,     /* bad host argument (nothing launched) */
    SEMIPD_ERR_OOM = 2,         /* alloc: sum(n_blocks) > free blocks; a normal outcome */
    SEMIPD_ERR_UNKNOWN_REQ = 3, /* free of a request holding no blocks / repeated id */
    SEMIPD_ERR_TABLE_FULL = 4,  /* alloc would exceed max_blocks_per_req */
    SEMIPD_ERR_BAD_BLOCK = 5,   /* attention met a block-table entry outside [0, num_blocks) */
    SEMIPD_ERR_CUDA = 6,        /* a CUDA runtime error (launch / attribute) */
    SEMIPD_ERR_UNSUPPORTED = 7  /* valid but unsupported shape / dtype combination */
} semipd_status;

/* Pool element dtype.  SEMIPD_FP8_E4M3 ("FP8 precision", DESIGN.md
 * reading R31): pages hold OCP E4M3 codes (1 byte); a bf16 element x is written as
 * E4M3_rne_satfinite(fl32(x / s)) and read as s * value(code), s the layer's tensor scale
 * (semipd_set_kv_scales).  Activations (q, k_new, v_new, out) of an FP8 pool are bf16.
 * Supported geometry: head_dim_k == head_dim_v == 128, block_size 64, even num_kv_heads, not
 * kv_shared (create returns UNSUPPORTED otherwise). */
typedef enum { SEMIPD_BF16 = 0, SEMIPD_FP32 = 1, SEMIPD_FP8_E4M3 = 2 } semipd_dtype;

/* Pool geometry.  One block id spans all layers (reading R8).
 * Layout in the caller's memory (device), every region 1 KiB aligned:
 *   [state words | free_stack int32[num_blocks] | nblk int32[max_reqs] |
 *    block_tables int32[max_reqs][max_blocks_per_req] | op log int32[oplog_words] |
 *    for l in layers: K_l [num_blocks][num_kv_heads][block_size][head_dim_k],
 *                     V_l [num_blocks][num_kv_heads][block_size][head_dim_v] (absent if kv_shared)]
 * "HND" pages: one (block, kv head) page is contiguous (4 KiB at bs 16, d 128, bf16). */
typedef struct {
    int32_t num_layers;
    int32_t num_blocks;         /* N_B */
    int32_t block_size;         /* tokens per block: 16, 32, 64 or 128 */
    int32_t num_kv_heads;       /* Hkv (per rank under TP) */
    int32_t head_dim_k;         /* dk */
    int32_t head_dim_v;         /* dv */
    int32_t kv_shared;          /* 1 = MLA latent cache: V aliases K[..., :head_dim_v] (dv <= dk) */
    int32_t max_reqs;           /* rows of the block table; request ids are in [0, max_reqs) */
    int32_t max_blocks_per_req; /* MBR */
    int32_t dtype;              /* semipd_dtype */
    int32_t device;             /* CUDA device ordinal the memory lives on */
    int32_t oplog_words;        /* int32 capacity of the allocator op log (0 = no log) */
} semipd_pool_config;

/* Bytes of device memory semipd_kv_pool_create needs for cfg (host; 0 if cfg invalid). */
size_t semipd_kv_pool_bytes(const semipd_pool_config* cfg);

/* Carve `mem` (>= semipd_kv_pool_bytes(cfg) bytes, 1 KiB aligned, device memory on
 * cfg->device) into the pool and initialise it on stream s: free stack
 * [N_B-1 ... 0] (first pops return 0, 1, 2, ...), top = N_B, tables = -1, counts 0,
 * K/V zero-filled.  Writes the new handle to *out (host).  The memory stays owned by
 * the caller and must outlive the pool.  Errors: INVALID (bad cfg / NULL), CUDA. */
semipd_status semipd_kv_pool_create(const semipd_pool_config* cfg, void* mem, size_t bytes,
                                    semipd_stream_t s, semipd_pool_t* out);

/* Release the handle (host state only; the caller frees the memory). */
semipd_status semipd_kv_pool_destroy(semipd_pool_t pool);

/* Borrowed device views (any pointer may be NULL): layer's K and V base
 * ([N_B][Hkv][bs][d]; V == K for kv_shared), block_tables [max_reqs][MBR], nblk
 * [max_reqs].  INVALID if layer is out of range. */
semipd_status semipd_kv_pool_views(semipd_pool_t pool, int32_t layer, void** k, void** v,
                                   int32_t** block_tables, int32_t** nblk);

/* ---- Unified memory manager: atomic block allocator (§4.4) ----
 * alloc: for i in argument order, append n_blocks[i] blocks (popped from the LIFO
 * free stack) to row req_ids[i].  All-or-nothing per call (reading R10): INVALID
 * (id outside [0,max_reqs) or n_blocks[i] < 1), else OOM if
 * sum(n_blocks) > free, else TABLE_FULL if a row would exceed MBR; any error
 * leaves the state unchanged.  The query -> get -> update sequence runs inside a
 * device lock (acquire/release) held by one CTA, so calls from different streams
 * linearise; each call's linearisation order is recorded in the op log.
 *   req_ids, n_blocks: device int32[n].  n: host.  status_dev: device int32 or NULL. */
semipd_status semipd_alloc_blocks(semipd_pool_t pool, const int32_t* req_ids,
                                  const int32_t* n_blocks, int32_t n, int32_t* status_dev,
                                  semipd_stream_t s);

/* free: push every block of each listed request back in table order, reset its
 * row to -1 and its count to 0.  UNKNOWN_REQ if a request holds no blocks or is
 * listed twice (double release); INVALID if an id is out of range; any error
 * rejects the whole call unchanged.  Stream order with the last kernel that read
 * those blocks is the caller's job (hazard H2). */
semipd_status semipd_free_blocks(semipd_pool_t pool, const int32_t* req_ids, int32_t n,
                                 int32_t* status_dev, semipd_stream_t s);

/* ceil(tokens / block_size); 0 -> 0; -1 if tokens < 0 or block_size <= 0. */
int32_t semipd_blocks_for_tokens(int32_t tokens, int32_t block_size);

/* Host-out stats: current free blocks and the minimum ever seen (utilisation
 * high-water).  Synchronises stream s. */
semipd_status semipd_pool_stats(semipd_pool_t pool, int32_t* free_blocks,
                                int32_t* min_free_seen, semipd_stream_t s);

/* Test hook (synchronises s): copy the op log to host_buf (<= bytes) and report
 * its length in int32 words (*n_words) and the number of ops not logged because
 * the log was full (*dropped).  Record: {seq, kind (1 alloc, 2 free), n, status,
 * req_ids[n], (alloc only) n_blocks[n]}, in linearisation (seq) order. */
semipd_status semipd_pool_oplog(semipd_pool_t pool, int32_t* host_buf, size_t bytes,
                                int64_t* n_words, int64_t* dropped, semipd_stream_t s);

/* ---- Computational resource controller ----
 * Set the (x, y) SM percentages of the prefill and decode phases, 0 < x, y <= 100;
 * x + y > 100 is allowed (oversubscription).  Budgets are
 * n = clamp(floor(num_SMs * pct / 100 + 1/2), 1, num_SMs).  Thread-safe atomic
 * host store; each phase adopts it at its next launch (delayed + asynchronous
 * switching); the pool, and so the KV cache, never moves.  INVALID if out of range. */
semipd_status semipd_set_partition(semipd_pool_t pool, double x_prefill_pct,
                                   double y_decode_pct);
/* Host-out current budgets (CTAs each phase's persistent grid is capped to). */
semipd_status semipd_get_sm_budgets(semipd_pool_t pool, int32_t* n_prefill,
                                    int32_t* n_decode);
/* SM count of the pool's device (host). */
int32_t semipd_num_sms(semipd_pool_t pool);

/* ---- Prefill attention (P:184, P:355, P:365 chunked prefill) ----
 * For request i (block-table row req_ids[i]) with chunk rows cu_seqlens_q[i] ..
 * cu_seqlens_q[i+1]-1 and prefix_lens[i] tokens already cached:
 *   1. writes k_new/v_new rows into the pool slots prefix_lens[i] + t (bit-exact);
 *   2. O[t,h,:] = sum_{j <= P_i + t} softmax_j(softmax_scale * q[t,h]·k[j,g(h)]) v[j,g(h)],
 *      g(h) = h / (num_q_heads / Hkv), keys read from the paged pool (bottom-right
 *      causal alignment).
 * Blocks covering positions [0, P_i + C_i) must be allocated (semipd_alloc_blocks);
 * an entry outside [0, N_B) sets *status_dev = BAD_BLOCK and is read as zeros.
 *   q [T][Hq][dk], k_new [T][Hkv][dk], v_new [T][Hkv][dv] (v_new ignored if
 *   kv_shared), out [T][Hq][dv] or, if out_head_major, [Hq][T][dv];
 *   cu_seqlens_q device int32[n+1], req_ids / prefix_lens device int32[n];
 *   total_q (host) = T = cu_seqlens_q[n]; max_chunk_len (host) >= every C_i;
 *   sm_budget (host): > 0 caps the persistent grid to that many CTAs, 0 = the
 *   partition's prefill budget, -1 = non-persistent (one CTA per work unit; the
 *   "(100,100) uncontrolled" baseline).
 * bf16 with dk = dv = 128 and (Hq/Hkv) | 128 runs the tcgen05/TMEM/TMA kernel;
 * other shapes run the generic CUDA-core kernel.  Output is bitwise identical
 * for every sm_budget (the work decomposition depends on shapes only).
 * FP8 pools (reading R31): step 1 quantises the rows; in step 2 keys j < P_i are the pool's
 * dequantised values (staged through the FP8 prefill scratch) and keys j >= P_i the chunk's
 * own bf16 rows; the tcgen05 kernel runs as for bf16.  Needs the scratch
 * (semipd_set_fp8_prefill_scratch) and no peer epilogue (else UNSUPPORTED); with RoPE set
 * (semipd_set_rope) step 1 rotates q / k_new in place and writes the rotated rows' codes in the
 * same pass. */
semipd_status semipd_prefill_attn(semipd_pool_t pool, int32_t layer, const void* q,
                                  const void* k_new, const void* v_new,
                                  const int32_t* cu_seqlens_q, const int32_t* req_ids,
                                  const int32_t* prefix_lens, int32_t n, int32_t total_q,
                                  int32_t max_chunk_len, int32_t num_q_heads,
                                  float softmax_scale, void* out, int32_t out_head_major,
                                  int32_t sm_budget, int32_t* status_dev, semipd_stream_t s);

/* ---- Decode attention (P:184, P:229 PagedAttention) ----
 * For each b: writes k_new[b]/v_new[b] to slot ctx_lens[b] (tokens cached BEFORE
 * the step, reading R5) of row req_ids[b] (the block covering that slot must be
 * allocated), then O[b,h,:] = attention of q[b,h] over keys 0 .. ctx_lens[b]
 * inclusive.  Split-K: keys are cut into S_b = ceil((ctx+1)/4096) splits of equal
 * 32-key-rounded length; partials are merged in split-index order by the last CTA
 * to finish (fused, no extra launch).
 *   q [B][Hq][dk], k_new [B][Hkv][dk], v_new [B][Hkv][dv], out [B][Hq][dv] or
 *   [Hq][B][dv] if out_head_major; req_ids / ctx_lens device int32[B];
 *   max_ctx_len (host) >= every ctx_lens[b];
 *   workspace: device scratch of >= semipd_decode_workspace_bytes(...) bytes,
 *   ZERO-FILLED before its first use (the kernels leave their counters at zero);
 *   sm_budget as in semipd_prefill_attn (0 = partition's decode budget).
 * FP8 pools (reading R31): the appended row is quantised and every key / value (the appended
 * one included) is read back dequantised; num_q_heads / Hkv <= 8; the peer epilogue
 * (semipd_set_decode_peers) is supported as for bf16; with RoPE set the rotation pass writes
 * the quantised rows and the kernel skips its own append.  Kernel: head-pair E4M3 boxes converted to f16 in registers,
 * f16 mma.sync with fp32 accumulation (kernel kind 9). */
semipd_status semipd_decode_attn(semipd_pool_t pool, int32_t layer, const void* q,
                                 const void* k_new, const void* v_new, const int32_t* req_ids,
                                 const int32_t* ctx_lens, int32_t batch, int32_t max_ctx_len,
                                 int32_t num_q_heads, float softmax_scale, void* out,
                                 int32_t out_head_major, void* workspace, size_t ws_bytes,
                                 int32_t sm_budget, int32_t* status_dev, semipd_stream_t s);

/* Workspace bytes for decode calls with batch <= max_batch and ctx <= max_ctx (host). */
size_t semipd_decode_workspace_bytes(semipd_pool_t pool, int32_t max_batch,
                                     int32_t num_q_heads, int32_t max_ctx);

/* ---- Instrumentation (host) ----
 * Number of kernels this pool handle has launched so far (every launch the
 * library issues is counted).  Used for bench.py's "gpu_launches". */
int64_t semipd_launch_count(semipd_pool_t pool);

/* Optional CTA trace for co-run evidence: when buf (device int32, capacity
 * `cap` records of 4 words) is non-NULL every attention CTA appends
 * {phase (1 prefill, 2 decode), %smid, blockIdx.x, kernel kind (0 CUDA-core generic,
 * 1 tcgen05 prefill, 2 split-K decode, 3 MLA mma.sync decode, 4 MLA tcgen05 decode,
 * 5 MLA tcgen05 prefill, 6 / 7 / 8 wide-box split-K decode: head pairs at 64-token pages /
 * whole 128-token pages / head pairs at 16-token pages, 9 FP8 E4M3 head-pair decode)};
 * *counter_dev (device int32)
 * is the append cursor.  Pass buf = NULL to disable. */
semipd_status semipd_set_trace(semipd_pool_t pool, int32_t* buf, int32_t cap,
                               int32_t* counter_dev);

/* Device-side launch timing (measurement hook; SURVEY §8(d) "Timing").  buf: device array of
 * cap x 8 uint64, zero-filled by the caller, owned by the caller.  From this call on, the
 * i-th attention kernel launched through this pool (the tcgen05 / split-K / MLA kernels of
 * either phase; the generic CUDA-core path records nothing) uses record i % cap, and every CTA stamps %globaltimer at entry and after its last barrier; the CTA
 * that finishes last folds the launch into the record:
 *   [2] += end - start (ns, start = first CTA entry, end = last CTA exit), [3] += 1,
 *   [5] / [6] = that launch's start / end; [0], [1], [4] are running state (zero between
 *   launches).
 * A launch captured into a CUDA graph keeps its record, so [2] / [3] average it over the
 * replays.  The host cursor restarts at 0 with every call.  buf = NULL disables (default).
 * Errors: INVALID (NULL pool, cap <= 0 with a buffer). */
semipd_status semipd_set_spans(semipd_pool_t pool, uint64_t* buf, int32_t cap);

/* ---- Head-output all-gather over peer memory (TP by KV head) ----
 * P:232 §4.5: the prefill workers (and, separately, the decode workers) of a TP group
 * exchange only among themselves.  With attention sharded by KV head the one exchange is
 * the all-gather of head-major shards [Hq/TP, T, dv] into [Hq, T, dv] on every rank.
 * These calls do it with the copy engines and GPU-front-end stream memory operations, so
 * the gather occupies no SM of either partition (NCCL's all-gather runs CTAs).
 *
 * semipd_ipc_alloc: the ONE call that allocates device memory: `bytes` (> 0) of zeroed
 *   cudaMalloc memory on the current device, exportable to other processes.  *dev_ptr
 *   receives it, handle_out (host, SEMIPD_IPC_HANDLE_BYTES bytes) its IPC handle.  Owned by
 *   the caller; release with semipd_ipc_free.  Errors: INVALID (NULL / 0), CUDA.
 * semipd_ipc_open: map a peer's handle (host bytes) into this process (peer access enabled
 *   lazily); *dev_ptr is the peer allocation's base.  Unmap with semipd_ipc_close.  A handle
 *   cannot be opened in the process that created it (CUDA rule): CUDA.
 * semipd_peer_gather: on stream s, for rank `rank` of `world` (1..SEMIPD_MAX_PEERS):
 *   - entry handshake: set peer_flags[k][world + rank] for every k != rank, then wait for
 *     my_flags[world + k] to be set by every k != rank and reset it (every peer has reached
 *     this call in its stream order, so its reads of the previous gather are done);
 *   - copy `bytes` from src (device, this rank's shard) to dsts[k] for every k (host array of
 *     `world` device pointers: rank k's gathered buffer, already offset to this rank's shard;
 *     dsts[rank] == src skips the local copy);
 *   - set peer_flags[k][rank] (host array of `world` device pointers to each rank's flag
 *     array as mapped in this process; the write is fenced after the copies);
 *   - wait for my_flags[k] to be set by every k != rank and reset it (my_flags: this rank's
 *     own 2*world uint32 flag array, zero-initialised, used by one stream at a time).
 *   Flags only take the values 0 / 1 and every call issues the same operations, so the call
 *   may be captured into a CUDA graph and replayed.  After the call's stream position the
 *   gathered buffer holds every rank's shard.  All ranks must make the same sequence of
 *   calls on a given flag array.  Errors: INVALID (bad rank / world / NULL), UNSUPPORTED (no
 *   stream memory operations), CUDA. */
#define SEMIPD_IPC_HANDLE_BYTES 64
#define SEMIPD_MAX_PEERS 8
semipd_status semipd_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out);
semipd_status semipd_ipc_free(void* dev_ptr);
semipd_status semipd_ipc_open(const void* handle, void** dev_ptr);
semipd_status semipd_ipc_close(void* dev_ptr);
semipd_status semipd_peer_gather(const void* src, size_t bytes, void* const* dsts,
                                 uint32_t* const* peer_flags, uint32_t* my_flags, int32_t world,
                                 int32_t rank, semipd_stream_t s);

/* ---- The decode head gather fused into the decode kernel's epilogue ----
 * semipd_set_decode_peers: later semipd_decode_attn calls on this pool ALSO store every output
 * vector to peer_out[k] + (the same element offset as in `out`), k < n (host array of device
 * pointers, n <= SEMIPD_MAX_PEERS - 1; n = 0 clears).  With head-major output
 * ([Hq/TP, B, dv], out_head_major = 1, required) and peer_out[k] = peer k's gathered buffer
 * [Hq, B, dv] as mapped in this process, offset to this rank's head slice, the kernel's
 * epilogue performs this rank's part of the all-gather itself (posted NVLink stores, no
 * copies).  Bracket each such decode call with semipd_peer_handshake: which = 0 ("ready")
 * before it, so no peer is still reading the buffer, and which = 1 ("landed") after it, which
 * fences the kernel's stores and waits until every peer's have landed here.  Only the split-K
 * decode kernels (bf16 and E4M3 pages) support peers: other decode paths return UNSUPPORTED, row-major
 * output INVALID.  `tokens` (> 0 when n > 0) is the token count B the gathered buffers were
 * sized for ([Hq, tokens, dv]): the peer offsets depend on it, so a later decode call whose
 * batch differs returns INVALID (and launches nothing) instead of storing at wrong offsets or
 * past a peer's buffer.  Errors: INVALID (NULL pool, n out of range, NULL / unaligned pointer,
 * tokens <= 0 with n > 0).
 * semipd_peer_handshake: one of the two handshakes semipd_peer_gather performs (flag arrays
 * as there; which: 0 = ready, 1 = landed), as one batched stream-memory-operation call. */
semipd_status semipd_set_decode_peers(semipd_pool_t pool, void* const* peer_out, int32_t n,
                                      int32_t tokens);
/* The same for semipd_prefill_attn (tcgen05 GQA path only; 16-byte aligned pointers): full
 * output tiles then take the direct 16-byte-store epilogue instead of the TMA store, and
 * every output vector also goes to each peer.  `tokens` = the total_q the gathered buffers
 * were sized for; a prefill call with another total_q returns INVALID. */
semipd_status semipd_set_prefill_peers(semipd_pool_t pool, void* const* peer_out, int32_t n,
                                       int32_t tokens);
semipd_status semipd_peer_handshake(uint32_t* const* peer_flags, uint32_t* my_flags,
                                    int32_t world, int32_t rank, int32_t which, semipd_stream_t s);

/* ---- Rotary position embedding of the step's new rows ----
 * P:355 §6: "To support the Llama3.1 series model, we also modify the RoPE kernel."
 * Rotates q [num_tokens][num_q_heads][head_dim] and k [num_tokens][num_kv_heads][head_dim]
 * (device, token-major, contiguous, 16-byte aligned, pool dtype `dtype`) IN PLACE for the
 * token positions positions[num_tokens] (device int32), before the attention call that
 * writes k into the pool.  Only columns [rot_offset, rot_offset + rot_dim) of each row
 * rotate (Llama: 0, head_dim; the MLA latent row's decoupled rope part: 512, 64); the other
 * columns are not touched.  With R = rot_dim (reading R27):
 *   pairs: (i, i + R/2) if interleaved == 0 (Llama / NeoX), (2i, 2i + 1) otherwise
 *          (GPT-J / DeepSeek), i < R/2;
 *   f_i = theta^(-2i/R); if factor > 1, the Llama-3.1 rescaling with wavelength
 *   w_i = 2 pi / f_i and L0 = original_max_pos: w_i < L0/high_freq_factor -> f_i;
 *   w_i > L0/low_freq_factor -> f_i / factor; otherwise (1-a) f_i / factor + a f_i with
 *   a = (L0 / w_i - low_freq_factor) / (high_freq_factor - low_freq_factor);
 *   phi = pos * f_i;  (x, y) of pair i -> (x cos phi - y sin phi, y cos phi + x sin phi).
 * The frequencies, the angle and its sine / cosine are formed in fp64, the rotation in fp32.
 * factor <= 1 disables the rescaling (plain RoPE).  q (k) may be NULL when its head count is
 * 0.  Errors: INVALID (negative sizes, odd / empty rot_dim, range outside the row,
 * theta <= 1, bad scaling parameters, NULL), UNSUPPORTED (head_dim, rot_offset or the
 * per-vector span (R/2 half-split, R interleaved) not a multiple of 8 (bf16) / 4 (fp32)
 * elements, R > 256, misaligned rows), CUDA.  num_tokens == 0 is a no-op. */
semipd_status semipd_rope(void* q, void* k, const int32_t* positions, int32_t num_tokens,
                          int32_t num_q_heads, int32_t num_kv_heads, int32_t head_dim,
                          int32_t rot_offset, int32_t rot_dim, int32_t interleaved, int32_t dtype,
                          double theta, double factor, double low_freq_factor,
                          double high_freq_factor, int32_t original_max_pos, semipd_stream_t s);

/* ---- RoPE fused with the K/V write of the attention calls ----
 * semipd_set_rope: from now on, every semipd_prefill_attn / semipd_decode_attn on this pool
 * first rotates the step's new rows exactly as semipd_rope would (same definition, same fp64
 * angles, same fp32 rotation: bit-identical rows) at the positions the call's layout implies
 *   prefill: row t of request r (chunk-relative) sits at prefix_lens[r] + t   (R4)
 *   decode:  request b's new row sits at ctx_lens[b]                           (R5)
 * and in the SAME pass writes the rotated k rows (and v) into the pool slots of those
 * positions, replacing both the separate semipd_rope pass and the attention kernels' own
 * K/V write / append (one pass over q / k / v instead of two; R28).  q and k_new
 * are rotated IN PLACE (the attention then reads the rotated rows).  On an FP8 (E4M3) pool the
 * pass writes the rows as codes with the pool's write rule (R31), the bytes the FP8 calls' own
 * write would store from the rotated rows.  cfg = NULL turns it off.
 * cfg fields as semipd_rope's arguments; head_dim = the pool's head_dim_k.  Errors: INVALID /
 * UNSUPPORTED as semipd_rope, plus INVALID for a NULL pool. */
typedef struct {
    double theta, factor, low_freq_factor, high_freq_factor;
    int32_t original_max_pos, rot_offset, rot_dim, interleaved;
} semipd_rope_config;
semipd_status semipd_set_rope(semipd_pool_t pool, const semipd_rope_config* cfg);

/* ---- FP8 (E4M3) pools (reading R31) ----
 * semipd_set_kv_scales: per-layer tensor scales (host float[num_layers] each, every value
 * finite and > 0; NULL leaves that tensor's scales unchanged).  Default 1.0.  Later K/V writes
 * quantise with them and later attention calls dequantise with them; changing a layer's scale
 * does not rewrite pages already stored.  INVALID on a bad value or a non-FP8 pool. */
semipd_status semipd_set_kv_scales(semipd_pool_t pool, const float* k_scales,
                                   const float* v_scales);

/* Prefill on an FP8 pool reads the cached prefix through a bf16 staging copy: before the
 * tcgen05 attention a dequantisation pass writes s * value(code) of every prefix page of the
 * call into caller-owned scratch (request i of the call gets pages [i * MBR, (i + 1) * MBR)).
 * semipd_fp8_prefill_scratch_bytes: bytes for calls of up to max_reqs_per_call requests (host;
 * 0 if the pool is not FP8 or the argument < 1).
 * semipd_set_fp8_prefill_scratch: hand the scratch (device, >= that many bytes, 1 KiB aligned,
 * owned by the caller and alive while prefill calls run; NULL detaches).  It initialises the
 * scratch's tables synchronously.  An FP8 prefill call with more requests than the scratch was
 * sized for, or with no scratch, returns INVALID. */
size_t semipd_fp8_prefill_scratch_bytes(semipd_pool_t pool, int32_t max_reqs_per_call);
semipd_status semipd_set_fp8_prefill_scratch(semipd_pool_t pool, void* mem, size_t bytes,
                                             int32_t max_reqs_per_call);

/* ---- Expanded-form MLA prefill (reading R32) ----
 * P:362-365 / P:395 run DeepSeek (MLA) models; the cache is the latent pool (kv_shared, one
 * 576-wide row per key: c_j = columns 0..511, k_pe_j = columns 512..575).  For request i
 * (block-table row req_ids[i], chunk rows cu_seqlens_q[i] .. cu_seqlens_q[i+1]-1, P_i =
 * prefix_lens[i] keys cached):
 *   1. writes kv_new rows into the pool slots P_i + t (bit copies);
 *   2. expands every key j < P_i + C_i of the request with the up-projections:
 *        k_nope[j][h] = bf16(W_UK[h] c_j) (128), v[j][h] = bf16(W_UV[h] c_j) (128)
 *      (fp32 accumulation on the tensor cores, one round-to-nearest-even to bf16);
 *   3. O[t,h,:] = sum_{j <= P_i + t} softmax_j(softmax_scale * q[t,h] . [k_nope[j][h] | k_pe_j])
 *      v[j][h] (causal, bottom-right aligned).
 *   q [T][H][192] bf16 (q_nope 128 | q_pe 64), kv_new [T][576] bf16, w_uk [H][128][512] and
 *   w_uv [H][128][512] bf16 (row-major, 16-byte aligned), out [T][H][128] bf16;
 *   cu_seqlens_q device int32[n+1], req_ids / prefix_lens device int32[n] (n <= 1024);
 *   total_q (host) = cu_seqlens_q[n]; max_chunk_len (host) >= every C_i;
 *   max_total_keys (host) >= sum_i (P_i + C_i) (a smaller sum than the device data sets
 *   *status_dev = INVALID and nothing is written);
 *   workspace: device scratch, 256-byte aligned, >= semipd_prefill_mla_expanded_workspace_bytes
 *   (pool, n, max_total_keys, H) bytes, owned by the caller (holds the expanded K / V; no
 *   zero-fill needed);
 *   sm_budget as in semipd_prefill_attn (caps each of the three persistent grids).
 * Pool: bf16, kv_shared, one KV head, head_dim_k 576, block_size in {16, 32, 64, 128}; H even,
 * <= 128 (else UNSUPPORTED / INVALID).  A block-table entry outside [0, N_B) sets BAD_BLOCK and
 * that key's latent is read as zeros.  No peer epilogue (UNSUPPORTED).  With RoPE set
 * (semipd_set_rope, rot_offset >= 512: MLA's decoupled k_pe columns, else UNSUPPORTED) the call
 * first rotates q_pe = q[..., 128 + (rot_offset - 512) ...] and kv_new's rope columns in place
 * at prefix_lens[r] + t, with the same frequencies, before the prep writes the latent rows.
 * Kernels: a prep pass (copies), a tcgen05 up-projection GEMM over TMA-gathered pool pages, a
 * tcgen05 causal attention kernel with dqk 192 / dv 128 (trace kernel kind 10); three launches,
 * each with a launch span (semipd_set_spans) in that order. */
size_t semipd_prefill_mla_expanded_workspace_bytes(semipd_pool_t pool, int32_t max_reqs,
                                                   int32_t max_total_keys, int32_t num_heads);
semipd_status semipd_prefill_mla_expanded(semipd_pool_t pool, int32_t layer, const void* q,
                                          const void* kv_new, const void* w_uk, const void* w_uv,
                                          const int32_t* cu_seqlens_q, const int32_t* req_ids,
                                          const int32_t* prefix_lens, int32_t n, int32_t total_q,
                                          int32_t max_chunk_len, int32_t max_total_keys,
                                          int32_t num_heads, float softmax_scale, void* out,
                                          void* workspace, size_t ws_bytes, int32_t sm_budget,
                                          int32_t* status_dev, semipd_stream_t s);

/* Library version string (host, static). */
const char* semipd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SEMIPD_H */
