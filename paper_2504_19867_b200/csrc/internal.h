// internal.h — host-side pool handle shared by the library's translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <utility>
#include <vector>

#include "semipd.h"

// Device-resident allocator / scheduler state (first region of the pool).
struct SpdDevState {
    unsigned int lock;             // allocator lock word (0 free, 1 held)
    int top;                       // free-stack height == free blocks
    int min_free;                  // high-water of utilisation (min free seen)
    int pad0;
    unsigned long long op_seq;     // linearisation sequence number of the next op
    long long oplog_len;           // int32 words used in the op log
    long long oplog_dropped;       // ops not logged (log full)
    unsigned int sched[16];        // persistent-grid work counters (prefill uses [0..1])
};

struct semipd_pool {
    semipd_pool_config cfg;
    int num_sms = 0;
    unsigned char* base = nullptr;
    SpdDevState* st = nullptr;
    int* free_stack = nullptr;
    int* nblk = nullptr;
    int* bt = nullptr;
    int* oplog = nullptr;
    unsigned char* kv = nullptr;
    size_t k_layer_bytes = 0, v_layer_bytes = 0, layer_stride = 0;
    size_t esize = 2;
    std::atomic<int> n_prefill{1}, n_decode{1};
    std::atomic<long long> epoch{0};
    std::atomic<long long> launches{0};
    // TMA descriptors of every layer's K and V pool ([N_B*Hkv] pages of
    // [bs][d]; box = 64 columns x min(bs, 32) rows, 128-byte swizzle).
    std::vector<CUtensorMap> kmap, vmap;
    // decode maps: 4-D (64 cols, dk/64 column blocks, bs rows, pages), box = one
    // whole page-row-block of min(bs, 64) rows x all column blocks, 128-byte swizzle
    std::vector<CUtensorMap> dkmap, dvmap;
    bool have_maps = false;   // 3-D page maps (prefill)
    bool have_dmaps = false;  // 4-D page maps (decode)
    // decode wide-box maps, 32 KiB per box: bs 64 with even Hkv -> 64 rows x 128 columns x 2
    // adjacent (block, head) pages; bs 128 -> one whole 128-row page
    std::vector<CUtensorMap> dkmap2, dvmap2;
    bool have_wide_maps = false;
    bool force_single = false;  // debug/bench: keep the one-head decode kernel
    bool force_pair = false;    // debug/bench: head-pair boxes at 64-token pages for any batch
    // decode epilogue peer stores (semipd_set_decode_peers; TP gather fused into the kernel)
    void* dec_peers[SEMIPD_MAX_PEERS - 1] = {};
    int dec_n_peers = 0;
    int dec_peer_tokens = 0;  // batch the decode peers' gathered buffers were sized for
    void* pre_peers[SEMIPD_MAX_PEERS - 1] = {};  // semipd_set_prefill_peers
    int pre_n_peers = 0;
    int pre_peer_tokens = 0;  // total_q the prefill peers' gathered buffers were sized for
    // MLA latent pool (kv_shared): 4-D (64 cols, rows, dk/64 blocks, pages), box 32 rows x all
    // column blocks (one 36 KiB TMA per 32-key stage at dk = 576)
    std::vector<CUtensorMap> mla_kmap;
    bool have_mla_map = false;
    // MLA tcgen05 decode (bs 64): the same 4-D view, boxes of 64 rows x column blocks
    // [0, 4) (32 KiB) and [4, 9) (40 KiB) — one page in two TMA boxes
    std::vector<CUtensorMap> mla_lo, mla_hi;
    bool have_mla_tc_maps = false;
    int box_rows = 16;
    int dbox_rows = 16;
    int* trace_buf = nullptr;
    int trace_cap = 0;
    int* trace_ctr = nullptr;
    // semipd_set_rope: RoPE of the step's new q / k rows fused with the K/V write
    bool rope_on = false;
    semipd_rope_config rope{};
    double rope_inv_freq[128] = {};
    unsigned long long* span_buf = nullptr;  // semipd_set_spans: 8 x u64 per launch slot
    int span_cap = 0;
    int span_next = 0;
    // FP8 E4M3 pools (reading R31): per-layer tensor scales, decode head-pair maps (128 code
    // bytes x 64 rows x 2 pages per box), and the prefill staging scratch with its bf16 maps
    std::vector<float> k_scale, v_scale;
    std::vector<CUtensorMap> f8kmap, f8vmap;
    bool have_f8_maps = false;
    unsigned char* f8s = nullptr;
    int f8s_cap = 0;
    CUtensorMap f8s_kmap{}, f8s_vmap{};
    bool have_f8s_maps = false;
    void* timeline = nullptr;      // debug builds (SPD_TIMELINE): prefill clock64 stamps
    int* timeline_ctr = nullptr;

    void* k_layer(int l) const { return kv + (size_t)l * layer_stride; }
    void* v_layer(int l) const {
        return cfg.kv_shared ? k_layer(l) : (void*)(kv + (size_t)l * layer_stride + k_layer_bytes);
    }
};

// Trace sink passed by value to kernels.
struct SpdTrace {
    int* buf;
    int cap;
    int* ctr;
};

inline SpdTrace spd_trace(const semipd_pool* p) { return SpdTrace{p->trace_buf, p->trace_cap, p->trace_ctr}; }

// launch-span slot of the next attention launch (semipd_set_spans), or nullptr when off
inline unsigned long long* spd_next_span(semipd_pool* p) {
    if (!p->span_buf || p->span_cap <= 0) return nullptr;
    unsigned long long* r = p->span_buf + 8 * (size_t)(p->span_next % p->span_cap);
    p->span_next += 1;
    return r;
}

// budget resolution (host): >0 cap, 0 partition, -1 non-persistent
inline int spd_resolve_budget(const semipd_pool* p, int requested, bool prefill) {
    if (requested > 0) return requested < p->num_sms ? requested : p->num_sms;
    if (requested == 0) return prefill ? p->n_prefill.load() : p->n_decode.load();
    return -1;
}

// TMA encode through the driver entry point (no -lcuda link dependency)
bool spd_encode_tiled_4d(CUtensorMap* map, CUtensorMapDataType dt, void* gaddr, const uint64_t* dims,
                         const uint64_t* strides_bytes /* 3 */, const uint32_t* box,
                         CUtensorMapSwizzle swz);
bool spd_encode_tiled_3d(CUtensorMap* map, CUtensorMapDataType dt, void* gaddr, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint64_t s1_bytes, uint64_t s2_bytes,
                         uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swz);

// Decode workspace (every decode kernel): [sched 256 B | split counters, 4 B each] from the
// front, the fp32 split partials (m, l, acc) packed against the END of the caller's buffer.
// Counters must be zero when a kernel starts (kernels reset the ones they use); a counter byte
// is never a partial byte of any call, whatever its batch size, because
// semipd_decode_workspace_bytes() reserves counters for max_batch plus the largest partial set.
struct SpdWs {
    unsigned* sched;
    int* cnt;
    float* m;
    float* l;
    float* acc;
};
inline size_t spd_al256(size_t x) { return (x + 255) / 256 * 256; }
inline size_t spd_ws_counter_bytes(size_t n_cnt) { return spd_al256(256 + 4 * n_cnt); }
inline size_t spd_ws_partial_bytes(size_t rows, size_t S, size_t dv) {  // rows = B x Hq
    return 2 * spd_al256(rows * S * 4) + spd_al256(rows * S * dv * 4);
}
inline bool spd_ws_carve(void* ws, size_t ws_bytes, size_t n_cnt, size_t rows, size_t S, size_t dv,
                         SpdWs* o) {
    const size_t cb = spd_ws_counter_bytes(n_cnt), pb = spd_ws_partial_bytes(rows, S, dv);
    if (!ws || ws_bytes < cb + pb) return false;
    unsigned char* b = static_cast<unsigned char*>(ws);
    const size_t base = (ws_bytes - pb) & ~static_cast<size_t>(255);
    if (base < cb) return false;
    o->sched = reinterpret_cast<unsigned*>(b);
    o->cnt = reinterpret_cast<int*>(b + 256);
    o->m = reinterpret_cast<float*>(b + base);
    o->l = reinterpret_cast<float*>(b + base + spd_al256(rows * S * 4));
    o->acc = reinterpret_cast<float*>(b + base + 2 * spd_al256(rows * S * 4));
    return true;
}

// kernels launched from other TUs
bool spd_mla_decode_ok(const semipd_pool* p, int Hq);
size_t spd_mla_ws_bytes(int B, int max_ctx);
semipd_status spd_launch_decode_mla(semipd_pool_t pool, int layer, const void* q, const void* k_new,
                                    const int* req_ids, const int* ctx_lens, int batch,
                                    int max_ctx_len, int Hq, float scale, void* out,
                                    int out_head_major, void* workspace, size_t ws_bytes,
                                    int budget, int* status_dev, cudaStream_t st);
bool spd_mla_prefill_ok(const semipd_pool* p, int Hq);
semipd_status spd_launch_prefill_mla(semipd_pool_t pool, int layer, const void* q,
                                     const int* cu_seqlens, const int* req_ids,
                                     const int* prefix_lens, int n, int total_q, int max_chunk_len,
                                     int Hq, float scale, void* out, int out_head_major,
                                     int budget, int* status_dev, cudaStream_t st);
bool spd_mla_tc_ok(const semipd_pool* p, int Hq);
size_t spd_mla_tc_ws_bytes(int B, int max_ctx);
semipd_status spd_launch_decode_mla_tc(semipd_pool_t pool, int layer, const void* q,
                                       const void* k_new, const int* req_ids, const int* ctx_lens,
                                       int batch, int max_ctx_len, int Hq, float scale, void* out,
                                       int out_head_major, void* workspace, size_t ws_bytes,
                                       int budget, int* status_dev, cudaStream_t st);
// RoPE of q / k_new in place at the rows' positions (prefill: prefix + chunk index; decode:
// ctx) fused with the K/V write of the rotated rows into the pool (rope.cu)
semipd_status spd_launch_rope_write(semipd_pool_t p, int layer, void* q, void* k_new,
                                    const void* v_new, const int* cu_seqlens, const int* req_ids,
                                    const int* base_pos, int n, int T, int Hq, int* status_dev,
                                    cudaStream_t s);
// the same pass with q rows of q_dk columns rotated from column q_off (the pool's k columns from
// its rot_offset); write_pool = 0 rotates q / k_new in place only
semipd_status spd_launch_rope_write_ex(semipd_pool_t p, int layer, void* q, int q_dk, int q_off,
                                       void* k_new, const void* v_new, const int* cu_seqlens,
                                       const int* req_ids, const int* base_pos, int n, int T, int Hq,
                                       int write_pool, int* status_dev, cudaStream_t s);
semipd_status spd_launch_kv_write(semipd_pool_t p, int layer, const void* k_new, const void* v_new,
                                  const int* cu_seqlens, const int* req_ids, const int* pos0,
                                  int n, int total_rows, int mode, int* status_dev,
                                  cudaStream_t s);
// FP8 E4M3 pools (fp8.cu)
bool spd_fp8_geometry_ok(const semipd_pool_config* c);
int spd_fp8_pieces();  // split partials per 4096-key split of the FP8 decode kernel
bool spd_fp8_init_maps(semipd_pool* p);
semipd_status spd_launch_kv_write_fp8(semipd_pool_t p, int layer, const void* k_new, const void* v_new,
                                      const int* cu_seqlens, const int* req_ids, const int* pos0,
                                      int n, int total_rows, int* status_dev, cudaStream_t s);
semipd_status spd_launch_dequant_prefix(semipd_pool_t p, int layer, const int* req_ids,
                                        const int* prefix_lens, int n, int budget, int* status_dev,
                                        cudaStream_t s);
void spd_fp8_prefill_view(const semipd_pool* p, const int** ids, const int** bt, int* n_blocks);
semipd_status spd_launch_decode_fp8(semipd_pool_t pool, int layer, const void* q, const void* k_new,
                                    const void* v_new, const int* req_ids, const int* ctx_lens,
                                    int batch, int max_ctx_len, int Hq, float scale, void* out,
                                    int out_head_major, void* workspace, size_t ws_bytes, int budget,
                                    int* status_dev, cudaStream_t st);
semipd_status spd_launch_simt_attn(semipd_pool_t p, int layer, const void* q, const int* cu_seqlens,
                                   const int* req_ids, const int* pos0, int n, int total_rows,
                                   int mode, int Hq, float scale, void* out, int out_head_major,
                                   int budget, int* status_dev, cudaStream_t s);

// Launch `k` on st with programmatic stream serialization (PDL): the kernel's prologue may
// overlap the previous kernel's tail; every kernel launched this way calls pdl_wait() before
// its first dependent global access.  SEMIPD_NO_PDL=1 in the environment launches plainly (A/B).
bool spd_pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t spd_launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                           Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = spd_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

