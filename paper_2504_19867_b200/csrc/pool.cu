// pool.cu — unified paged KV pool (§4.4): layout carve, init, views,
// stats, op log, partition (§4.3), TMA descriptors.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <new>

#include "common.cuh"
#include "internal.h"
#include <cstdlib>

namespace {

constexpr size_t kAlign = 1024;
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Layout {
    size_t off_state, off_free, off_nblk, off_bt, off_oplog, off_kv;
    size_t k_layer, v_layer, layer_stride, total;
};

size_t elem_bytes(int dtype) { return dtype == SEMIPD_BF16 ? 2 : dtype == SEMIPD_FP32 ? 4 : 1; }

bool valid_cfg(const semipd_pool_config* c) {
    if (!c) return false;
    if (c->num_layers < 1 || c->num_blocks < 1 || c->block_size < 1 || c->num_kv_heads < 1)
        return false;
    if (c->head_dim_k < 1 || c->head_dim_k > 1024 || c->head_dim_v < 1 || c->head_dim_v > 1024)
        return false;
    if (c->kv_shared && c->head_dim_v > c->head_dim_k) return false;
    if (c->max_reqs < 1 || c->max_blocks_per_req < 1 || c->oplog_words < 0) return false;
    if (c->dtype != SEMIPD_BF16 && c->dtype != SEMIPD_FP32 && c->dtype != SEMIPD_FP8_E4M3) return false;
    const size_t eb = elem_bytes(c->dtype);
    if ((c->head_dim_k * eb) % 16 || (c->head_dim_v * eb) % 16) return false;  // 16-B rows
    return true;
}

Layout layout_of(const semipd_pool_config* c) {
    Layout L{};
    const size_t eb = elem_bytes(c->dtype);
    size_t o = 0;
    L.off_state = o;
    o = align_up(o + sizeof(SpdDevState), kAlign);
    L.off_free = o;
    o = align_up(o + sizeof(int) * (size_t)c->num_blocks, kAlign);
    L.off_nblk = o;
    o = align_up(o + sizeof(int) * (size_t)c->max_reqs, kAlign);
    L.off_bt = o;
    o = align_up(o + sizeof(int) * (size_t)c->max_reqs * c->max_blocks_per_req, kAlign);
    L.off_oplog = o;
    o = align_up(o + sizeof(int) * (size_t)c->oplog_words, kAlign);
    L.off_kv = o;
    const size_t page = (size_t)c->num_blocks * c->num_kv_heads * c->block_size;
    L.k_layer = page * c->head_dim_k * eb;
    L.v_layer = c->kv_shared ? 0 : page * c->head_dim_v * eb;
    L.layer_stride = align_up(L.k_layer + L.v_layer, kAlign);
    L.total = o + L.layer_stride * (size_t)c->num_layers;
    return L;
}

__global__ void init_pool_kernel(SpdDevState* st, int* free_stack, int* nblk, int* bt, int N_B,
                                 int R, long long nbt) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = tid; i < N_B; i += stride) free_stack[i] = N_B - 1 - (int)i;
    for (long long i = tid; i < R; i += stride) nblk[i] = 0;
    for (long long i = tid; i < nbt; i += stride) bt[i] = -1;
    if (tid == 0) {
        st->lock = 0u;
        st->top = N_B;
        st->min_free = N_B;
        st->op_seq = 0ull;
        st->oplog_len = 0;
        st->oplog_dropped = 0;
        for (int i = 0; i < 16; ++i) st->sched[i] = 0u;
    }
}

typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

PFN_encodeTiled_t get_encode() {
    static PFN_encodeTiled_t fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled_t>(p);
    }
    return fn;
}

}  // namespace

bool spd_encode_tiled_3d(CUtensorMap* map, CUtensorMapDataType dt, void* gaddr, uint64_t d0,
                         uint64_t d1, uint64_t d2, uint64_t s1_bytes, uint64_t s2_bytes,
                         uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swz) {
    PFN_encodeTiled_t enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {d0, d1, d2};
    cuuint64_t strides[2] = {s1_bytes, s2_bytes};
    cuuint32_t box[3] = {b0, b1, b2};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(map, dt, 3, gaddr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool spd_encode_tiled_4d(CUtensorMap* map, CUtensorMapDataType dt, void* gaddr, const uint64_t* dims,
                         const uint64_t* strides_bytes, const uint32_t* box,
                         CUtensorMapSwizzle swz) {
    PFN_encodeTiled_t enc = get_encode();
    if (!enc) return false;
    cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
    cuuint64_t st[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
    cuuint32_t b[4] = {box[0], box[1], box[2], box[3]};
    cuuint32_t e[4] = {1, 1, 1, 1};
    CUresult r = enc(map, dt, 4, gaddr, d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

extern "C" {

const char* semipd_version(void) { return "semipd-b200 0.1 (sm_100a)"; }

size_t semipd_kv_pool_bytes(const semipd_pool_config* cfg) {
    if (!valid_cfg(cfg)) return 0;
    return layout_of(cfg).total;
}

int32_t semipd_blocks_for_tokens(int32_t tokens, int32_t block_size) {
    if (tokens < 0 || block_size <= 0) return -1;
    return (int32_t)(((int64_t)tokens + block_size - 1) / block_size);
}

semipd_status semipd_kv_pool_create(const semipd_pool_config* cfg, void* mem, size_t bytes,
                                    semipd_stream_t s, semipd_pool_t* out) {
    if (!valid_cfg(cfg) || !mem || !out) return SEMIPD_ERR_INVALID;
    if (cfg->dtype == SEMIPD_FP8_E4M3 && !spd_fp8_geometry_ok(cfg)) return SEMIPD_ERR_UNSUPPORTED;
    if (reinterpret_cast<uintptr_t>(mem) % kAlign) return SEMIPD_ERR_INVALID;
    const Layout L = layout_of(cfg);
    if (bytes < L.total) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    int prev = 0;
    if (cudaGetDevice(&prev) != cudaSuccess) return SEMIPD_ERR_CUDA;
    if (cudaSetDevice(cfg->device) != cudaSuccess) return SEMIPD_ERR_INVALID;
    semipd_pool* p = new (std::nothrow) semipd_pool();
    if (!p) return SEMIPD_ERR_CUDA;
    p->cfg = *cfg;
    if (cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, cfg->device) !=
        cudaSuccess) {
        delete p;
        cudaSetDevice(prev);
        return SEMIPD_ERR_CUDA;
    }
    p->base = static_cast<unsigned char*>(mem);
    p->st = reinterpret_cast<SpdDevState*>(p->base + L.off_state);
    p->free_stack = reinterpret_cast<int*>(p->base + L.off_free);
    p->nblk = reinterpret_cast<int*>(p->base + L.off_nblk);
    p->bt = reinterpret_cast<int*>(p->base + L.off_bt);
    p->oplog = reinterpret_cast<int*>(p->base + L.off_oplog);
    p->kv = p->base + L.off_kv;
    p->k_layer_bytes = L.k_layer;
    p->v_layer_bytes = L.v_layer;
    p->layer_stride = L.layer_stride;
    p->esize = elem_bytes(cfg->dtype);
    p->n_prefill = (p->num_sms + 1) / 2;
    p->n_decode = p->num_sms - p->n_prefill.load();
    // zero everything (K/V zero-filled: masked keys always read finite values)
    if (cudaMemsetAsync(mem, 0, L.total, st) != cudaSuccess) {
        delete p;
        cudaSetDevice(prev);
        return SEMIPD_ERR_CUDA;
    }
    const long long nbt = (long long)cfg->max_reqs * cfg->max_blocks_per_req;
    long long work = cfg->num_blocks > nbt ? cfg->num_blocks : nbt;
    int grid = (int)((work + 255) / 256);
    if (grid > 4 * p->num_sms) grid = 4 * p->num_sms;
    if (grid < 1) grid = 1;
    init_pool_kernel<<<grid, 256, 0, st>>>(p->st, p->free_stack, p->nblk, p->bt, cfg->num_blocks,
                                           cfg->max_reqs, nbt);
    p->launches += 1;
    if (cudaGetLastError() != cudaSuccess) {
        delete p;
        cudaSetDevice(prev);
        return SEMIPD_ERR_CUDA;
    }
    if (cfg->dtype == SEMIPD_FP8_E4M3 && !spd_fp8_init_maps(p)) {
        delete p;
        cudaSetDevice(prev);
        return SEMIPD_ERR_CUDA;
    }
    // TMA descriptors: bf16 pools with 64-multiple head dims (the tensor-core paths)
    if (cfg->dtype == SEMIPD_BF16 && cfg->head_dim_k % 64 == 0 && cfg->head_dim_v % 64 == 0) {
        // prefill prefix page boxes: min(bs, SPD_PREFIX_BOX_ROWS) rows x 64 columns (the TMA
        // unit's cost is per box, so the largest box a page allows)
#ifndef SPD_PREFIX_BOX_ROWS
#define SPD_PREFIX_BOX_ROWS 128
#endif
        p->box_rows = cfg->block_size < SPD_PREFIX_BOX_ROWS ? cfg->block_size : SPD_PREFIX_BOX_ROWS;
        const uint64_t pages = (uint64_t)cfg->num_blocks * cfg->num_kv_heads;
        p->kmap.resize(cfg->num_layers);
        p->vmap.resize(cfg->num_layers);
        p->dkmap.resize(cfg->num_layers);
        p->dvmap.resize(cfg->num_layers);
        p->dbox_rows = cfg->block_size < 64 ? cfg->block_size : 64;
        const bool pow2 = (cfg->block_size & (cfg->block_size - 1)) == 0;
        bool ok = true, dok = pow2 && cfg->block_size >= 16;
        for (int l = 0; l < cfg->num_layers && ok; ++l) {
            const uint64_t kr = (uint64_t)cfg->head_dim_k * 2;
            ok = spd_encode_tiled_3d(&p->kmap[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, p->k_layer(l),
                                     cfg->head_dim_k, cfg->block_size, pages, kr,
                                     kr * cfg->block_size, 64, p->box_rows, 1,
                                     CU_TENSOR_MAP_SWIZZLE_128B);
            const uint64_t vr = cfg->kv_shared ? kr : (uint64_t)cfg->head_dim_v * 2;
            ok = ok && spd_encode_tiled_3d(&p->vmap[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                           p->v_layer(l), cfg->head_dim_v, cfg->block_size, pages,
                                           vr, vr * cfg->block_size, 64, p->box_rows, 1,
                                           CU_TENSOR_MAP_SWIZZLE_128B);
            // decode: (64 cols, rows [row pitch], column blocks [128 B], pages [page pitch]);
            // box = min(bs, 64) rows x all column blocks of one page -> smem
            // [column block][rows][128 B] (conflict-free 128-byte swizzle per 8 rows)
            const uint64_t kd[4] = {64, (uint64_t)cfg->block_size, (uint64_t)cfg->head_dim_k / 64, pages};
            const uint64_t ks[3] = {kr, 128, kr * cfg->block_size};
            const uint32_t kb[4] = {64, (uint32_t)p->dbox_rows, (uint32_t)cfg->head_dim_k / 64, 1};
            bool okd = spd_encode_tiled_4d(&p->dkmap[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                           p->k_layer(l), kd, ks, kb, CU_TENSOR_MAP_SWIZZLE_128B);
            const uint64_t vd[4] = {64, (uint64_t)cfg->block_size, (uint64_t)cfg->head_dim_v / 64, pages};
            const uint64_t vs[3] = {vr, 128, vr * cfg->block_size};
            const uint32_t vb[4] = {64, (uint32_t)p->dbox_rows, (uint32_t)cfg->head_dim_v / 64, 1};
            okd = okd && spd_encode_tiled_4d(&p->dvmap[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                           p->v_layer(l), vd, vs, vb, CU_TENSOR_MAP_SWIZZLE_128B);
            dok = dok && okd;
        }
        p->have_dmaps = dok;
        const bool wide64 = cfg->block_size == 64 && cfg->num_kv_heads % 2 == 0;
        const bool wide128 = cfg->block_size == 128;
        const bool wide16 = cfg->block_size == 16 && cfg->num_kv_heads % 2 == 0;
        if (dok && (wide64 || wide128 || wide16) && cfg->head_dim_k == 128 && cfg->head_dim_v == 128 &&
            !cfg->kv_shared) {
            p->dkmap2.resize(cfg->num_layers);
            p->dvmap2.resize(cfg->num_layers);
            bool pok = true;
            for (int l = 0; l < cfg->num_layers && pok; ++l) {
                const uint64_t r = 256;
                const uint64_t dd[4] = {64, (uint64_t)cfg->block_size, 2, pages};
                const uint64_t ds[3] = {r, 128, r * cfg->block_size};
                // (64 cols, rows, 2 halves, pages): 64-token pages -> 64 rows x 2 adjacent
                // head pages; 128 -> one whole page; 16 -> 16 rows x 2 adjacent head pages
                const uint32_t db[4] = {64, wide64 ? 64u : wide16 ? 16u : 128u, 2,
                                        (wide64 || wide16) ? 2u : 1u};
                pok = spd_encode_tiled_4d(&p->dkmap2[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                          p->k_layer(l), dd, ds, db, CU_TENSOR_MAP_SWIZZLE_128B) &&
                      spd_encode_tiled_4d(&p->dvmap2[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                          p->v_layer(l), dd, ds, db, CU_TENSOR_MAP_SWIZZLE_128B);
            }
            p->have_wide_maps = pok;
            p->force_single = getenv("SEMIPD_DECODE_SINGLE") != nullptr;  // A/B debugging only
            p->force_pair = getenv("SEMIPD_DECODE_PAIR64") != nullptr;    // A/B debugging only
        }
        if (cfg->kv_shared && cfg->block_size % 32 == 0 && pow2) {
            p->mla_kmap.resize(cfg->num_layers);
            bool mok = true;
            for (int l = 0; l < cfg->num_layers && mok; ++l) {
                const uint64_t kr = (uint64_t)cfg->head_dim_k * 2;
                const uint64_t md[4] = {64, (uint64_t)cfg->block_size, (uint64_t)cfg->head_dim_k / 64,
                                        (uint64_t)cfg->num_blocks * cfg->num_kv_heads};
                const uint64_t ms[3] = {kr, 128, kr * cfg->block_size};
                const uint32_t mb[4] = {64, 32, (uint32_t)cfg->head_dim_k / 64, 1};
                mok = spd_encode_tiled_4d(&p->mla_kmap[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                          p->k_layer(l), md, ms, mb, CU_TENSOR_MAP_SWIZZLE_128B);
            }
            p->have_mla_map = mok;
            if (cfg->block_size == 64 && cfg->head_dim_k == 576 && cfg->num_kv_heads == 1) {
                p->mla_lo.resize(cfg->num_layers);
                p->mla_hi.resize(cfg->num_layers);
                bool tok = true;
                for (int l = 0; l < cfg->num_layers && tok; ++l) {
                    const uint64_t kr = (uint64_t)cfg->head_dim_k * 2;
                    const uint64_t md[4] = {64, 64, 9, (uint64_t)cfg->num_blocks};
                    const uint64_t ms[3] = {kr, 128, kr * 64};
                    const uint32_t lo[4] = {64, 64, 4, 1}, hi[4] = {64, 64, 5, 1};
                    tok = spd_encode_tiled_4d(&p->mla_lo[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                              p->k_layer(l), md, ms, lo, CU_TENSOR_MAP_SWIZZLE_128B) &&
                          spd_encode_tiled_4d(&p->mla_hi[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                              p->k_layer(l), md, ms, hi, CU_TENSOR_MAP_SWIZZLE_128B);
                }
                p->have_mla_tc_maps = tok;
            }
        }
        p->have_maps = ok;
    }
    cudaSetDevice(prev);
    *out = p;
    return SEMIPD_OK;
}

semipd_status semipd_kv_pool_destroy(semipd_pool_t pool) {
    if (!pool) return SEMIPD_ERR_INVALID;
    delete pool;
    return SEMIPD_OK;
}

semipd_status semipd_kv_pool_views(semipd_pool_t pool, int32_t layer, void** k, void** v,
                                   int32_t** block_tables, int32_t** nblk) {
    if (!pool || layer < 0 || layer >= pool->cfg.num_layers) return SEMIPD_ERR_INVALID;
    if (k) *k = pool->k_layer(layer);
    if (v) *v = pool->v_layer(layer);
    if (block_tables) *block_tables = pool->bt;
    if (nblk) *nblk = pool->nblk;
    return SEMIPD_OK;
}

semipd_status semipd_pool_stats(semipd_pool_t pool, int32_t* free_blocks, int32_t* min_free_seen,
                                semipd_stream_t s) {
    if (!pool) return SEMIPD_ERR_INVALID;
    int h[2];
    cudaStream_t st = static_cast<cudaStream_t>(s);
    if (cudaMemcpyAsync(h, &pool->st->top, sizeof(int) * 2, cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    if (free_blocks) *free_blocks = h[0];
    if (min_free_seen) *min_free_seen = h[1];
    return SEMIPD_OK;
}

semipd_status semipd_pool_oplog(semipd_pool_t pool, int32_t* host_buf, size_t bytes,
                                int64_t* n_words, int64_t* dropped, semipd_stream_t s) {
    if (!pool) return SEMIPD_ERR_INVALID;
    cudaStream_t st = static_cast<cudaStream_t>(s);
    long long hdr[2];
    if (cudaMemcpyAsync(hdr, &pool->st->oplog_len, sizeof(hdr), cudaMemcpyDeviceToHost, st) !=
            cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
        return SEMIPD_ERR_CUDA;
    if (n_words) *n_words = hdr[0];
    if (dropped) *dropped = hdr[1];
    size_t want = (size_t)hdr[0] * sizeof(int);
    if (host_buf && bytes) {
        size_t cp = want < bytes ? want : bytes;
        if (cp && (cudaMemcpyAsync(host_buf, pool->oplog, cp, cudaMemcpyDeviceToHost, st) !=
                       cudaSuccess ||
                   cudaStreamSynchronize(st) != cudaSuccess))
            return SEMIPD_ERR_CUDA;
    }
    return SEMIPD_OK;
}

semipd_status semipd_set_partition(semipd_pool_t pool, double x, double y) {
    if (!pool) return SEMIPD_ERR_INVALID;
    if (!(x > 0.0) || x > 100.0 || !(y > 0.0) || y > 100.0) return SEMIPD_ERR_INVALID;
    auto budget = [&](double pct) {
        int n = (int)std::floor((double)pool->num_sms * pct / 100.0 + 0.5);
        if (n < 1) n = 1;
        if (n > pool->num_sms) n = pool->num_sms;
        return n;
    };
    pool->n_prefill.store(budget(x));
    pool->n_decode.store(budget(y));
    pool->epoch.fetch_add(1);
    return SEMIPD_OK;
}

semipd_status semipd_get_sm_budgets(semipd_pool_t pool, int32_t* n_prefill, int32_t* n_decode) {
    if (!pool) return SEMIPD_ERR_INVALID;
    if (n_prefill) *n_prefill = pool->n_prefill.load();
    if (n_decode) *n_decode = pool->n_decode.load();
    return SEMIPD_OK;
}

int32_t semipd_num_sms(semipd_pool_t pool) { return pool ? pool->num_sms : -1; }

int64_t semipd_launch_count(semipd_pool_t pool) { return pool ? pool->launches.load() : -1; }

semipd_status semipd_set_trace(semipd_pool_t pool, int32_t* buf, int32_t cap, int32_t* counter_dev) {
    if (!pool) return SEMIPD_ERR_INVALID;
    if (buf && (cap <= 0 || !counter_dev)) return SEMIPD_ERR_INVALID;
    pool->trace_buf = buf;
    pool->trace_cap = buf ? cap : 0;
    pool->trace_ctr = buf ? counter_dev : nullptr;
    return SEMIPD_OK;
}

semipd_status semipd_set_spans(semipd_pool_t pool, uint64_t* buf, int32_t cap) {
    if (!pool || (buf && cap <= 0)) return SEMIPD_ERR_INVALID;
    pool->span_buf = reinterpret_cast<unsigned long long*>(buf);
    pool->span_cap = buf ? cap : 0;
    pool->span_next = 0;
    return SEMIPD_OK;
}

}  // extern "C"

#ifdef SPD_TIMELINE
// Debug builds only (not part of the ABI): prefill phase timeline of CTA 0.
extern "C" semipd_status semipd_debug_set_timeline(semipd_pool_t pool, void* buf, int32_t* ctr) {
    if (!pool) return SEMIPD_ERR_INVALID;
    pool->timeline = buf;
    pool->timeline_ctr = ctr;
    return SEMIPD_OK;
}
#endif

bool spd_pdl_enabled() {
    static const bool on = getenv("SEMIPD_NO_PDL") == nullptr;
    return on;
}

