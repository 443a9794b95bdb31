/*
 * semipd_oracle.c — plain, slow, obviously-correct CPU oracle for the semi-PD
 * co-run attention hot path (arXiv 2504.19867).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, constant or helper with the CUDA path under
 * paper_2504_19867_b200/ (and includes none of it).
 *
 * What it computes:
 *   - Exact scaled-dot-product attention, fp64, sums in key-index order.
 *     The paper never writes the formula; it cites the Transformer (§2.1),
 *     FlashAttention (§6) and PagedAttention (§4.4).
 *       z_j = s * sum_c q_c k_jc ;  M = max_j z_j ;  w_j = exp(z_j - M)
 *       o   = sum_j w_j v_j / sum_j w_j
 *   - KV written by prefill / appended by decode into the paged pool
 *     ("the generated K, V projection of the request is written into the KV
 *     cache", "at each decode iteration, the KV cache ... is updated", §4.2).
 *   - Paged access "through the block table index" (§4.4):
 *       key j of request r, kv head g = pool[bt[r][j / bs]][g][j % bs][:]
 *   - GQA (§6) with g(h) = floor(h / (Hq/Hkv))      (reading R3).
 *   - The atomic block allocator of P:229 §4.4 ("the memory utilization is
 *     locked until the update step finishes") as a SEQUENTIAL state machine:
 *     a linearizable concurrent allocator must equal it replayed in its
 *     linearisation order.
 *
 * Inputs arrive in their storage dtype (bf16 bit patterns or fp32) and are
 * converted exactly to fp64 on read.  Writes into the pool copy raw elements.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_BF16 0
#define ORC_FP32 1

/* Oracle status codes (restated, not shared). */
#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_OOM 2
#define ORC_UNKNOWN_REQ 3
#define ORC_TABLE_FULL 4
#define ORC_BAD_BLOCK 5

static size_t esize(int dtype) { return dtype == ORC_BF16 ? 2 : 4; }

/* Exact widening of one stored element to fp64. */
static double ld(const void* base, size_t idx, int dtype) {
    if (dtype == ORC_BF16) {
        uint16_t h = ((const uint16_t*)base)[idx];
        uint32_t u = ((uint32_t)h) << 16;
        float f;
        memcpy(&f, &u, 4);
        return (double)f;
    }
    return (double)((const float*)base)[idx];
}

static void copy_elem(void* dst, size_t di, const void* src, size_t si, int dtype) {
    size_t e = esize(dtype);
    memcpy((char*)dst + di * e, (const char*)src + si * e, e);
}

/* ---------------------------------------------------------------------------
 * One query row against n keys, plain definition (S1).  Keys/values are
 * addressed through index arrays so that contiguous and paged callers share
 * this single definition.
 *   q      : dk elements at q_base[q_off + c]
 *   key j  : k_base[k_off[j] + c]   (c < dk)
 *   val j  : v_base[v_off[j] + c]   (c < dv)
 * Output: o[dv] in fp64.  n == 0 leaves o = 0 (never called that way: a query
 * always sees at least itself, S4/S5).
 * ------------------------------------------------------------------------- */
static void attend_row(const void* q_base, size_t q_off, const void* k_base,
                       const size_t* k_off, const void* v_base, const size_t* v_off,
                       int n, int dk, int dv, double scale, int dtype, double* z,
                       double* o) {
    double M = -INFINITY;
    for (int j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int c = 0; c < dk; ++c)
            dot += ld(q_base, q_off + c, dtype) * ld(k_base, k_off[j] + c, dtype);
        z[j] = scale * dot;
        if (z[j] > M) M = z[j];
    }
    double denom = 0.0;
    for (int c = 0; c < dv; ++c) o[c] = 0.0;
    for (int j = 0; j < n; ++j) {
        double w = exp(z[j] - M);
        denom += w;
        for (int c = 0; c < dv; ++c) o[c] += w * ld(v_base, v_off[j] + c, dtype);
    }
    for (int c = 0; c < dv; ++c) o[c] /= denom;
}

/* ---------------------------------------------------------------------------
 * Contiguous attention (used by invariants: paged == contiguous).
 *   q [nq][Hq][dk], k [nk][Hkv][dk], v [nk][Hkv][dv], out [nq][Hq][dv] (fp64)
 *   row t sees keys j <= causal_offset + t  (causal_offset < 0 : all keys)
 * ------------------------------------------------------------------------- */
int semipd_ref_attention_contig(int nq, int nk, int Hq, int Hkv, int dk, int dv,
                                int dtype, const void* q, const void* k, const void* v,
                                int causal_offset, double scale, double* out) {
    if (nq < 0 || nk < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv) return ORC_INVALID;
    int G = Hq / Hkv;
    int fail = 0;
#pragma omp parallel
    {
        size_t* koff = (size_t*)malloc(sizeof(size_t) * (size_t)(nk > 0 ? nk : 1));
        size_t* voff = (size_t*)malloc(sizeof(size_t) * (size_t)(nk > 0 ? nk : 1));
        double* z = (double*)malloc(sizeof(double) * (size_t)(nk > 0 ? nk : 1));
#pragma omp for schedule(dynamic, 1) collapse(2)
        for (int t = 0; t < nq; ++t)
            for (int h = 0; h < Hq; ++h) {
                int g = h / G;
                int n = causal_offset < 0 ? nk : causal_offset + t + 1;
                if (n > nk) n = nk;
                if (n <= 0) {
#pragma omp atomic write
                    fail = 1;
                    continue;
                }
                for (int j = 0; j < n; ++j) {
                    koff[j] = ((size_t)j * Hkv + g) * dk;
                    voff[j] = ((size_t)j * Hkv + g) * dv;
                }
                attend_row(q, ((size_t)t * Hq + h) * dk, k, koff, v, voff, n, dk, dv,
                           scale, dtype, z, out + ((size_t)t * Hq + h) * dv);
            }
        free(koff);
        free(voff);
        free(z);
    }
    return fail ? ORC_INVALID : ORC_OK;
}

/* Paged-pool element offsets.  K pool [N_B][Hkv][bs][dk]; V pool
 * [N_B][Hkv][bs][dv]; for kv_shared (MLA latent, S19) V aliases the K rows:
 * value j = first dv elements of key row j. */
static size_t k_elem(int blk, int g, int slot, int Hkv, int bs, int dk) {
    return (((size_t)blk * Hkv + g) * bs + slot) * dk;
}

/* ---------------------------------------------------------------------------
 * Prefill (chunked, causal, GQA, paged prefix), P:184 + P:229 + P:355 + P:365.
 *   Request i (table row req_ids[i]) owns chunk rows cu[i] .. cu[i+1]-1; chunk
 *   row t sits at absolute position P_i + t (bottom-right causal alignment, S4).
 *   Step 1: k_new/v_new rows are written into pool slots P_i + t.
 *   Step 2: every (t, h) attends keys j in [0, P_i + t], all read from the pool
 *   through the block table (keys j < P_i were cached by earlier chunks).
 *   rows_mask (nullable, [T]) restricts step 2 to sampled rows (for full-size
 *   parity); step 1 always runs.  Rows not computed are left untouched in out.
 * Returns ORC_BAD_BLOCK if a needed table entry is outside [0, N_B).
 * ------------------------------------------------------------------------- */
int semipd_ref_prefill(int n_req, const int* cu_seqlens, const int* req_ids,
                       const int* prefix_lens, int Hq, int Hkv, int dk, int dv, int bs,
                       int kv_shared, int dtype, const void* q, const void* k_new,
                       const void* v_new, void* Kpool, void* Vpool, int N_B,
                       const int* block_tables, int MBR, double scale, double* out,
                       const unsigned char* rows_mask) {
    if (n_req < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || bs <= 0) return ORC_INVALID;
    if (kv_shared && dv > dk) return ORC_INVALID;
    int G = Hq / Hkv;
    /* step 1: KV write, bit-exact element copies */
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t) {
            int pos = prefix_lens[i] + (t - cu_seqlens[i]);
            if (pos / bs >= MBR) return ORC_BAD_BLOCK;
            int blk = bt[pos / bs];
            if (blk < 0 || blk >= N_B) return ORC_BAD_BLOCK;
            for (int g = 0; g < Hkv; ++g) {
                size_t ko = k_elem(blk, g, pos % bs, Hkv, bs, dk);
                for (int c = 0; c < dk; ++c)
                    copy_elem(Kpool, ko + c, k_new, ((size_t)t * Hkv + g) * dk + c, dtype);
                if (!kv_shared) {
                    size_t vo = k_elem(blk, g, pos % bs, Hkv, bs, dv);
                    for (int c = 0; c < dv; ++c)
                        copy_elem(Vpool, vo + c, v_new, ((size_t)t * Hkv + g) * dv + c,
                                  dtype);
                }
            }
        }
    }
    /* step 2: attention over the paged keys (every page it reads must be valid) */
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        int nk = prefix_lens[i] + cu_seqlens[i + 1] - cu_seqlens[i];
        for (int p = 0; p * bs < nk; ++p)
            if (p >= MBR || bt[p] < 0 || bt[p] >= N_B) return ORC_BAD_BLOCK;
    }
    int T = n_req > 0 ? cu_seqlens[n_req] : 0;
    int maxkeys = 1;
    for (int i = 0; i < n_req; ++i) {
        int nk = prefix_lens[i] + cu_seqlens[i + 1] - cu_seqlens[i];
        if (nk > maxkeys) maxkeys = nk;
    }
    int* row_req = (int*)malloc(sizeof(int) * (size_t)(T > 0 ? T : 1));
    for (int i = 0; i < n_req; ++i)
        for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t) row_req[t] = i;
    const void* vbase = kv_shared ? (const void*)Kpool : (const void*)Vpool;
#pragma omp parallel
    {
        size_t* koff = (size_t*)malloc(sizeof(size_t) * (size_t)maxkeys);
        size_t* voff = (size_t*)malloc(sizeof(size_t) * (size_t)maxkeys);
        double* z = (double*)malloc(sizeof(double) * (size_t)maxkeys);
#pragma omp for schedule(dynamic, 1) collapse(2)
        for (int t = 0; t < T; ++t)
            for (int h = 0; h < Hq; ++h) {
                if (rows_mask && !rows_mask[t]) continue;
                int i = row_req[t];
                int g = h / G;
                const int* bt = block_tables + (size_t)req_ids[i] * MBR;
                int n = prefix_lens[i] + (t - cu_seqlens[i]) + 1;
                for (int j = 0; j < n; ++j) {
                    int blk = bt[j / bs];
                    koff[j] = k_elem(blk, g, j % bs, Hkv, bs, dk);
                    voff[j] = kv_shared ? koff[j] : k_elem(blk, g, j % bs, Hkv, bs, dv);
                }
                attend_row(q, ((size_t)t * Hq + h) * dk, Kpool, koff, vbase, voff, n, dk,
                           dv, scale, dtype, z, out + ((size_t)t * Hq + h) * dv);
            }
        free(koff);
        free(voff);
        free(z);
    }
    free(row_req);
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Decode step (§2.1, §4.2, §4.4).  ctx_lens[b] = tokens cached
 * BEFORE the step (S5).  Step 1: k_new/v_new go to slot ctx.  Step 2: the new
 * query attends keys 0 .. ctx inclusive (ctx + 1 keys).
 *   q [B][Hq][dk], k_new [B][Hkv][dk], v_new [B][Hkv][dv], out [B][Hq][dv]
 * ------------------------------------------------------------------------- */
int semipd_ref_decode(int B, const int* req_ids, const int* ctx_lens, int Hq, int Hkv,
                      int dk, int dv, int bs, int kv_shared, int dtype, const void* q,
                      const void* k_new, const void* v_new, void* Kpool, void* Vpool,
                      int N_B, const int* block_tables, int MBR, double scale,
                      double* out) {
    if (B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || bs <= 0) return ORC_INVALID;
    if (kv_shared && dv > dk) return ORC_INVALID;
    int G = Hq / Hkv;
    int maxkeys = 1;
    for (int b = 0; b < B; ++b) {
        const int* bt = block_tables + (size_t)req_ids[b] * MBR;
        int pos = ctx_lens[b];
        if (pos < 0 || pos / bs >= MBR) return ORC_BAD_BLOCK;
        for (int p = 0; p <= pos / bs; ++p)
            if (bt[p] < 0 || bt[p] >= N_B) return ORC_BAD_BLOCK;
        int blk = bt[pos / bs];
        for (int g = 0; g < Hkv; ++g) {
            size_t ko = k_elem(blk, g, pos % bs, Hkv, bs, dk);
            for (int c = 0; c < dk; ++c)
                copy_elem(Kpool, ko + c, k_new, ((size_t)b * Hkv + g) * dk + c, dtype);
            if (!kv_shared) {
                size_t vo = k_elem(blk, g, pos % bs, Hkv, bs, dv);
                for (int c = 0; c < dv; ++c)
                    copy_elem(Vpool, vo + c, v_new, ((size_t)b * Hkv + g) * dv + c, dtype);
            }
        }
        if (pos + 1 > maxkeys) maxkeys = pos + 1;
    }
    const void* vbase = kv_shared ? (const void*)Kpool : (const void*)Vpool;
#pragma omp parallel
    {
        size_t* koff = (size_t*)malloc(sizeof(size_t) * (size_t)maxkeys);
        size_t* voff = (size_t*)malloc(sizeof(size_t) * (size_t)maxkeys);
        double* z = (double*)malloc(sizeof(double) * (size_t)maxkeys);
#pragma omp for schedule(dynamic, 1) collapse(2)
        for (int b = 0; b < B; ++b)
            for (int h = 0; h < Hq; ++h) {
                int g = h / G;
                const int* bt = block_tables + (size_t)req_ids[b] * MBR;
                int n = ctx_lens[b] + 1;
                for (int j = 0; j < n; ++j) {
                    int blk = bt[j / bs];
                    koff[j] = k_elem(blk, g, j % bs, Hkv, bs, dk);
                    voff[j] = kv_shared ? koff[j] : k_elem(blk, g, j % bs, Hkv, bs, dv);
                }
                attend_row(q, ((size_t)b * Hq + h) * dk, Kpool, koff, vbase, voff, n, dk,
                           dv, scale, dtype, z, out + ((size_t)b * Hq + h) * dv);
            }
        free(koff);
        free(voff);
        free(z);
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Split-K partial and merge (flash-decoding, cited P:127).  Used only by the
 * oracle's own invariant tests: merging the partials of ANY partition of the
 * keys must reproduce the unsplit row.
 *   partial over keys [j0, j1) of fp64 arrays k[n][dk], v[n][dv], q[dk]:
 *     m = max z_j ; l = sum exp(z_j - m) ; acc = sum exp(z_j - m) v_j
 *   merge of S partials: M = max m_s ;
 *     o = sum_s e^{m_s - M} acc_s / sum_s e^{m_s - M} l_s   (split-index order)
 * ------------------------------------------------------------------------- */
void semipd_ref_partial(const double* q, const double* k, const double* v, int j0, int j1,
                        int dk, int dv, double scale, double* m, double* l, double* acc) {
    double M = -INFINITY;
    for (int j = j0; j < j1; ++j) {
        double dot = 0.0;
        for (int c = 0; c < dk; ++c) dot += q[c] * k[(size_t)j * dk + c];
        if (scale * dot > M) M = scale * dot;
    }
    double L = 0.0;
    for (int c = 0; c < dv; ++c) acc[c] = 0.0;
    for (int j = j0; j < j1; ++j) {
        double dot = 0.0;
        for (int c = 0; c < dk; ++c) dot += q[c] * k[(size_t)j * dk + c];
        double w = exp(scale * dot - M);
        L += w;
        for (int c = 0; c < dv; ++c) acc[c] += w * v[(size_t)j * dv + c];
    }
    *m = M;
    *l = L;
}

void semipd_ref_merge(int S, int dv, const double* m, const double* l, const double* acc,
                      double* out) {
    double M = -INFINITY;
    for (int s = 0; s < S; ++s)
        if (m[s] > M) M = m[s];
    double L = 0.0;
    for (int c = 0; c < dv; ++c) out[c] = 0.0;
    for (int s = 0; s < S; ++s) {
        double w = exp(m[s] - M);
        L += w * l[s];
        for (int c = 0; c < dv; ++c) out[c] += w * acc[(size_t)s * dv + c];
    }
    for (int c = 0; c < dv; ++c) out[c] /= L;
}

/* ---------------------------------------------------------------------------
 * Block allocator, sequential model of the atomic allocator (§4.4;
 * SPEC S:234-251; readings R7-R12).
 *   state: free_stack[N_B], *top, bt[R][MBR] (-1 = empty), nblk[R], *min_free
 *   init : free_stack[i] = N_B-1-i, top = N_B  => first pops return 0,1,2,...
 *   alloc(ids[n], counts[n]):  checks in order
 *      INVALID    any id outside [0,R) or any count < 1   (0 blocks is a
 *                 contract violation)
 *      OOM        sum(counts) > top                      (normal outcome)
 *      TABLE_FULL any row would exceed MBR
 *      else for i in argument order, for c < counts[i]:
 *           bt[id_i][nblk[id_i]++] = free_stack[--top]
 *      min_free = min(min_free, top).  Any error: no state change (all or nothing).
 *   free(ids[n]):
 *      INVALID     id outside [0,R)
 *      UNKNOWN_REQ nblk[id] == 0 or id repeated in the call (double release,
 *                  S:250)
 *      else for each id in order, j = 0..nblk-1: free_stack[top++] = bt[id][j];
 *           row := -1, nblk := 0.
 *   n == 0 is a no-op returning OK (S27).
 * ------------------------------------------------------------------------- */
void semipd_ref_alloc_init(int N_B, int R, int MBR, int* free_stack, int* top, int* bt,
                           int* nblk, int* min_free) {
    for (int i = 0; i < N_B; ++i) free_stack[i] = N_B - 1 - i;
    *top = N_B;
    for (size_t i = 0; i < (size_t)R * MBR; ++i) bt[i] = -1;
    for (int r = 0; r < R; ++r) nblk[r] = 0;
    *min_free = N_B;
}

int semipd_ref_alloc(int N_B, int R, int MBR, int* free_stack, int* top, int* bt,
                     int* nblk, int* min_free, int n, const int* ids, const int* counts) {
    (void)N_B;
    if (n == 0) return ORC_OK;
    long long total = 0;
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= R || counts[i] < 1) return ORC_INVALID;
        total += counts[i];
    }
    if (total > *top) return ORC_OOM;
    for (int i = 0; i < n; ++i) {
        long long want = nblk[ids[i]];
        for (int k = 0; k < n; ++k)
            if (ids[k] == ids[i]) want += counts[k];
        if (want > MBR) return ORC_TABLE_FULL;
    }
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < counts[i]; ++c) {
            int id = ids[i];
            bt[(size_t)id * MBR + nblk[id]] = free_stack[--(*top)];
            nblk[id] += 1;
        }
    if (*top < *min_free) *min_free = *top;
    return ORC_OK;
}

int semipd_ref_free(int N_B, int R, int MBR, int* free_stack, int* top, int* bt, int* nblk,
                    int n, const int* ids) {
    (void)N_B;
    if (n == 0) return ORC_OK;
    for (int i = 0; i < n; ++i)
        if (ids[i] < 0 || ids[i] >= R) return ORC_INVALID;
    for (int i = 0; i < n; ++i) {
        if (nblk[ids[i]] == 0) return ORC_UNKNOWN_REQ;
        for (int k = 0; k < i; ++k)
            if (ids[k] == ids[i]) return ORC_UNKNOWN_REQ;
    }
    for (int i = 0; i < n; ++i) {
        int id = ids[i];
        for (int j = 0; j < nblk[id]; ++j) {
            free_stack[(*top)++] = bt[(size_t)id * MBR + j];
            bt[(size_t)id * MBR + j] = -1;
        }
        nblk[id] = 0;
    }
    return ORC_OK;
}

/* ---------------------------------------------------------------------------
 * Partition map (§4.3; DESIGN reading R14):
 *   n = clamp(floor(N * pct / 100 + 1/2), 1, N) for each phase independently
 *   (x + y > 100 is allowed: oversubscription).
 * effective_shares is SPEC's model view, reported, not enforced.
 * ------------------------------------------------------------------------- */
int semipd_ref_sm_budget(int num_sms, double pct) {
    if (!(pct > 0.0) || pct > 100.0 || num_sms <= 0) return -1;
    int n = (int)floor((double)num_sms * pct / 100.0 + 0.5);
    if (n < 1) n = 1;
    if (n > num_sms) n = num_sms;
    return n;
}

void semipd_ref_effective_shares(double x, double y, double* xe, double* ye) {
    if (x + y <= 100.0) {
        *xe = x;
        *ye = y;
    } else {
        *xe = 100.0 * x / (x + y);
        *ye = 100.0 * y / (x + y);
    }
}

int semipd_ref_blocks_for_tokens(int tokens, int bs) {
    if (tokens < 0 || bs <= 0) return -1;
    return (tokens + bs - 1) / bs;
}

/* ---- Rotary position embedding ----
 * PAPER P:355 §6: "To support the Llama3.1 series model, we also modify the RoPE kernel."
 * The paper gives no formula; reading R27 fixes it as RoFormer's rotation with
 * Llama's half-split pairing (i, i + d/2) and the Llama-3.1 frequency rescaling.
 *
 * semipd_ref_rope_inv_freq: the d/2 frequencies, step by step:
 *   f_i = theta^(-2i/d)                                    (RoFormer)
 *   if factor > 1 (Llama 3.1), with w_i = 2 pi / f_i:
 *     w_i < L0 / hf            -> f_i           (high frequencies kept)
 *     w_i > L0 / lf            -> f_i / factor  (low frequencies stretched)
 *     otherwise                -> (1 - a) f_i / factor + a f_i,  a = (L0 / w_i - lf) / (hf - lf) */
void semipd_ref_rope_inv_freq(int d, double theta, double factor, double lf, double hf, double L0,
                              double* out) {
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < d / 2; ++i) {
        double f = pow(theta, -2.0 * (double)i / (double)d);
        if (factor > 1.0) {
            double w = 2.0 * pi / f;
            if (w < L0 / hf) {
                /* unchanged */
            } else if (w > L0 / lf) {
                f = f / factor;
            } else {
                double a = (L0 / w - lf) / (hf - lf);
                f = (1.0 - a) * f / factor + a * f;
            }
        }
        out[i] = f;
    }
}

/* semipd_ref_rope: x [T][H][d] (stored dtype, widened exactly) -> out [T][H][d] fp64.
 * Columns outside [off, off + rd) are copied.  Pair i (i < rd/2) is (off + i, off + rd/2 + i)
 * (half-split) or (off + 2i, off + 2i + 1) (interleaved); with f = inv_freq(rd):
 *   phi = pos_t * f_i;  (x, y) -> (x cos phi - y sin phi, y cos phi + x sin phi). */
void semipd_ref_rope(int T, int H, int d, int off, int rd, int inter, const void* x, int dtype,
                     const int* pos, double theta, double factor, double lf, double hf, double L0,
                     double* out) {
    double* f = (double*)malloc(sizeof(double) * (size_t)(rd / 2));
    semipd_ref_rope_inv_freq(rd, theta, factor, lf, hf, L0, f);
    for (int t = 0; t < T; ++t)
        for (int h = 0; h < H; ++h) {
            size_t row = ((size_t)t * H + h) * d;
            for (int c = 0; c < d; ++c) out[row + c] = ld(x, row + c, dtype);
            for (int i = 0; i < rd / 2; ++i) {
                size_t ix = row + off + (inter ? 2 * i : i);
                size_t iy = row + off + (inter ? 2 * i + 1 : rd / 2 + i);
                double phi = (double)pos[t] * f[i];
                double x0 = ld(x, ix, dtype), x1 = ld(x, iy, dtype);
                out[ix] = x0 * cos(phi) - x1 * sin(phi);
                out[iy] = x1 * cos(phi) + x0 * sin(phi);
            }
        }
    free(f);
}

/* ---- FP8 (E4M3) KV pages (§7.1 "deployed ... with FP8 precision") ----
 * The paper names FP8 for DeepSeek-V3 and nothing more; reading R31 fixes the form:
 *   - a page element is one OCP FP8 E4M3 code (the "fn" variant GPUs implement): sign bit,
 *     4 exponent bits with bias 7, 3 mantissa bits; exponent 15 with mantissa 7 is NaN; no
 *     infinities; largest finite 448 = 1.75 * 2^8; subnormals m * 2^-9, m = 1..7.
 *   - write:  code = E4M3( fl32(x / s) ), x the bf16 input element, s > 0 the layer's fp32
 *     tensor scale (k_scale for K, v_scale for V), fl32 one IEEE single-precision division,
 *     E4M3 round-to-nearest-even onto the finite codes with saturation to +-448 ("satfinite").
 *   - read:   value = s * e4m3_value(code)  (exact in fp64).
 *   - attention reads every cached key / value through "read"; a prefill chunk's own keys and
 *     values (the rows it writes this step) enter at input precision (bf16), as the step's
 *     K / V projections are in hand before they are cached.  Decode attends the
 *     appended row as stored (it is read back from the pool, "the KV cache ... is
 *     updated" before attention).
 * ------------------------------------------------------------------------------------------ */

/* value of an E4M3 code, straight from the bit fields (NaN codes -> NaN) */
double semipd_ref_e4m3_value(int code) {
    int s = (code >> 7) & 1, e = (code >> 3) & 15, m = code & 7;
    double v;
    if (e == 15 && m == 7) return NAN;
    if (e == 0) v = (double)m * ldexp(1.0, -9);            /* subnormal: (m/8) * 2^(1-7) */
    else v = (1.0 + (double)m / 8.0) * ldexp(1.0, e - 7);  /* normal */
    return s ? -v : v;
}

/* round-to-nearest-even onto the 127 finite non-negative codes by exhaustive search (ties go
 * to the even code, i.e. the even mantissa); |x| beyond 448 lands on 448 (satfinite) */
int semipd_ref_e4m3_encode(float x) {
    if (isnan(x)) return 0x7F;
    int sign = signbit(x) ? 0x80 : 0;
    double a = fabs((double)x);
    int best = 0;
    double bd = INFINITY;
    for (int c = 0; c <= 0x7E; ++c) {
        double d = fabs(semipd_ref_e4m3_value(c) - a);
        if (d < bd || (d == bd && (c & 1) == 0)) {
            bd = d;
            best = c;
        }
    }
    return sign | best;
}

/* the write rule: bf16 element (bits) divided by s in fp32, then encoded */
static unsigned char quant_e4m3(uint16_t bf16_bits, float s) {
    uint32_t u = ((uint32_t)bf16_bits) << 16;
    float x;
    memcpy(&x, &u, 4);
    volatile float q = x / s; /* one IEEE fp32 division, not contracted or widened */
    return (unsigned char)semipd_ref_e4m3_encode(q);
}

/* bulk helpers for the tests: codes of n bf16 elements at scale s / values of n codes */
void semipd_ref_e4m3_quantize(int n, const uint16_t* x, float s, unsigned char* codes) {
    for (int i = 0; i < n; ++i) codes[i] = quant_e4m3(x[i], s);
}
void semipd_ref_e4m3_values(int n, const unsigned char* codes, double* out) {
    for (int i = 0; i < n; ++i) out[i] = semipd_ref_e4m3_value(codes[i]);
}

/* The attention definition over materialised fp64 rows (same formula as attend_row). */
static void attend_f64(const double* q, const double* k, const double* v, int n, int dk, int dv,
                       double scale, double* z, double* o) {
    double M = -INFINITY;
    for (int j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int c = 0; c < dk; ++c) dot += q[c] * k[(size_t)j * dk + c];
        z[j] = scale * dot;
        if (z[j] > M) M = z[j];
    }
    double denom = 0.0;
    for (int c = 0; c < dv; ++c) o[c] = 0.0;
    for (int j = 0; j < n; ++j) {
        double w = exp(z[j] - M);
        denom += w;
        for (int c = 0; c < dv; ++c) o[c] += w * v[(size_t)j * dv + c];
    }
    for (int c = 0; c < dv; ++c) o[c] /= denom;
}

/* Decode step on an E4M3 pool (bf16 q / k_new / v_new; pools of codes [N_B][Hkv][bs][d]).
 * Step 1: quantise k_new / v_new into slot ctx.  Step 2: attention over keys 0 .. ctx, every
 * key and value read back from the pool (value = scale * e4m3_value(code)). */
int semipd_ref_decode_fp8(int B, const int* req_ids, const int* ctx_lens, int Hq, int Hkv, int dk,
                          int dv, int bs, const uint16_t* q, const uint16_t* k_new,
                          const uint16_t* v_new, unsigned char* Kpool, unsigned char* Vpool,
                          int N_B, const int* block_tables, int MBR, float k_scale, float v_scale,
                          double scale, double* out) {
    if (B < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || bs <= 0 || !(k_scale > 0) || !(v_scale > 0))
        return ORC_INVALID;
    int G = Hq / Hkv;
    int maxkeys = 1;
    for (int b = 0; b < B; ++b) {
        const int* bt = block_tables + (size_t)req_ids[b] * MBR;
        int pos = ctx_lens[b];
        if (pos < 0 || pos / bs >= MBR) return ORC_BAD_BLOCK;
        for (int p = 0; p <= pos / bs; ++p)
            if (bt[p] < 0 || bt[p] >= N_B) return ORC_BAD_BLOCK;
        int blk = bt[pos / bs];
        for (int g = 0; g < Hkv; ++g) {
            for (int c = 0; c < dk; ++c)
                Kpool[k_elem(blk, g, pos % bs, Hkv, bs, dk) + c] =
                    quant_e4m3(k_new[((size_t)b * Hkv + g) * dk + c], k_scale);
            for (int c = 0; c < dv; ++c)
                Vpool[k_elem(blk, g, pos % bs, Hkv, bs, dv) + c] =
                    quant_e4m3(v_new[((size_t)b * Hkv + g) * dv + c], v_scale);
        }
        if (pos + 1 > maxkeys) maxkeys = pos + 1;
    }
#pragma omp parallel
    {
        double* qd = (double*)malloc(sizeof(double) * (size_t)dk);
        double* kd = (double*)malloc(sizeof(double) * (size_t)maxkeys * dk);
        double* vd = (double*)malloc(sizeof(double) * (size_t)maxkeys * dv);
        double* z = (double*)malloc(sizeof(double) * (size_t)maxkeys);
#pragma omp for schedule(dynamic, 1) collapse(2)
        for (int b = 0; b < B; ++b)
            for (int h = 0; h < Hq; ++h) {
                int g = h / G;
                const int* bt = block_tables + (size_t)req_ids[b] * MBR;
                int n = ctx_lens[b] + 1;
                for (int c = 0; c < dk; ++c) qd[c] = ld(q, ((size_t)b * Hq + h) * dk + c, ORC_BF16);
                for (int j = 0; j < n; ++j) {
                    int blk = bt[j / bs];
                    for (int c = 0; c < dk; ++c)
                        kd[(size_t)j * dk + c] =
                            (double)k_scale * semipd_ref_e4m3_value(Kpool[k_elem(blk, g, j % bs, Hkv, bs, dk) + c]);
                    for (int c = 0; c < dv; ++c)
                        vd[(size_t)j * dv + c] =
                            (double)v_scale * semipd_ref_e4m3_value(Vpool[k_elem(blk, g, j % bs, Hkv, bs, dv) + c]);
                }
                attend_f64(qd, kd, vd, n, dk, dv, scale, z, out + ((size_t)b * Hq + h) * dv);
            }
        free(qd);
        free(kd);
        free(vd);
        free(z);
    }
    return ORC_OK;
}

/* Chunked causal GQA prefill on an E4M3 pool.  Step 1: quantise the chunk rows into slots
 * P_i + t.  Step 2: row t of request i attends keys j in [0, P_i + t]: j < P_i read back from
 * the pool (cached by earlier chunks), j >= P_i the chunk's own bf16 rows k_new / v_new
 * [cu_i + j - P_i].  rows_mask as in semipd_ref_prefill. */
int semipd_ref_prefill_fp8(int n_req, const int* cu_seqlens, const int* req_ids,
                           const int* prefix_lens, int Hq, int Hkv, int dk, int dv, int bs,
                           const uint16_t* q, const uint16_t* k_new, const uint16_t* v_new,
                           unsigned char* Kpool, unsigned char* Vpool, int N_B,
                           const int* block_tables, int MBR, float k_scale, float v_scale,
                           double scale, double* out, const unsigned char* rows_mask) {
    if (n_req < 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv || bs <= 0 || !(k_scale > 0) ||
        !(v_scale > 0))
        return ORC_INVALID;
    int G = Hq / Hkv;
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        int nk = prefix_lens[i] + cu_seqlens[i + 1] - cu_seqlens[i];
        for (int p = 0; p * bs < nk; ++p)
            if (p >= MBR || bt[p] < 0 || bt[p] >= N_B) return ORC_BAD_BLOCK;
    }
    /* step 1: quantised K/V write */
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t) {
            int pos = prefix_lens[i] + (t - cu_seqlens[i]);
            int blk = bt[pos / bs];
            for (int g = 0; g < Hkv; ++g) {
                for (int c = 0; c < dk; ++c)
                    Kpool[k_elem(blk, g, pos % bs, Hkv, bs, dk) + c] =
                        quant_e4m3(k_new[((size_t)t * Hkv + g) * dk + c], k_scale);
                for (int c = 0; c < dv; ++c)
                    Vpool[k_elem(blk, g, pos % bs, Hkv, bs, dv) + c] =
                        quant_e4m3(v_new[((size_t)t * Hkv + g) * dv + c], v_scale);
            }
        }
    }
    /* step 2 */
    int T = n_req > 0 ? cu_seqlens[n_req] : 0;
    int maxkeys = 1;
    for (int i = 0; i < n_req; ++i) {
        int nk = prefix_lens[i] + cu_seqlens[i + 1] - cu_seqlens[i];
        if (nk > maxkeys) maxkeys = nk;
    }
    int* row_req = (int*)malloc(sizeof(int) * (size_t)(T > 0 ? T : 1));
    for (int i = 0; i < n_req; ++i)
        for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t) row_req[t] = i;
#pragma omp parallel
    {
        double* qd = (double*)malloc(sizeof(double) * (size_t)dk);
        double* kd = (double*)malloc(sizeof(double) * (size_t)maxkeys * dk);
        double* vd = (double*)malloc(sizeof(double) * (size_t)maxkeys * dv);
        double* z = (double*)malloc(sizeof(double) * (size_t)maxkeys);
#pragma omp for schedule(dynamic, 1) collapse(2)
        for (int t = 0; t < T; ++t)
            for (int h = 0; h < Hq; ++h) {
                if (rows_mask && !rows_mask[t]) continue;
                int i = row_req[t];
                int g = h / G;
                const int* bt = block_tables + (size_t)req_ids[i] * MBR;
                int P = prefix_lens[i];
                int n = P + (t - cu_seqlens[i]) + 1;
                for (int c = 0; c < dk; ++c) qd[c] = ld(q, ((size_t)t * Hq + h) * dk + c, ORC_BF16);
                for (int j = 0; j < n; ++j) {
                    if (j < P) {
                        int blk = bt[j / bs];
                        for (int c = 0; c < dk; ++c)
                            kd[(size_t)j * dk + c] = (double)k_scale *
                                semipd_ref_e4m3_value(Kpool[k_elem(blk, g, j % bs, Hkv, bs, dk) + c]);
                        for (int c = 0; c < dv; ++c)
                            vd[(size_t)j * dv + c] = (double)v_scale *
                                semipd_ref_e4m3_value(Vpool[k_elem(blk, g, j % bs, Hkv, bs, dv) + c]);
                    } else {
                        size_t r = (size_t)cu_seqlens[i] + (size_t)(j - P);
                        for (int c = 0; c < dk; ++c)
                            kd[(size_t)j * dk + c] = ld(k_new, (r * Hkv + g) * dk + c, ORC_BF16);
                        for (int c = 0; c < dv; ++c)
                            vd[(size_t)j * dv + c] = ld(v_new, (r * Hkv + g) * dv + c, ORC_BF16);
                    }
                }
                attend_f64(qd, kd, vd, n, dk, dv, scale, z, out + ((size_t)t * Hq + h) * dv);
            }
        free(qd);
        free(kd);
        free(vd);
        free(z);
    }
    free(row_req);
    return ORC_OK;
}

/* ---- Expanded-form MLA prefill (reading R32) ----
 * DeepSeek MLA caches per token one latent row [c (dc = 512) | k_pe (dr = 64)] (the pool's
 * kv_shared rows, dk = 576).  The absorbed form (semipd_ref_prefill with kv_shared) attends
 * over the latent directly; the expanded form first projects every key's latent to per-head
 * keys and values with the up-projections W_UK, W_UV (h < H, rows d < dn / dv, columns c < dc):
 *   k_nope[j][h][d] = bf16( sum_c W_UK[h][d][c] * c_j[c] )   (fp64 sum, one RNE to bf16)
 *   v     [j][h][d] = bf16( sum_c W_UV[h][d][c] * c_j[c] )
 *   K[j][h] = [k_nope[j][h] | k_pe_j]  (dn + dr dims),  V[j][h] = v[j][h]  (dv dims)
 * and runs plain causal MHA per head with q [T][H][dn + dr] (q_nope | q_pe):
 *   o[t][h] = sum_{j <= P_i + t} softmax_j(scale * q[t][h] . K[j][h]) V[j][h].
 * The bf16 rounding of the projected K / V is R32's reading (they are activations, the
 * projection GEMM's output dtype).  Step 1 copies the chunk's latent rows into the
 * pool first, so every key's latent is read from the pool through the block table. */
/* one round-to-nearest-even of a double onto bf16 (8 significant bits, fp32's exponent range,
 * subnormal spacing 2^-133), straight from the definition */
static double round_bf16(double x) {
    if (x == 0.0 || !isfinite(x)) return x;
    int e;
    frexp(x, &e); /* |x| = m * 2^e, m in [0.5, 1) */
    double ulp = ldexp(1.0, e - 8 > -133 ? e - 8 : -133);
    return rint(x / ulp) * ulp;
}
double semipd_ref_round_bf16(double x) { return round_bf16(x); }

int semipd_ref_prefill_mla_expanded(int n_req, const int* cu_seqlens, const int* req_ids,
                                    const int* prefix_lens, int H, int dn, int dr, int dv, int dc,
                                    int bs, const uint16_t* q, const uint16_t* kv_new,
                                    uint16_t* pool, int N_B, const int* block_tables, int MBR,
                                    const uint16_t* w_uk, const uint16_t* w_uv, double scale,
                                    double* out, const unsigned char* rows_mask) {
    const int dl = dc + dr; /* latent row width */
    if (n_req < 0 || H <= 0 || dn <= 0 || dr < 0 || dv <= 0 || dc <= 0 || bs <= 0) return ORC_INVALID;
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        int nk = prefix_lens[i] + cu_seqlens[i + 1] - cu_seqlens[i];
        for (int p = 0; p * bs < nk; ++p)
            if (p >= MBR || bt[p] < 0 || bt[p] >= N_B) return ORC_BAD_BLOCK;
    }
    /* step 1: latent rows of the chunk into the pool (element copies) */
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t) {
            int pos = prefix_lens[i] + (t - cu_seqlens[i]);
            size_t dst = ((size_t)bt[pos / bs] * bs + pos % bs) * dl;
            for (int c = 0; c < dl; ++c) pool[dst + c] = kv_new[(size_t)t * dl + c];
        }
    }
    int T = n_req > 0 ? cu_seqlens[n_req] : 0;
    for (int i = 0; i < n_req; ++i) {
        const int* bt = block_tables + (size_t)req_ids[i] * MBR;
        int P = prefix_lens[i], C = cu_seqlens[i + 1] - cu_seqlens[i], nk = P + C;
        /* step 2: expanded keys / values of this request (bf16-rounded projections) */
        double* K = (double*)malloc(sizeof(double) * (size_t)nk * H * (dn + dr));
        double* V = (double*)malloc(sizeof(double) * (size_t)nk * H * dv);
#pragma omp parallel for schedule(dynamic, 4)
        for (int j = 0; j < nk; ++j) {
            const uint16_t* lat = pool + ((size_t)bt[j / bs] * bs + j % bs) * dl;
            for (int h = 0; h < H; ++h) {
                for (int d = 0; d < dn; ++d) {
                    double acc = 0.0;
                    for (int c = 0; c < dc; ++c)
                        acc += ld(w_uk, ((size_t)h * dn + d) * dc + c, ORC_BF16) * ld(lat, c, ORC_BF16);
                    K[((size_t)j * H + h) * (dn + dr) + d] = round_bf16(acc);
                }
                for (int d = 0; d < dr; ++d)
                    K[((size_t)j * H + h) * (dn + dr) + dn + d] = ld(lat, dc + d, ORC_BF16);
                for (int d = 0; d < dv; ++d) {
                    double acc = 0.0;
                    for (int c = 0; c < dc; ++c)
                        acc += ld(w_uv, ((size_t)h * dv + d) * dc + c, ORC_BF16) * ld(lat, c, ORC_BF16);
                    V[((size_t)j * H + h) * dv + d] = round_bf16(acc);
                }
            }
        }
        /* step 3: causal MHA per head */
#pragma omp parallel
        {
            double* qd = (double*)malloc(sizeof(double) * (size_t)(dn + dr));
            double* kh = (double*)malloc(sizeof(double) * (size_t)nk * (dn + dr));
            double* vh = (double*)malloc(sizeof(double) * (size_t)nk * dv);
            double* z = (double*)malloc(sizeof(double) * (size_t)nk);
#pragma omp for schedule(dynamic, 1) collapse(2)
            for (int t = cu_seqlens[i]; t < cu_seqlens[i + 1]; ++t)
                for (int h = 0; h < H; ++h) {
                    if (rows_mask && !rows_mask[t]) continue;
                    int n = P + (t - cu_seqlens[i]) + 1;
                    for (int c = 0; c < dn + dr; ++c) qd[c] = ld(q, ((size_t)t * H + h) * (dn + dr) + c, ORC_BF16);
                    for (int j = 0; j < n; ++j) {
                        for (int c = 0; c < dn + dr; ++c) kh[(size_t)j * (dn + dr) + c] = K[((size_t)j * H + h) * (dn + dr) + c];
                        for (int c = 0; c < dv; ++c) vh[(size_t)j * dv + c] = V[((size_t)j * H + h) * dv + c];
                    }
                    attend_f64(qd, kh, vh, n, dn + dr, dv, scale, z, out + ((size_t)t * H + h) * dv);
                }
            free(qd);
            free(kh);
            free(vh);
            free(z);
        }
        free(K);
        free(V);
    }
    (void)T;
    return ORC_OK;
}
