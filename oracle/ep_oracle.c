/*
 * ep_oracle.c — plain-C99 restatement of the reference spliced-attention path.
 *
 * TEST INFRASTRUCTURE ONLY (see ep_oracle.h). Each function cites the
 * reference routine it restates; citations are into
 * /root/reference/proj/core/src. The arithmetic order (max-shifted two-pass
 * softmax per segment, then a log-add-exp fold in segment order) follows the
 * reference so the fp64 results agree to rounding.
 */
#define _GNU_SOURCE
#include "ep_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

static const double kNegInf = -INFINITY;

/* matrix.cpp:88-93 — -inf is the identity; otherwise shift by the max. */
double epo_log_add_exp(double a, double b) {
    if (isinf(a) && a < 0) return b;
    if (isinf(b) && b < 0) return a;
    double m = a > b ? a : b;
    return m + log(exp(a - m) + exp(b - m));
}

/* attention.cpp:29-33 — keys are a contiguous run from k_off; a query at
 * absolute position p sees keys at positions <= p, i.e. always a prefix. */
size_t epo_visible_keys(size_t q_off, size_t k_off, size_t n_keys, size_t i) {
    size_t qpos = q_off + i;
    if (qpos < k_off) return 0;
    size_t vis = qpos - k_off + 1;
    return vis < n_keys ? vis : n_keys;
}

/* One query row against the visible prefix of one segment: pass 1 scores and
 * max, pass 2 exp-weights, value accumulation, normalisation and lse
 * (attention.cpp:89-111). scratch holds >= vis doubles. */
static void partial_row(const double* qi, const double* k, size_t ldk, const double* v,
                        size_t ldv, size_t vis, size_t d, double scale, double* scratch,
                        double* oi, double* lse_i) {
    double m = kNegInf;
    for (size_t j = 0; j < vis; ++j) {
        const double* kj = k + j * ldk;
        double dot = 0.0;
        for (size_t c = 0; c < d; ++c) dot += qi[c] * kj[c];
        scratch[j] = dot * scale;
        if (scratch[j] > m) m = scratch[j];
    }
    double denom = 0.0;
    for (size_t c = 0; c < d; ++c) oi[c] = 0.0;
    for (size_t j = 0; j < vis; ++j) {
        double w = exp(scratch[j] - m);
        denom += w;
        const double* vj = v + j * ldv;
        for (size_t c = 0; c < d; ++c) oi[c] += w * vj[c];
    }
    double inv = 1.0 / denom;
    for (size_t c = 0; c < d; ++c) oi[c] *= inv;
    *lse_i = m + log(denom);
}

/* attention.cpp:80-114 */
int epo_partial_attention(const double* q, size_t ldq, size_t n_q, const double* k,
                          size_t ldk, const double* v, size_t ldv, size_t n_keys, size_t d,
                          size_t q_off, size_t k_off, double* out, double* lse) {
    if (d == 0) return EPO_EINVAL;
    double scale = 1.0 / sqrt((double)d);
    double* scratch = (double*)malloc((n_keys ? n_keys : 1) * sizeof(double));
    if (!scratch) return EPO_EINVAL;
    for (size_t i = 0; i < n_q; ++i) {
        size_t vis = epo_visible_keys(q_off, k_off, n_keys, i);
        double* oi = out + i * d;
        if (vis == 0) { /* identity row (attention.cpp:91) */
            for (size_t c = 0; c < d; ++c) oi[c] = 0.0;
            lse[i] = kNegInf;
            continue;
        }
        partial_row(q + i * ldq, k, ldk, v, ldv, vis, d, scale, scratch, oi, &lse[i]);
    }
    free(scratch);
    return EPO_OK;
}

/* attention.cpp:45-78 — same arithmetic without the lse; a row with no
 * visible key is a domain error (attention.cpp:52-56). */
int epo_full_attention(const double* q, size_t n_q, const double* k, const double* v,
                       size_t n_keys, size_t d, size_t q_off, size_t k_off, double* out) {
    if (d == 0) return EPO_EINVAL;
    for (size_t i = 0; i < n_q; ++i)
        if (epo_visible_keys(q_off, k_off, n_keys, i) == 0) return EPO_EMASKED;
    double* lse = (double*)malloc((n_q ? n_q : 1) * sizeof(double));
    int rc = epo_partial_attention(q, d, n_q, k, d, v, d, n_keys, d, q_off, k_off, out, lse);
    free(lse);
    return rc;
}

/* attention.cpp:116-145 — fold lse with log_add_exp in part order, then
 * out = sum_p exp(lse_p - total) * out_p, skipping zero weights. */
int epo_merge_partials(size_t n_parts, const double* const* outs, const double* const* lses,
                       size_t n_q, size_t d, double* out, double* lse) {
    if (n_parts == 0) return EPO_EINVAL;
    for (size_t i = 0; i < n_q; ++i) {
        double total = kNegInf;
        for (size_t p = 0; p < n_parts; ++p) total = epo_log_add_exp(total, lses[p][i]);
        lse[i] = total;
        double* oi = out + i * d;
        for (size_t c = 0; c < d; ++c) oi[c] = 0.0;
        if (isinf(total) && total < 0) continue;
        for (size_t p = 0; p < n_parts; ++p) {
            double alpha = exp(lses[p][i] - total);
            if (alpha == 0.0) continue;
            const double* pi = outs[p] + i * d;
            for (size_t c = 0; c < d; ++c) oi[c] += alpha * pi[c];
        }
    }
    return EPO_OK;
}

/* attention.cpp:147-156 */
int epo_fuse_partials(size_t n_parts, const double* const* outs, const double* const* lses,
                      size_t n_q, size_t d, double* out) {
    double* lse = (double*)malloc((n_q ? n_q : 1) * sizeof(double));
    int rc = epo_merge_partials(n_parts, outs, lses, n_q, d, out, lse);
    if (rc == EPO_OK) {
        for (size_t i = 0; i < n_q; ++i)
            if (isinf(lse[i]) && lse[i] < 0) { rc = EPO_EMASKED; break; }
    }
    free(lse);
    return rc;
}

/* model.cpp:248-255 */
uint32_t epo_argmax(const double* logits, size_t n) {
    size_t best = 0;
    for (size_t i = 1; i < n; ++i)
        if (logits[i] > logits[best]) best = i;
    return (uint32_t)best;
}

/* model.cpp:131-150 */
void epo_layer_norm_row(const double* x, size_t n, double* out) {
    double mean = 0.0;
    for (size_t c = 0; c < n; ++c) mean += x[c];
    mean /= (double)n;
    double var = 0.0;
    for (size_t c = 0; c < n; ++c) {
        double dx = x[c] - mean;
        var += dx * dx;
    }
    var /= (double)n;
    double inv = 1.0 / sqrt(var + 1e-5);
    for (size_t c = 0; c < n; ++c) out[c] = (x[c] - mean) * inv;
}

/* ------------------------------------------------------------------------ */
/* Dtype helpers                                                             */
/* ------------------------------------------------------------------------ */

static inline double bf16_to_f64(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

static inline uint16_t f32_to_bf16_rn(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)((u >> 16) | ((u & 0xffff) ? 0x40 : 0));
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7fffu + lsb;
    return (uint16_t)(u >> 16);
}

static inline double load_elem(int dtype, const void* base, size_t idx) {
    switch (dtype) {
    case EPO_DT_BF16: return bf16_to_f64(((const uint16_t*)base)[idx]);
    case EPO_DT_F32: return (double)((const float*)base)[idx];
    default: return ((const double*)base)[idx];
    }
}

/* rng.hpp:15-27 evaluated at draw index i: the state after i+1 increments is
 * seed + (i+1) * golden (mod 2^64), so draws are independent of each other. */
static inline uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

void epo_fill_uniform(int dtype, void* dst, size_t n, uint64_t seed, double lo, double hi) {
    for (size_t i = 0; i < n; ++i) {
        double u = (double)(splitmix_at(seed, i) >> 11) * 0x1.0p-53;
        double x = lo + (hi - lo) * u;
        switch (dtype) {
        case EPO_DT_BF16: ((uint16_t*)dst)[i] = f32_to_bf16_rn((float)x); break;
        case EPO_DT_F32: ((float*)dst)[i] = (float)x; break;
        default: ((double*)dst)[i] = x; break;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Batched spliced attention                                                 */
/* ------------------------------------------------------------------------ */

typedef struct {
    const epo_splice_batch* s;
    const int64_t* units;
    int64_t n_units;
    int64_t next; /* guarded by mu */
    pthread_mutex_t mu;
    double* out;
    double* lse;
    int rc;
} unit_pool;

/* One (request, q-head) unit = the per-head body of transformer_layer's
 * attention block (model.cpp:168-181): a partial per visible segment with
 * CausalSpan{query_offset, seg.pos_offset}, then fuse in segment order.
 * Segment K/V are gathered from pages into a contiguous fp64 copy, like the
 * reference's per-head col_slice copies (model.cpp:171-173). */
static int run_unit(const epo_splice_batch* s, int64_t unit, double* out, double* lse) {
    const int Hq = s->n_q_heads, Hkv = s->n_kv_heads, d = s->d_head, P = s->page_tokens;
    const int group = Hq / Hkv;
    const int64_t b = unit / Hq;
    const int h = (int)(unit % Hq), g = h / group;
    const int n_q = s->n_q;
    const int64_t s0 = s->seg_indptr[b], s1 = s->seg_indptr[b + 1];
    const int64_t n_seg = s1 - s0;
    if (n_seg <= 0) return EPO_EINVAL;

    double* q = (double*)malloc((size_t)n_q * d * sizeof(double));
    double** outs = (double**)calloc((size_t)n_seg, sizeof(double*));
    double** lses = (double**)calloc((size_t)n_seg, sizeof(double*));
    int rc = EPO_OK;
    for (int i = 0; i < n_q; ++i)
        for (int c = 0; c < d; ++c)
            q[(size_t)i * d + c] =
                load_elem(s->q_dtype, s->q, (((size_t)b * n_q + i) * Hq + h) * d + c);

    for (int64_t si = 0; si < n_seg && rc == EPO_OK; ++si) {
        const epo_segment* seg = &s->segs[s0 + si];
        size_t n = (size_t)seg->len;
        double* kb = (double*)malloc((n ? n : 1) * d * sizeof(double));
        double* vb = (double*)malloc((n ? n : 1) * d * sizeof(double));
        for (size_t t = 0; t < n; ++t) {
            int64_t page = s->page_table[seg->page_off + (int64_t)(t / P)];
            size_t slot = t % P;
            size_t base = (((size_t)page * Hkv + g) * P + slot) * d;
            for (int c = 0; c < d; ++c) {
                kb[t * d + c] = load_elem(s->kv_dtype, s->k_pages, base + c);
                vb[t * d + c] = load_elem(s->kv_dtype, s->v_pages, base + c);
            }
        }
        outs[si] = (double*)malloc((size_t)n_q * d * sizeof(double));
        lses[si] = (double*)malloc((size_t)n_q * sizeof(double));
        rc = epo_partial_attention(q, d, n_q, kb, d, vb, d, n, d, (size_t)s->q_pos[b],
                                   (size_t)seg->pos_offset, outs[si], lses[si]);
        free(kb);
        free(vb);
    }
    if (rc == EPO_OK) {
        double* mo = (double*)malloc((size_t)n_q * d * sizeof(double));
        double* ml = (double*)malloc((size_t)n_q * sizeof(double));
        rc = epo_merge_partials((size_t)n_seg, (const double* const*)outs,
                                (const double* const*)lses, n_q, d, mo, ml);
        for (int i = 0; i < n_q; ++i) {
            size_t row = ((size_t)b * n_q + i) * Hq + h;
            memcpy(out + row * d, mo + (size_t)i * d, d * sizeof(double));
            lse[row] = ml[i];
        }
        free(mo);
        free(ml);
    }
    for (int64_t si = 0; si < n_seg; ++si) {
        free(outs[si]);
        free(lses[si]);
    }
    free(outs);
    free(lses);
    free(q);
    return rc;
}

static void* unit_worker(void* arg) {
    unit_pool* pool = (unit_pool*)arg;
    for (;;) {
        pthread_mutex_lock(&pool->mu);
        int64_t i = pool->next++;
        pthread_mutex_unlock(&pool->mu);
        if (i >= pool->n_units) break;
        int64_t unit = pool->units ? pool->units[i] : i;
        int rc = run_unit(pool->s, unit, pool->out, pool->lse);
        if (rc != EPO_OK) pool->rc = rc;
    }
    return NULL;
}

int epo_spliced_attention(const epo_splice_batch* s, int n_threads, const int64_t* unit_list,
                          int64_t n_units, double* out, double* lse) {
    if (!s || s->n_kv_heads <= 0 || s->n_q_heads % s->n_kv_heads != 0 || s->d_head <= 0 ||
        s->page_tokens <= 0 || s->n_q <= 0)
        return EPO_EINVAL;
    unit_pool pool;
    pool.s = s;
    pool.units = unit_list;
    pool.n_units = unit_list ? n_units : (int64_t)s->batch * s->n_q_heads;
    pool.next = 0;
    pool.out = out;
    pool.lse = lse;
    pool.rc = EPO_OK;
    pthread_mutex_init(&pool.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int t = 0; t < n_threads; ++t) pthread_create(&th[t], NULL, unit_worker, &pool);
    for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&pool.mu);
    return pool.rc;
}

/* Verify: per row, LN then @ w_score (unembed_logits, model.cpp:238-246),
 * greedy argmax (model.cpp:248-255); accept the longest draft prefix that the
 * target reproduces. */
int epo_verify_greedy(const double* attn_out, int batch, int n_q, int width,
                      const double* w_score, int vocab, const int32_t* drafts,
                      int32_t* target_ids, int32_t* n_accepted, double* top2_gap) {
    if (batch < 0 || n_q < 1 || width < 1 || vocab < 1) return EPO_EINVAL;
    double* normed = (double*)malloc((size_t)width * sizeof(double));
    double* logits = (double*)malloc((size_t)vocab * sizeof(double));
    const int k = n_q - 1;
    for (int b = 0; b < batch; ++b) {
        for (int r = 0; r < n_q; ++r) {
            const double* row = attn_out + ((size_t)b * n_q + r) * width;
            epo_layer_norm_row(row, (size_t)width, normed);
            for (int t = 0; t < vocab; ++t) logits[t] = 0.0;
            for (int c = 0; c < width; ++c) {
                const double a = normed[c];
                if (a == 0.0) continue;
                const double* wr = w_score + (size_t)c * vocab;
                for (int t = 0; t < vocab; ++t) logits[t] += a * wr[t];
            }
            uint32_t best = epo_argmax(logits, (size_t)vocab);
            target_ids[(size_t)b * n_q + r] = (int32_t)best;
            if (top2_gap) {
                double second = -INFINITY;
                for (int t = 0; t < vocab; ++t)
                    if ((uint32_t)t != best && logits[t] > second) second = logits[t];
                top2_gap[(size_t)b * n_q + r] = logits[best] - second;
            }
        }
        int n = 0;
        while (n < k && drafts[(size_t)b * k + n] == target_ids[(size_t)b * n_q + n]) ++n;
        n_accepted[b] = n;
    }
    free(normed);
    free(logits);
    return EPO_OK;
}

/* ------------------------------------------------------------------------ */
/* KV ingest (wire.cpp:119-221, edge.cpp:61-67)                              */
/* ------------------------------------------------------------------------ */

static uint32_t rd_u32(const uint8_t* b) {
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}
static uint16_t rd_u16(const uint8_t* b) { return (uint16_t)(b[0] | (b[1] << 8)); }
static double rd_f64(const uint8_t* b) {
    uint64_t bits = 0;
    double d;
    for (int i = 0; i < 8; ++i) bits |= (uint64_t)b[i] << (8 * i);
    memcpy(&d, &bits, 8);
    return d;
}

int epo_kv_frame_decode(const uint8_t* frame, size_t n, epo_kv_frame_info* info, double* k,
                        double* v) {
    /* decode_header (wire.cpp:138-162) */
    if (n < 10) return EPO_WIRE_TRUNCATED;
    if (frame[0] != 'E' || frame[1] != 'P' || frame[2] != 'K' || frame[3] != 'V') return EPO_WIRE_BAD_MAGIC;
    if (frame[4] != 0x01) return EPO_WIRE_BAD_VERSION;
    if (frame[5] > 4) return EPO_WIRE_MALFORMED;
    const uint32_t len = rd_u32(frame + 6);
    if (len > (1u << 30)) return EPO_WIRE_LENGTH_OVERFLOW;
    /* decode_frame (wire.cpp:209-219): exactly one frame */
    if (n != 10 + (size_t)len) return EPO_WIRE_TRUNCATED;
    /* decode_payload of the other message types (wire.cpp:165-184, :202-208):
     * short payloads are truncated reads, trailing bytes are malformed */
    switch (frame[5]) {
    case 0: return len < 20 ? EPO_WIRE_TRUNCATED : len > 20 ? EPO_WIRE_MALFORMED : EPO_WIRE_NOT_KV;
    case 1: return len < 6 ? EPO_WIRE_TRUNCATED : len > 6 ? EPO_WIRE_MALFORMED : EPO_WIRE_NOT_KV;
    case 3: return len != 0 ? EPO_WIRE_MALFORMED : EPO_WIRE_NOT_KV;
    case 4: return len < 4 ? EPO_WIRE_TRUNCATED : EPO_WIRE_NOT_KV;
    default: break;
    }
    /* decode_payload, kv_frame (wire.cpp:185-201) */
    const uint8_t* p = frame + 10;
    if (len < 14) return EPO_WIRE_TRUNCATED;
    epo_kv_frame_info f;
    f.session_id = rd_u32(p);
    f.layer = rd_u16(p + 4);
    f.seq_len = rd_u32(p + 6);
    f.n_heads = rd_u16(p + 10);
    f.d_head = rd_u16(p + 12);
    f.pad = 0;
    const uint64_t vals = (uint64_t)f.seq_len * f.n_heads * f.d_head;
    if ((uint64_t)(len - 14) != 16 * vals) return EPO_WIRE_MALFORMED;
    if (info) *info = f;
    if (k)
        for (uint64_t i = 0; i < vals; ++i) k[i] = rd_f64(p + 14 + 8 * i);
    if (v)
        for (uint64_t i = 0; i < vals; ++i) v[i] = rd_f64(p + 14 + 8 * (vals + i));
    return EPO_WIRE_OK;
}

float epo_f64_to_f32(double x) { return (float)x; }

/* Correct RNE f64 -> bf16: f64 -> f32 rounded to ODD, then f32 -> bf16 RNE
 * (round-to-odd keeps 16 > 2 guard bits, so the double rounding is exact). */
uint16_t epo_f64_to_bf16(double x) {
    if (x != x) return 0x7FC0;
    float f = (float)x; /* RN */
    if (fabs((double)f) > fabs(x)) f = nextafterf(f, 0.0f); /* -> toward zero */
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((double)f != x) u |= 1u; /* inexact: set the sticky (odd) bit */
    if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)(u >> 16); /* inf */
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}

int epo_kv_ingest(const uint8_t* frame, size_t n, int kv_dtype, int page_tokens,
                  const int32_t* page_table, void* k_pages, void* v_pages, epo_kv_frame_info* info) {
    epo_kv_frame_info f;
    int rc = epo_kv_frame_decode(frame, n, &f, NULL, NULL);
    if (rc) return rc;
    if (info) *info = f;
    const size_t H = f.n_heads, d = f.d_head, row = H * d;
    const uint8_t* kd = frame + 24;
    const uint8_t* vd = kd + 8 * (size_t)f.seq_len * row;
    for (size_t t = 0; t < f.seq_len; ++t) {
        const size_t page = (size_t)page_table[t / (size_t)page_tokens], slot = t % (size_t)page_tokens;
        for (size_t h = 0; h < H; ++h)
            for (size_t c = 0; c < d; ++c) {
                const size_t src = t * row + h * d + c;
                const size_t dst = ((page * H + h) * (size_t)page_tokens + slot) * d + c;
                const double a = rd_f64(kd + 8 * src), b = rd_f64(vd + 8 * src);
                if (kv_dtype == EPO_DT_BF16) {
                    ((uint16_t*)k_pages)[dst] = epo_f64_to_bf16(a);
                    ((uint16_t*)v_pages)[dst] = epo_f64_to_bf16(b);
                } else {
                    ((float*)k_pages)[dst] = epo_f64_to_f32(a);
                    ((float*)v_pages)[dst] = epo_f64_to_f32(b);
                }
            }
    }
    return EPO_WIRE_OK;
}
