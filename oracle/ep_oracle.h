/*
 * ep_oracle.h — CPU restatement of EdgePrompt's spliced-attention path.
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * legs may load it. The product path (libep_b200.so) never links it.
 *
 * Every function restates one reference routine (file:line into
 * /root/reference/proj/core) in plain C99 with fp64 arithmetic, and is
 * pinned against the reference itself (oracle/_ref, built from the
 * unmodified sources by oracle/Makefile) and against the known answers of
 * the reference's own tests (tests/test_oracle_golden.py).
 */
#ifndef EP_ORACLE_H
#define EP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { EPO_OK = 0, EPO_EINVAL = 1, EPO_EMASKED = 2 };

/* matrix.cpp:88-93 */
double epo_log_add_exp(double a, double b);

/* attention.cpp:29-33 — number of visible keys of a segment for query row i */
size_t epo_visible_keys(size_t q_off, size_t k_off, size_t n_keys, size_t i);

/* attention.cpp:80-114. Row-major q [n_q x d], k/v [n_keys x d] with leading
 * dims ldq/ldk/ldv (elements). out [n_q x d] (ld = d), lse [n_q].
 * Returns EPO_EINVAL for d == 0 (attention.cpp:15). */
int epo_partial_attention(const double* q, size_t ldq, size_t n_q, const double* k,
                          size_t ldk, const double* v, size_t ldv, size_t n_keys, size_t d,
                          size_t q_off, size_t k_off, double* out, double* lse);

/* attention.cpp:45-78. EPO_EMASKED if any row sees no key. */
int epo_full_attention(const double* q, size_t n_q, const double* k, const double* v,
                       size_t n_keys, size_t d, size_t q_off, size_t k_off, double* out);

/* attention.cpp:116-145. outs[p] is [n_q x d], lses[p] is [n_q]. */
int epo_merge_partials(size_t n_parts, const double* const* outs, const double* const* lses,
                       size_t n_q, size_t d, double* out, double* lse);

/* attention.cpp:147-156 (EPO_EMASKED when a row is masked in every part) */
int epo_fuse_partials(size_t n_parts, const double* const* outs, const double* const* lses,
                      size_t n_q, size_t d, double* out);

/* model.cpp:248-255: first index of the maximum (strict >). */
uint32_t epo_argmax(const double* logits, size_t n);

/* model.cpp:131-150: parameterless LayerNorm of one row, eps 1e-5. */
void epo_layer_norm_row(const double* x, size_t n, double* out);

/* ------------------------------------------------------------------------ */
/* Batched spliced attention over a paged splice table: the attention block  */
/* of transformer_layer (model.cpp:161-182) applied to every (request,       */
/* q-head) of a batch, with GQA as KV-head indexing (q-head h reads KV head  */
/* h / (Hq/Hkv)). Layout is the one the CUDA path consumes.   */
/* ------------------------------------------------------------------------ */

enum { EPO_DT_F32 = 0, EPO_DT_BF16 = 1, EPO_DT_F64 = 2 };

typedef struct {
    int32_t origin;     /* 0 cloud, 1 edge, 2 generated (cache.hpp:11) */
    int32_t len;        /* tokens in the segment */
    int64_t pos_offset; /* absolute position of its first token */
    int64_t page_off;   /* index into page_table of its first page */
} epo_segment;

typedef struct {
    int kv_dtype;             /* EPO_DT_F32 / EPO_DT_BF16 (bf16 as raw uint16) */
    int n_kv_heads, n_q_heads, d_head, page_tokens;
    const void* k_pages;      /* [num_pages][Hkv][page_tokens][d] */
    const void* v_pages;
    int batch;
    int n_q;                  /* query rows per request */
    const int64_t* seg_indptr;  /* [batch+1] */
    const epo_segment* segs;
    const int32_t* page_table;
    const int64_t* q_pos;     /* [batch] absolute position of query row 0 */
    int q_dtype;              /* EPO_DT_F32 / EPO_DT_BF16 */
    const void* q;            /* [batch][n_q][Hq][d] */
} epo_splice_batch;

/* out [batch][n_q][Hq][d], lse [batch][n_q][Hq] (natural log). Units
 * (request, q-head) are spread over n_threads pthreads. If unit_list is
 * non-NULL only those n_units units (b * Hq + h) are computed. */
int epo_spliced_attention(const epo_splice_batch* s, int n_threads, const int64_t* unit_list,
                          int64_t n_units, double* out, double* lse);

/* Greedy speculative verify, constructed from prefill + unembed_logits +
 * argmax (model.cpp:211-255). attn_out [batch][n_q][Hq*d]
 * (n_q = k+1 rows: last accepted token then k drafts), w_score [Hq*d][vocab],
 * drafts [batch][k]. Writes target ids g [batch][n_q], accepted counts
 * n_acc [batch] (0..k) and the top-2 logit gap per row (for the margin guard). */
int epo_verify_greedy(const double* attn_out, int batch, int n_q, int width,
                      const double* w_score, int vocab, const int32_t* drafts,
                      int32_t* target_ids, int32_t* n_accepted, double* top2_gap);

/* SplitMix64 (rng.hpp:10-29), vectorised: dst[i] = uniform(lo,hi) from the
 * i-th draw of SplitMix64(seed), rounded to dtype (f64 -> f32 RN -> bf16 RN). */
void epo_fill_uniform(int dtype, void* dst, size_t n, uint64_t seed, double lo, double hi);

/* ------------------------------------------------------------------------ */
/* KV ingest: an EPKV kv_frame (wire.hpp:59-75) decoded into device-layout   */
/* pages.                                                */
/* ------------------------------------------------------------------------ */

/* WireError::Kind (wire.hpp:94-104) + 1; EPO_WIRE_NOT_KV: a valid frame of
 * another message type. */
enum { EPO_WIRE_OK = 0, EPO_WIRE_BAD_MAGIC = 1, EPO_WIRE_BAD_VERSION = 2, EPO_WIRE_TRUNCATED = 3,
       EPO_WIRE_LENGTH_OVERFLOW = 4, EPO_WIRE_MALFORMED = 5, EPO_WIRE_NOT_KV = 6 };

typedef struct {
    uint32_t session_id;
    uint32_t seq_len;
    uint16_t layer;
    uint16_t n_heads;
    uint16_t d_head;
    uint16_t pad;
} epo_kv_frame_info;

/* decode_frame restricted to kv frames (wire.cpp:138-221): validates the
 * 10-byte header and the 14-byte body header, fills *info and, when k / v are
 * non-NULL, the seq_len x (n_heads*d_head) row-major doubles. Returns an
 * EPO_WIRE_* code. */
int epo_kv_frame_decode(const uint8_t* frame, size_t n, epo_kv_frame_info* info, double* k,
                        double* v);

/* f64 -> bf16 (raw) and f64 -> f32, round to nearest even, correctly rounded. */
uint16_t epo_f64_to_bf16(double x);
float epo_f64_to_f32(double x);

/* The ingest: token t of the frame -> page page_table[t / page_tokens], slot
 * t % page_tokens; frame head h (columns [h*d, (h+1)*d), segment_from_frame,
 * edge.cpp:61-67) -> kv head h of the page. Pages [num][n_heads][page_tokens][d]
 * in kv_dtype (EPO_DT_F32 / EPO_DT_BF16). Returns an EPO_WIRE_* code. */
int epo_kv_ingest(const uint8_t* frame, size_t n, int kv_dtype, int page_tokens,
                  const int32_t* page_table, void* k_pages, void* v_pages, epo_kv_frame_info* info);

#ifdef __cplusplus
}
#endif
#endif
