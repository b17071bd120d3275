/*
 * ep_attn.h — C-ABI of the B200 spliced-KV attention library (libep_b200.so).
 *
 * This is the drop-in boundary for EdgePrompt's attention/splice path. The
 * reference exposes it as C++ (namespace edgeprompt) in
 *   /root/reference/proj/core/include/edgeprompt/attention.hpp:13-52
 *   /root/reference/proj/core/include/edgeprompt/cache.hpp:11-61
 * and the reference's link-level swap point is attention.cpp in
 * proj/core/CMakeLists.txt:1-14. Every entry point below names the reference
 * interface it replaces. Plain pointers and sizes only; no CUDA or torch types
 * (streams are passed as void* = cudaStream_t). No exceptions cross the ABI:
 * every call returns an ep_status and sets a thread-local message readable with
 * ep_last_error().
 *
 * Ownership: the caller owns every host and device buffer passed in. The
 * library allocates only inside objects it creates (ep_handle, ep_plan,
 * ep_cache) and frees them in the matching destroy call.
 *
 * Threading: an ep_handle may be used by one host thread at a time; separate
 * handles are independent. Device entry points (*_dev, ep_spliced_*) are
 * stream-ordered and asynchronous; host-buffer entry points (*_f64) are
 * synchronous, like the reference functions they replace.
 */
#ifndef EP_ATTN_H
#define EP_ATTN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EP_ABI_VERSION 1

typedef enum ep_status {
    EP_OK = 0,
    EP_EINVAL = 1,       /* std::invalid_argument in the reference (attention.cpp:14-25, :117) */
    EP_EMASKED = 2,      /* std::domain_error: a row sees no key (attention.cpp:52-56, :150-153) */
    EP_ECUDA = 3,        /* CUDA runtime / launch failure */
    EP_ENCCL = 4,        /* NCCL failure (split-KV combine) */
    EP_ENOMEM = 5,       /* device or host allocation failed */
    EP_EUNSUPPORTED = 6, /* shape/dtype combination without a kernel instance */
    EP_EWIRE = 7         /* malformed EPKV frame (wire::WireError, wire.hpp:94-104) */
} ep_status;

/* Numbering matches oracle/ep_oracle.h (EPO_DT_*). bf16 is raw uint16 storage. */
typedef enum ep_dtype { EP_F32 = 0, EP_BF16 = 1, EP_F64 = 2 } ep_dtype;

typedef struct ep_context* ep_handle;
typedef struct ep_plan_s* ep_plan;
typedef void* ep_stream; /* cudaStream_t; NULL = legacy default stream */

int ep_abi_version(void);
const char* ep_last_error(void);

/* Binds to a CUDA device and creates the per-handle workspace. */
int ep_create(int device, ep_handle* out);
int ep_destroy(ep_handle h);

/* ==================================================================== */
/* 1. Drop-in, host buffers, fp64 (synchronous). Replaces attention.cpp. */
/*    Row-major, leading dimension = d. q [n_q x d], k/v [n_keys x d],  */
/*    out [n_q x d], lse [n_q] (natural log; -inf for masked rows).     */
/* ==================================================================== */

/* edgeprompt::partial_attention (attention.hpp:39-40, attention.cpp:80-114) */
int ep_partial_attention_f64(ep_handle h, const double* q, size_t n_q, const double* k,
                             const double* v, size_t n_keys, size_t d, size_t query_offset,
                             size_t key_offset, double* out, double* lse);

/* edgeprompt::full_attention (attention.hpp:35, attention.cpp:45-78).
 * EP_EMASKED if any row has no visible key. */
int ep_full_attention_f64(ep_handle h, const double* q, size_t n_q, const double* k,
                          const double* v, size_t n_keys, size_t d, size_t query_offset,
                          size_t key_offset, double* out);

/* edgeprompt::merge_partials (attention.hpp:52, attention.cpp:116-145).
 * outs[p] -> [n_q x d], lses[p] -> [n_q]. EP_EINVAL when n_parts == 0. */
int ep_merge_partials_f64(ep_handle h, size_t n_parts, const double* const* outs,
                          const double* const* lses, size_t n_q, size_t d, double* out,
                          double* lse);

/* edgeprompt::fuse_partials (attention.hpp:47, attention.cpp:147-156).
 * EP_EMASKED when some row is masked in every part. */
int ep_fuse_partials_f64(ep_handle h, size_t n_parts, const double* const* outs,
                         const double* const* lses, size_t n_q, size_t d, double* out);

/* ==================================================================== */
/* 2. Device buffers, stream-ordered. Same math as section 1 on device  */
/*    pointers; dt = EP_F64 or EP_F32 (q, k, v, out and lse share dt).   */
/* ==================================================================== */

int ep_partial_attention_dev(ep_handle h, ep_dtype dt, const void* q, size_t ldq, size_t n_q,
                             const void* k, size_t ldk, const void* v, size_t ldv,
                             size_t n_keys, size_t d, size_t query_offset, size_t key_offset,
                             void* out, size_t ldo, void* lse, ep_stream stream);

/* K2: LSE merge of n_parts partials in part order. outs: [n_parts][rows][d],
 * lses: [n_parts][rows]; out [rows][d], lse [rows]. dt = EP_F64 or EP_F32. */
int ep_merge_partials_dev(ep_handle h, ep_dtype dt, size_t n_parts, const void* outs,
                          const void* lses, size_t rows, size_t d, void* out, void* lse,
                          ep_stream stream);

/* K5, cross-GPU split-KV combine: n_parts rank partials packed as
 * [part][rows*d fp32 o | rows fp32 lse (natural log)] — exactly what one
 * all-gather of every rank's ep_spliced_attention(o_dtype EP_F32, lse) output
 * yields — merged in part (= rank = KV segment) order like merge_partials
 * (attention.cpp:116-145). out [rows][d] in out_dtype (EP_F32/EP_BF16), lse
 * [rows] natural log (may be NULL). d <= 256. */
int ep_merge_partials_packed_dev(ep_handle h, int32_t n_parts, const float* packed, int32_t rows,
                                 int32_t d, int32_t out_dtype, void* out, float* lse,
                                 ep_stream stream);

/* ==================================================================== */
/* 3. Paged splice table (cache.hpp:11-61 made device-resident).        */
/* ==================================================================== */

/* One KV segment of one request (KVSegment, cache.hpp:18-28): `len` tokens
 * at absolute positions [pos_offset, pos_offset+len), stored in pages
 * page_table[page_off ...], filling each page from slot 0. Pages may be
 * shared between requests (a cloud prompt is stored once). */
typedef struct ep_segment {
    int32_t origin;     /* 0 cloud, 1 edge, 2 generated (SegmentOrigin, cache.hpp:11) */
    int32_t len;
    int64_t pos_offset;
    int64_t page_off;
} ep_segment;

/* Device page pool: K and V as [num_pages][n_kv_heads][page_tokens][d_head]
 * (one contiguous page_tokens x d_head tile per (page, head)). */
typedef struct ep_kv_pool {
    int32_t dtype;      /* EP_F32 or EP_BF16 */
    int32_t n_kv_heads;
    int32_t d_head;     /* 64 or 128 */
    int32_t page_tokens;/* multiple of 64 */
    int64_t num_pages;
    void* k_pages;
    void* v_pages;
} ep_kv_pool;

/* Builds the launch plan for one batch from a HOST copy of the splice table
 * (seg_indptr [batch+1], segs, page_table, q_pos [batch] = absolute position
 * of each request's first query row). n_q query rows per request, n_q_heads
 * query heads (GQA group = n_q_heads / n_kv_heads). The plan owns its device
 * descriptors and fp32 partial workspace. ctas_per_sm = 0 picks the default. */
int ep_plan_create(ep_handle h, const ep_kv_pool* pool, int32_t n_q_heads, int32_t n_q,
                   int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                   const int32_t* page_table, const int64_t* q_pos, int32_t ctas_per_sm,
                   ep_plan* out);
/* Re-plans in place (e.g. after appending generated tokens); device buffers are
 * reused when large enough, so captured CUDA graphs stay valid. */
int ep_plan_update(ep_plan p, const int64_t* seg_indptr, const ep_segment* segs,
                   const int32_t* page_table, const int64_t* q_pos, ep_stream stream);
/* ==================================================================== */
/* 2b. Splice state: SegmentedCache (cache.hpp:30-61) as a C-ABI object.  */
/* ==================================================================== */

/* Per layer and request, an ordered list of segments {origin, pos_offset,
 * len, pages} over the layer's page pool — the reference's per-layer
 * KVSegment lists with the K/V living in device pages. Host-only (no CUDA
 * calls); not thread-safe (one mutator per cache). */
typedef struct ep_cache_s* ep_cache;
int ep_cache_create(int32_t n_layers, int32_t batch, int32_t page_tokens, ep_cache* out);
int ep_cache_destroy(ep_cache c);
/* SegmentedCache::end_position (cache.cpp:21-24): layer 0's end; -1 for a bad request. */
int64_t ep_cache_end_position(ep_cache c, int32_t b);
/* SegmentedCache::append (cache.cpp:25-53) for request b: layer = -1 appends
 * the segment to every layer (the common case: page ids shared by the layers'
 * pools), layer >= 0 to that layer only (K/V arriving layer by layer). Every
 * invariant is checked for every affected layer before anything changes
 * (atomic): contiguous with the end, non-empty, origin order cloud -> edge ->
 * generated; EP_EINVAL with the reference's messages. */
int ep_cache_append(ep_cache c, int32_t layer, int32_t b, int32_t origin, int64_t pos_offset, int32_t len,
                    const int32_t* pages, int32_t n_pages);
/* append_generated_token (cache.cpp:55-80) for the whole batch, every layer:
 * request b's trailing generated segment grows by n_tokens[b] (created at the
 * end if absent), no copy — the new tokens take the last page's free slots,
 * then pages new_pages[b * max_new ..] (pages_used[b] of them). dst_page /
 * dst_slot [sum n_tokens] receive where each new token's K/V row goes (for
 * ep_kv_append or a projection epilogue). */
int ep_cache_append_generated(ep_cache c, const int32_t* n_tokens, const int32_t* new_pages, int32_t max_new,
                              int32_t* dst_page, int32_t* dst_slot, int32_t* pages_used);
/* Drops the last n_tokens of request b's generated segment in every layer
 * (rejected speculative drafts); pages no longer used are written to
 * released (may be NULL) and counted in n_released. */
int ep_cache_truncate(ep_cache c, int32_t b, int32_t n_tokens, int32_t* released, int32_t* n_released);
/* SegmentedCache::check_consistent (cache.cpp:82-103): gapless coverage,
 * origin order and identical position ranges across layers, per request;
 * EP_EINVAL with the reference's description ("gap in position coverage",
 * "origin order violated", "layers cover different position ranges", ...). */
int ep_cache_check_consistent(ep_cache c);
/* One layer's table in the ep_plan_create layout (seg_indptr [batch+1],
 * segs, page_table); seg_indptr = NULL only reports the sizes. */
int ep_cache_layer_arrays(ep_cache c, int32_t layer, int64_t* seg_indptr, ep_segment* segs, int64_t segs_cap,
                          int32_t* page_table, int64_t pages_cap, int64_t* n_segs, int64_t* n_pages);
/* Plans straight from the cache: request b's queries are its last n_q
 * positions (decode_step: n_q = 1; verify: k + 1). ep_plan_update_cache
 * re-plans after the cache grew (per-token growth: a host rebuild of a few
 * microseconds plus one async upload). */
int ep_plan_create_cache(ep_handle h, const ep_kv_pool* pool, ep_cache c, int32_t layer, int32_t n_q_heads,
                         int32_t n_q, ep_plan* out);
int ep_plan_update_cache(ep_plan p, ep_cache c, int32_t layer, int32_t n_q, ep_stream stream);

/* Prefill plan — the cloud-prompt / edge prefill attention tiles (prefill,
 * model.cpp:211-236 -> transformer_layer's attention block, model.cpp:161-182;
 * CloudServer::serve_stream, cloud.cpp:160-172). The LAST n_new[b] tokens of
 * request b's spliced sequence are queries; query t attends to every key at a
 * position <= its own (CausalSpan rule, attention.cpp:29-33). Their K/V must
 * already be in the pool as part of the segments. q / o are token-major
 * [sum n_new][n_q_heads][d_head], lse [sum n_new][n_q_heads]; run with
 * ep_spliced_attention. bf16 KV with d_head 128: tcgen05 tiles of 128/G query
 * tokens x G heads (o_dtype EP_BF16 uses a bf16 P operand, EP_F32 a hi+lo
 * split). Otherwise (f32 or bf16 KV, d_head 64/128, G <= 8): CUDA-core chunks
 * of 8/G query tokens on the decode kernel. */
int ep_plan_create_prefill(ep_handle h, const ep_kv_pool* pool, int32_t n_q_heads, int32_t batch,
                           const int64_t* seg_indptr, const ep_segment* segs,
                           const int32_t* page_table, const int32_t* n_new, ep_plan* out);
int ep_plan_destroy(ep_plan p);
/* Introspection: number of CTAs, work items and pages in the plan. */
int ep_plan_info(ep_plan p, int64_t* n_ctas, int64_t* n_items, int64_t* n_pages);

/* K1 + K2: spliced attention for every (request, query row, q-head) of the
 * plan. q [batch][n_q][n_q_heads][d] (q_dtype EP_F32/EP_BF16); o same layout
 * (o_dtype EP_F32/EP_BF16); lse [batch][n_q][n_q_heads] fp32 natural log
 * (may be NULL). Reproduces transformer_layer's attention block
 * (model.cpp:161-182): a per-segment partial with CausalSpan{q_pos,
 * seg.pos_offset} merged in segment order — here as one online-softmax pass
 * over the pages, so no spliced copy of the cache is materialised. */
int ep_spliced_attention(ep_handle h, ep_plan p, const ep_kv_pool* pool, int32_t q_dtype,
                         const void* q, int32_t o_dtype, void* o, float* lse, ep_stream stream);

/* For cross-GPU split-KV each rank calls ep_spliced_attention on its own KV
 * shard with o_dtype = EP_F32 and a non-NULL lse: (o, lse) of that shard's keys
 * only, which ep_merge_partials_dev (or ep_splitkv_combine in the NCCL build)
 * recombines in rank = segment order. */

/* ---- Speculative verify: fused score + greedy accept (K4) ----------- */
/* Constructed from prefill + unembed_logits + argmax_token (model.cpp:211-255,
 * SURVEY a16): for verify row j of a request (the last accepted token, then
 * drafts d1..dk), g_j = argmax(LayerNorm(attn_row_j) @ W_score), ties to the
 * lowest id; accepted n = largest n <= k with d_i == g_{i-1} for all i <= n
 * (emit d1..dn, then g_n). */
typedef struct ep_verifier_s* ep_verifier;

/* w_score_t: device bf16 [vocab][width] (W_score transposed, K-major), kept
 * by reference; width % 64 == 0, vocab % 256 == 0. */
int ep_verifier_create(ep_handle h, int32_t width, int32_t vocab, const void* w_score_t,
                       ep_verifier* out);
int ep_verifier_destroy(ep_verifier v);

/* attn_out: device [batch * n_q][width] in attn_dtype (the ep_spliced_attention
 * output [batch][n_q][n_q_heads][d], width = n_q_heads * d). EP_F32 (preferred)
 * is scored as a bf16 hi+lo pair at ~fp32 accuracy; EP_BF16 in one pass.
 * drafts [batch][n_q-1], target_ids [batch][n_q], n_accepted [batch] (device
 * int32). logits: NULL, or a device fp32 [batch * n_q][vocab] buffer receiving
 * LayerNorm(row) @ W_score (diagnostics). */
int ep_verify_greedy(ep_handle h, ep_verifier v, int32_t batch, int32_t n_q, int32_t attn_dtype,
                     const void* attn_out, const int32_t* drafts, int32_t* target_ids,
                     int32_t* n_accepted, float* logits, ep_stream stream);

/* Appends n_tok token rows per request into the pool (the device form of
 * SegmentedCache::append_generated_token, cache.cpp:55-80, without its
 * whole-segment copy). k_new/v_new: [n_rows][n_kv_heads][d_head] in the pool
 * dtype; row i goes to page dst_page[i], slot dst_slot[i] (device int32).
 * Stream-ordered; launched with programmatic dependent launch, so a caller's
 * own PDL-launched successor kernel must execute griddepcontrol.wait before
 * it reads the pool (ordinary launches and this library's kernels do). The
 * same holds for the descriptor patch of ep_plan_update_cache. */
int ep_kv_append(ep_handle h, const ep_kv_pool* pool, int32_t n_rows, const int32_t* dst_page,
                 const int32_t* dst_slot, const void* k_new, const void* v_new,
                 ep_stream stream);

/* KV ingest: one EPKV kv_frame as the reference's
 * encode_frame writes it (wire.hpp:59-75, wire.cpp:70-136: 10-byte header,
 * 14-byte body header, then K and V as seq_len x (n_heads*d_head) row-major
 * little-endian doubles) decoded straight into the page pool: frame token t
 * -> page page_table[t / page_tokens], slot t % page_tokens; frame head h
 * (columns [h*d, (h+1)*d), segment_from_frame, edge.cpp:61-67) -> kv head h;
 * values rounded to the pool dtype (f64 -> bf16 / f32, round to nearest even).
 * frame may be device memory, pinned host memory (read in place by the
 * kernel: decode + convert + scatter in one pass) or pageable host memory
 * (staged). Validation mirrors decode_frame (wire.cpp:138-221): EP_EWIRE
 * with info->wire_error = WireError::Kind + 1 (1 bad_magic, 2 bad_version,
 * 3 truncated, 4 length_overflow, 5 malformed) or 6 for a valid frame that
 * is not a kv frame. EP_EINVAL when n_heads / d_head do not match the pool,
 * seq_len is 0 (expect_kv_frame, edge.cpp:41-60) or n_pages is too small.
 * page_table: device int32 [n_pages]. Stream-ordered; a pinned or device
 * frame must stay valid until the stream reaches this point. */
typedef struct ep_kv_frame_info {
    uint32_t session_id;
    uint32_t seq_len;
    uint16_t layer;
    uint16_t n_heads;
    uint16_t d_head;
    uint16_t pad;
    int32_t wire_error;
} ep_kv_frame_info;

int ep_kv_ingest_frame(ep_handle h, const ep_kv_pool* pool, const void* frame, size_t frame_bytes,
                       const int32_t* page_table, int32_t n_pages, ep_kv_frame_info* info,
                       ep_stream stream);

/* Deferred-check form of ep_kv_ingest_frame for device-resident frames
 * (GPUDirect receive buffers): no host synchronisation. The host derives
 * seq_len from frame_bytes and the pool's head shape and launches at once;
 * the kernel re-parses the 24-byte header (the same decode_frame rules) and,
 * when it disagrees, writes nothing and records the first failure in a
 * per-handle status word. ep_kv_ingest_poll synchronises `stream`, returns
 * that failure (EP_EWIRE with info->wire_error, or EP_EINVAL for the pool
 * checks) and clears it. Host frames, and device frames whose length does not
 * fit the pool's head shape, take the synchronous path (immediate errors). */
int ep_kv_ingest_frame_async(ep_handle h, const ep_kv_pool* pool, const void* frame, size_t frame_bytes,
                             const int32_t* page_table, int32_t n_pages, ep_stream stream);
int ep_kv_ingest_poll(ep_handle h, ep_stream stream, ep_kv_frame_info* info);

/* ==================================================================== */
/* 3b. Cross-GPU split-KV combine over NVLink peer memory (config 4).   */
/* ==================================================================== */

/* The reference fuses any ordered partition of a row's keys with
 * merge_partials (attention.cpp:116-156). When the partition is across the
 * GPUs of one box, each rank's fp32 (o, lse) partial is pushed straight into
 * every peer's receive buffer over NVLink (remote stores of {value, flag}
 * words) and merged there in rank order by the same kernel — no NCCL on the
 * data path, one launch, graph-capturable. Collective: every rank creates,
 * connects, combines and destroys in the same order (barrier before
 * destroy). The group owns one device allocation: receive words
 * [2][world][rows_max][d/2 + 1] x 16 B + per-CTA epochs. d even, <= 256. */
typedef struct ep_peer_group_s* ep_peer_group;
#define EP_IPC_HANDLE_BYTES 64

int ep_peer_group_create(ep_handle h, int32_t world, int32_t rank, int32_t rows_max, int32_t d,
                         ep_peer_group* out);
/* cudaIpcMemHandle_t of the group's allocation (EP_IPC_HANDLE_BYTES bytes) for
 * a cross-process exchange (e.g. torch.distributed.all_gather_object). */
int ep_peer_group_export(ep_peer_group g, void* ipc_handle);
/* Device base pointer of the allocation, for ranks that share one process. */
int ep_peer_group_base(ep_peer_group g, void** base);
/* handles: world * EP_IPC_HANDLE_BYTES bytes in rank order (own entry ignored). */
int ep_peer_group_connect_ipc(ep_peer_group g, const void* handles);
/* bases: world device pointers in rank order (own entry ignored); enables peer
 * access when the peer lives on another device of this process. */
int ep_peer_group_connect_ptrs(ep_peer_group g, void* const* bases);
/* o_part [rows][d] fp32 and lse_part [rows] (natural log) = this rank's
 * ep_spliced_attention output over its KV shard -> out [rows][d] (out_dtype
 * EP_F32/EP_BF16) and out_lse [rows] (may be NULL), identical on every rank.
 * rows <= rows_max. */
int ep_splitkv_combine_dev(ep_handle h, ep_peer_group g, int32_t rows, const float* o_part,
                           const float* lse_part, int32_t out_dtype, void* out, float* out_lse,
                           ep_stream stream);
int ep_peer_group_destroy(ep_peer_group g);

/* Split-KV attention with the cross-GPU combine fused into the decode
 * kernel (config 4): plan p covers this rank's KV shard of every request
 * (every rank the same requests, the same query rows); the K1 pass over the
 * shard pushes each (request, kv-head) unit's merged fp32 (o, lse) rows into
 * every rank's receive buffer of group g over NVLink peer memory as soon as
 * the unit is done, and at the end of the kernel each unit's owner CTA
 * merges the W rank partials in rank (= segment) order (attention.cpp:
 * 116-145) into o / lse — one launch per rank, no separate combine. Every
 * rank ends with identical rows. Collective: every rank calls it once per
 * step with the same plan structure. A group serves either this call or
 * ep_splitkv_combine_dev, not both. EP_EUNSUPPORTED for plans not on K1
 * (shared-prefix cascade, tcgen05 tiles, the generic kernel, query chunks). */
int ep_spliced_attention_splitkv(ep_handle h, ep_plan p, const ep_kv_pool* pool, int32_t q_dtype,
                                 const void* q, ep_peer_group g, int32_t o_dtype, void* o, float* lse,
                                 ep_stream stream);

/* ==================================================================== */
/* 4. Utilities                                                         */
/* ==================================================================== */

/* dst[i] = uniform(lo, hi) of the i-th SplitMix64(seed) draw (rng.hpp:10-29),
 * rounded f64 -> f32 (RN) -> bf16 (RN) for EP_BF16. Device pointer. */
int ep_fill_uniform(ep_handle h, ep_dtype dt, void* dst, size_t n, uint64_t seed, double lo,
                    double hi, ep_stream stream);

/* Number of kernel launches issued by this handle since creation (evidence for
 * bench.py's gpu_launches). */
int64_t ep_launch_count(ep_handle h);

#ifdef __cplusplus
}
#endif
#endif /* EP_ATTN_H */
