/*
 * ep_model.h — the rest of the decoder layer on the GPU,
 * part of libep_b200.so.
 *
 * The reference runs the whole decoder on the host in fp64
 * (/root/reference/proj/core/src/model.cpp): init_model (:82-102), embed
 * (:104-129), layer_norm (:131-150), transformer_layer (:152-209), prefill
 * (:211-236), unembed_logits (:238-246), argmax_token (:248-255) and
 * decode_step (:257-283). This section keeps the model weights and one KV
 * page pool per layer resident in HBM and runs a forward pass of a batch of
 * requests through every layer with the spliced attention of ep_attn.h in
 * the middle, so a greedy rollout never leaves the device except for the
 * one token id per step the caller asks for.
 *
 * Same conventions as ep_attn.h: plain pointers, ep_status return codes,
 * ep_last_error(); the caller owns every buffer it passes in; stream-ordered.
 */
#ifndef EP_MODEL_H
#define EP_MODEL_H

#include "ep/ep_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ModelConfig (model.hpp:15-25) plus the storage dtype of the weights and
 * activations: EP_F64 keeps the reference's precision (its own tests'
 * tolerances hold), EP_F32 is the serving precision (BASELINE config 1). */
typedef struct ep_model_config {
    int32_t n_layers;
    int32_t n_heads;
    int32_t d_model;
    int32_t vocab_size;
    int32_t max_positions;
    int32_t dtype; /* EP_F64 or EP_F32 */
    uint64_t init_seed;
} ep_model_config;

typedef struct ep_model_s* ep_model;

/* init_model (model.cpp:82-102): every weight is the i-th draw of one
 * SplitMix64(init_seed) stream, uniform(-0.1, 0.1), in the order embedding,
 * per layer wq wk wv wo w1 b1 w2 b2, unembedding — drawn on the device in
 * fp64 and stored in cfg->dtype. Also allocates the per-layer KV page pools
 * [num_pages][n_heads][page_tokens][d_head] in kv_dtype (EP_F64 requires
 * dtype EP_F64; EP_F32 / EP_BF16 require dtype EP_F32). EP_EINVAL for the
 * configs ModelConfig::validate rejects (model.cpp:42-50). */
int ep_model_create(ep_handle h, const ep_model_config* cfg, int32_t kv_dtype,
                    int32_t page_tokens, int64_t num_pages, ep_model* out);
int ep_model_destroy(ep_model m);

/* Model::weight_sum (model.cpp:52-67): the fp64 draws summed in generation
 * order (synchronous). */
int ep_model_weight_sum(ep_model m, double* out);

/* The KV page pool of one layer (page ids are shared by all layers: a
 * segment's page list addresses the same pages in every layer's pool). */
int ep_model_kv_pool(ep_model m, int32_t layer, ep_kv_pool* out);

/* Device pointer + element count of one named weight tensor, row-major as in
 * LayerWeights (model.hpp:27-33): name = "embedding", "unembed", or per layer
 * "wq" "wk" "wv" "wo" "w1" "b1" "w2" "b2" (layer ignored for the first two). */
int ep_model_weight(ep_model m, const char* name, int32_t layer, void** ptr, size_t* count);

/* One forward pass: for every request b of the batch, the LAST n_new[b]
 * tokens of its spliced sequence (host splice table, as in ep_plan_create:
 * seg_indptr [batch+1], segs, page_table) are new tokens with ids
 * tokens[sum n_new] (host). Per layer (transformer_layer, model.cpp:152-209):
 * LayerNorm -> Q/K/V, the new K/V rows written into their pages (the segments
 * must already cover those positions), spliced causal attention over all of
 * the request's keys (its cached segments plus the new tokens themselves),
 * Wo + residual, LayerNorm -> W1 + b1 -> ReLU -> W2 + b2 + residual. Then per
 * request, unembed_logits + argmax_token of its last new row.
 *   hidden: NULL or device [sum n_new][d_model] (model dtype) final hidden rows
 *   logits: NULL or device [batch][vocab] (model dtype)
 *   next:   NULL or device int32 [batch] greedy next token (ties -> lowest id)
 * EP_EINVAL for unknown token ids or positions >= max_positions (embed's
 * std::out_of_range, model.cpp:104-129) and for splice tables the
 * SegmentedCache invariants reject. decode_step = one token per request;
 * prefill = a request's whole new segment. */
int ep_model_forward(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                     const int32_t* page_table, const int32_t* n_new, const int32_t* tokens,
                     void* hidden, void* logits, int32_t* next, ep_stream stream);

/* Greedy speculative verify on the decoder: per request
 * b, tokens [sum n_new] holds [last, d1..dk] (k = n_new[b] - 1) at the LAST
 * n_new[b] positions of its splice table — the reference's construction,
 * prefill(model, [last, d1..dk], generated, end_position, cache)
 * (model.cpp:211-236) — and every new row is unembedded and argmaxed
 * (unembed_logits + argmax_token, model.cpp:238-255):
 *   targets:    device int32 [sum n_new], g_j of row j (ties -> lowest id)
 *   n_accepted: device int32 [batch], the largest n <= k with d_i == g_{i-1}
 *               for all i <= n (emit d1..dn, then the bonus token g_n)
 *   logits:     NULL or device [sum n_new][vocab] (model dtype)
 * The K/V of all k+1 rows are written into their slots; a caller that keeps
 * n accepted drafts keeps positions up to last + n (the rest are rewritten by
 * later steps). Errors as ep_model_forward. */
int ep_model_verify(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                    const int32_t* page_table, const int32_t* n_new, const int32_t* tokens, void* logits,
                    int32_t* targets, int32_t* n_accepted, ep_stream stream);

/* decode_greedy (model.cpp:285-297) resident on the device: for every request
 * b, the LAST n_steps positions of its splice table (a trailing generated
 * segment the caller has reserved) are decoded autoregressively — the first
 * embeds first_tokens[b] (host), each later one the greedy argmax of the
 * step before (decode_step, model.cpp:257-283). out_tokens (host, [batch]
 * [n_steps]) receives the argmax after every step; the K/V of every step is
 * written into its reserved slot. One step (all layers + argmax + a position
 * advance) is captured into a CUDA graph once and replayed n_steps times:
 * no host work and no host round trip between steps. Synchronous on return.
 * EP_EINVAL as ep_model_forward, and for a request with no cached token
 * before the reserved positions (decode_step's empty-cache error). */
int ep_model_generate(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                      const int32_t* page_table, int32_t n_steps, const int32_t* first_tokens,
                      int32_t* out_tokens, ep_stream stream);

/* Which attention kernel the last ep_model_forward / ep_model_generate used: 1 = spliced decode /
 * prefill plans (K1/K3 of ep_attn.h), 2 = the generic paged kernel (fp64, or
 * d_head outside {64, 128}), 3 = the persistent rollout kernel (fp32 models of
 * <= 8 rows in ep_model_generate: all steps in one cooperative launch). */
int ep_model_last_attention_path(ep_model m);

#ifdef __cplusplus
}
#endif
#endif /* EP_MODEL_H */
