// model_internal.h — launchers of kern_model.cu (the decoder layer around the
// spliced attention). Not part of the ABI.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include "ep_internal.h"

namespace ep {

// Epilogues of the dense kernel (transformer_layer, model.cpp:161-205).
enum DenseEpi : int {
    kEpiStore = 0,  // out = acc                        (unembed_logits)
    kEpiQKV = 1,    // q -> q_out, k/v -> page slots    (Q/K/V projections + append)
    kEpiResid = 2,  // out = (resid + acc) [+ bias]     (Wo, W2 + b2)
    kEpiRelu = 3,   // out = max(acc + bias, 0)         (W1 + b1, ReLU)
};

// out[r][c] = epi( LN?(x[row_map ? row_map[r] : r]) @ W )[c]; W is n_wblk
// row-major [K][N / n_wblk] column blocks (wq | wk | wv for kEpiQKV).
struct DenseArgs {
    const void* x;
    const int32_t* row_map;  // gathered input rows (unembedding of the last rows), may be null
    int32_t n, K, N;
    const void* w[3];
    int32_t n_wblk;
    const void* bias;
    const void* resid;  // [n][N]
    void* out;          // [n][N]
    // kEpiQKV: q rows [n][N/3]; k/v into pages [page][H][P][dh] at (dst_page[r], dst_slot[r])
    void* q_out;
    void* k_pages;
    void* v_pages;
    int32_t kv_dtype, H, P, dh;
    const int32_t* dst_page;
    const int32_t* dst_slot;
    // rollout: device step counter; dst_page / dst_slot are [steps][n] and
    // row r of step s is entry s * n + r (null = a single forward)
    const int32_t* step;
    // fused embedding (LN kernels only): row r = embedding[token] + pe[pos],
    // token = tok[r] (step 0) or tok_prev[(step - 1) * n + r], pos = pos[step * n + r];
    // the embedded rows are also stored to x_store (the layer's residual input)
    const void* emb;
    const double* pe;
    const int32_t* tok;
    const int32_t* tok_prev;
    const int32_t* pos;
    void* x_store;
    // fused argmax (kEpiStore): the last CTA writes the first maximum of
    // every row of `out` to next[step * n + r], then advances the rollout
    // (*adv_step += 1, adv_qpos[0..n) += 1; either may be null)
    int32_t* next;
    int32_t* arrive;  // zero between launches
    int64_t* adv_qpos;
    int32_t* adv_step;
};

// Whether launch_dense runs the cluster GEMV for these arguments (the only
// kernel with the fused embedding / argmax).
bool dense_uses_gemv(const DenseArgs& a, bool ln);

// dt: EP_F64 or EP_F32 (x, W, bias, resid, out, q_out share it).
cudaError_t launch_dense(int dt, int epi, bool ln, const DenseArgs& a, cudaStream_t s);

// embed (model.cpp:104-129): out[r] = embedding[token] + sinusoid(pos). With
// a rollout step counter (step != null): token = tokens[r] at step 0, else
// prev[(step - 1) * n + r]; position pos[step * n + r].
cudaError_t launch_embed(int dt, const void* emb, const double* pe, const int32_t* tokens, const int32_t* prev,
                         const int32_t* step, const int32_t* pos, int n, int D, void* out,
                         cudaStream_t s);

// pe[p][c] = sin / cos(p * 10000^(-(c - c % 2) / D)) in fp64 (model.cpp:121-126).
cudaError_t launch_posenc(double* pe, int max_positions, int D, cudaStream_t s);

// Generic paged causal attention: one CTA per (query row, head); row r of
// request row_req[r] at position row_pos[r] (row_pos[step * n + r] in a
// rollout) attends to every key of that request's pages
// (pdesc[req_page_off[b]..]) at a position <= its own.
// q/out [n][H][dh] in dt (EP_F64/EP_F32); pages in kv_dtype.
cudaError_t launch_attention_generic(int dt, int kv_dtype, const void* q, int n, int H, int dh,
                                     const PageDesc* pdesc, const int64_t* req_page_off,
                                     const int32_t* row_req, const int32_t* row_pos,
                                     const int32_t* step, const void* k_pages,
                                     const void* v_pages, int P, void* out, cudaStream_t s);

// argmax_token (model.cpp:248-255) per row of logits [rows][V]: the first
// index of the maximum, into next[rows] (next[step * rows + r] in a rollout).
// Speculative verify's acceptance rule per request (model.cpp-built a16): the
// request's rows are [prev_last + 1, last_row[b]] (tokens [last, d1..dk]);
// n_accepted[b] = longest n with d_i == target[row_{i-1}] for all i <= n.
cudaError_t launch_accept_rows(const int32_t* tokens, const int32_t* targets, const int32_t* last_row, int batch,
                               int32_t* n_accepted, cudaStream_t s);
cudaError_t launch_argmax_rows(int dt, const void* logits, int rows, int V, const int32_t* step,
                               int32_t* next, cudaStream_t s);

// Rollout step end: *step += 1, q_pos[0..batch) += 1 (q_pos may be null).
cudaError_t launch_advance(int32_t* step, int64_t* q_pos, int batch, cudaStream_t s);

// K9: whole greedy rollout of a small fp32 decoder in one persistent
// cooperative kernel (kern_model_persist.cu).
struct PersistLayer {
    const float *wq, *wk, *wv, *wo, *w1, *b1, *w2, *b2;
    float *kp, *vp;  // this layer's K / V pages [page][H][P][dh]
};
struct PersistArgs {
    const PersistLayer* layers;  // device [L]
    int L, B, D, H, dh, F, V, P, n_steps, max_chunks;
    const float* emb;
    const double* pe;
    const float* unembed;
    const int32_t* first;      // [B] token of step 0
    const int32_t* pos;        // [n_steps][B]
    const int32_t* dst_page;   // [n_steps][B]
    const int32_t* dst_slot;   // [n_steps][B]
    const PageDesc* pdesc;     // every request's pages (final table)
    const int64_t* req_page_off;
    float *x, *x2, *q, *h1, *logits, *part, *att;  // scratch (att: merged attention rows [B][D])
    unsigned long long* keys;  // [n_ctas][B] per-CTA argmax candidates of the last unembedding
    int32_t* counters;         // [2 + B H]: grid barrier, unembedding, per-(row, head) attention arrivals (zeroed per launch)
    int32_t* out;              // [n_steps][B] greedy tokens
    unsigned long long* trace; // debug: [8 steps][32] barrier timestamps of CTA 0 (may be null)
    const float* image;        // every CTA's resident weight image (persist_image_floats, from launch_persist_image)
    float* image_out;          // launch_persist_image: where to build it
};
// n_ctas = n_sms: one CTA per SM; weights stay resident in shared memory
bool persist_supported(int L, int B, int D, int H, int F, int V, int P, int n_sms);
size_t persist_smem_bytes(int L, int B, int D, int F, int H, int V, int max_chunks, int n_sms);
// The resident weight images of n_ctas CTAs (layers / weights of a), built
// once per model and grid size; the rollout kernel bulk-copies its slice.
size_t persist_image_floats(int L, int D, int F, int V, int n_ctas);
cudaError_t launch_persist_image(const PersistArgs& a, int n_ctas, cudaStream_t s);
cudaError_t launch_decode_persist(const PersistArgs& a, int n_ctas, cudaStream_t s);


// dst[i] = uniform(lo, hi) of SplitMix64(seed) draw first + i (fp64 draw,
// stored in dt = EP_F64 / EP_F32 / EP_BF16).
cudaError_t launch_fill_uniform_at(int dt, void* dst, size_t n, uint64_t seed, uint64_t first,
                                   double lo, double hi, cudaStream_t s);

}  // namespace ep
