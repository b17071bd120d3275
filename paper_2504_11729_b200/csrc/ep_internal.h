// ep_internal.h — host-side internals of libep_b200.so (not part of the ABI).
#pragma once

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

#include "ep/ep_attn.h"

#define EP_CUDA_TRY(expr, where)                               \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return ep::cuda_fail(_e, where); \
    } while (0)

namespace ep {

// Sets the thread-local message returned by ep_last_error() and returns rc.
int fail(int rc, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

struct DeviceBuffer {
    void* ptr = nullptr;
    size_t bytes = 0;
    bool view = false;  // a slice of another buffer (a plan's arena): not freed here
    ~DeviceBuffer();
    cudaError_t reserve(size_t n);
};

}  // namespace ep

struct ep_context {
    int device = 0;
    int n_sms = 0;
    cudaStream_t stream = nullptr;  // used by the synchronous host-buffer entry points
    ep::DeviceBuffer scratch;       // staging for host-buffer calls
    void* pin = nullptr;            // pinned host staging of the host-buffer calls (one H2D + one D2H each)
    size_t pin_bytes = 0;
    ep::DeviceBuffer zero_rows;     // 64 zero rows of the widest KV row (page-tail fill)
    ep::DeviceBuffer ingest_stage;  // pageable / misaligned kv frames staged for ep_kv_ingest_frame
    cudaEvent_t ingest_done = nullptr;  // recorded after each launch that reads ingest_stage
    bool ingest_pending = false;        // ingest_done has been recorded at least once
    uint8_t* hdr_pinned = nullptr;  // pinned landing slot for a device kv frame's 24-byte header
    // deferred kv frame check (ep_kv_ingest_frame_async): device words
    // [0] = first failing kind (0 = none), [1..6] = that frame's header fields,
    // written by the kernels; ep_kv_ingest_poll reads them into the pinned copy
    int32_t* ingest_status = nullptr;
    int32_t* ingest_status_dev = nullptr;
    ep::DeviceBuffer scratch_status;  // backs ingest_status_dev
    std::atomic<int64_t> launches{0};
};

namespace ep {

// ---------------------------------------------------------- launchers --
// Each returns the launch status and counts launches into *counter.

cudaError_t launch_partial_generic(int dt, const void* q, size_t ldq, size_t n_q, const void* k,
                                   size_t ldk, const void* v, size_t ldv, size_t n_keys, size_t d,
                                   size_t q_off, size_t k_off, void* out, size_t ldo, void* lse,
                                   cudaStream_t s);

cudaError_t launch_merge_generic(int dt, size_t n_parts, const void* outs, const void* lses,
                                 size_t rows, size_t d, void* out, void* lse, cudaStream_t s);

cudaError_t launch_kv_append(int row_bytes, int n_kv_heads, int page_tokens, int n_rows,
                             const int32_t* dst_page, const int32_t* dst_slot, const void* k_new,
                             const void* v_new, void* k_pages, void* v_pages, cudaStream_t s,
                             int64_t num_pages = -1);

cudaError_t launch_merge_packed(int n_parts, const float* packed, int rows, int d, void* out,
                                int out_dtype, float* lse, cudaStream_t s);

cudaError_t launch_fill_uniform(int dt, void* dst, size_t n, uint64_t seed, double lo, double hi,
                                cudaStream_t s);

// Device-side descriptors of a spliced-decode plan (see plan.cpp).
struct PageDesc {
    int32_t page;   // page id in the pool
    int32_t n_tok;  // valid tokens (1..page_tokens)
    int64_t pos;    // absolute position of slot 0
};

struct WorkItem {
    int32_t b;     // (virtual) request whose page list the item walks
    int32_t g;     // kv head
    int32_t lp0;   // logical page range [lp0, lp1) of request b
    int32_t lp1;
    int32_t nblk;  // 64-token pipeline blocks in the range
    int32_t rq0;   // first real request of the item's query rows (K3 row groups)
    int32_t q0min; // smallest query position of those rows (all-visible fast path)
    int32_t pad;
};

// Fused split-KV combine (config 4): K1 on this rank's KV shard pushes every
// unit's merged (o, lse) rows into every rank's receive buffer over NVLink
// peer memory (kern_peer.cu's {value, flag} words), and each unit's owner CTA
// merges the W rank partials in rank order at the end of the kernel.
constexpr int kPeerMaxWorld = 8;
struct PeerLink {
    int32_t world = 0, rank = 0;        // world == 0: no exchange (plain decode)
    int64_t src_units = 0;              // 16-byte words per source slot: rows_max * (d/2 + 1)
    uint4* recv[kPeerMaxWorld] = {};    // rank p's receive area [2][world][src_units] (mapped here)
    uint32_t* epoch = nullptr;          // own per-unit step epochs
    const int32_t* cta_unit_ptr = nullptr;  // [n_ctas+1]: units whose final merge CTA c owns
};

struct DecodeArgs {
    const void* k_pages;
    const void* v_pages;
    int32_t n_kv_heads, n_q_heads, page_tokens, n_q;
    const PageDesc* pdesc;
    const int64_t* req_page_off;   // [batch+1]
    const WorkItem* items;
    const int32_t* cta_item_ptr;   // [n_ctas+1]
    const int32_t* cta_item_idx;   // K1: processing order of a CTA's items (split units first), null = in order
    const int32_t* unit_item_ptr;  // [batch*Hkv+1]
    const int64_t* q_pos;          // [batch]
    const void* q;
    int32_t q_dtype;
    float* o_part;    // [n_items][R][D]
    float* lse_part;  // [n_items][R] (log2 units)
    void* o;
    int32_t o_dtype;
    float* lse;       // natural log, may be null
    int32_t batch;
    float q_scale;            // log2(e) / sqrt(d)
    const void* zero_rows;    // >= 64 zero K/V rows (page-tail fill)
    int32_t* unit_counter;    // [batch*Hkv], zero between launches (fused K2)
    unsigned long long* trace;  // optional clock64 event trace of CTA 0 (debug, may be null)
    int32_t reqs_per_unit;    // K3: consecutive requests whose rows share one tile (cascade), else 1
    const int32_t* q_row0;    // per (virtual) request: first q/o token row; null = b * n_q (or chunks below)
    int32_t chunks;           // decode plans with more rows than K1 takes: each request's nq_total query
    int32_t nq_total;         // tokens cut into `chunks` virtual requests of n_q tokens (1 = not cut)
    int32_t pv_parts;         // K3: P as bf16 hi+lo (2) or bf16 (1)
    PeerLink peer;            // K1 fused split-KV combine (world 0 = off)
    int64_t num_pages;        // pool pages (checked build: page ids in range)
    int64_t n_q_rows;         // query / output token rows of the launch (checked build)
    int32_t n_items;          // work items of the sub-plan (checked build)
};

// The fused split-KV link of a peer group for a plan of n_units units and
// `rows` output rows of width d (kern_peer.cu); cta_unit_ptr is the plan's.
int peer_link_fill(ep_peer_group g, int64_t n_units, int64_t rows, int d, const int32_t* cta_unit_ptr,
                   PeerLink* out);

// Validates request b's segments of a host splice table with the
// SegmentedCache invariants (cache.cpp:25-53: gapless positions, origin
// order, pages inside the pool) and appends its page descriptors to out;
// *first_pages = descriptors of its first segment (plan.cpp).
int collect_request_pages(int page_tokens, int64_t num_pages, int b, const int64_t* seg_indptr,
                          const ep_segment* segs, const int32_t* page_table, std::vector<PageDesc>& out,
                          int64_t* first_pages);

// Per-token growth of a plan in place on the device (the fast path of
// ep_plan_update_cache): desc[idx[i]].n_tok = ntok[i], q_pos[req[i]] = qpos[i]
// for n entries, in one small kernel launch instead of a staged H2D copy.
constexpr int kPlanPatchMax = 128;
struct PlanPatch {
    PageDesc* pdesc;
    int64_t* q_pos;
    int32_t n;
    int32_t idx[kPlanPatchMax];
    int32_t ntok[kPlanPatchMax];
    int32_t req[kPlanPatchMax];
    int64_t qpos[kPlanPatchMax];
};
cudaError_t launch_plan_patch(const PlanPatch& pp, cudaStream_t s);

// ep_cache <-> plan: the plan remembers which cache (and structure version,
// layer) it was last fully built from; plan_grow_in_place then follows pure
// in-page growth of every request to ends[b] (query rows end - n_q) with an
// O(batch) page-descriptor refresh and one staged upload. Returns 1 applied,
// 0 a full rebuild is needed, < 0 an error (negated status).
void plan_mark_built(ep_plan p, const void* cache, uint64_t version, int layer);
int plan_grow_in_place(ep_plan p, const void* cache, uint64_t version, int layer, const int64_t* ends, int n_q,
                       cudaStream_t s);

// Device copy of a plan's per-request query positions (a device-resident
// rollout advances them in place, one token per step).
int64_t* plan_qpos_dev(ep_plan p);

// First q/o token row of (virtual) request b: prefill plans cut one request's
// queries into chunks that are separate virtual requests.
__host__ __device__ inline size_t q_row_base(const DecodeArgs& a, int b) {
    if (a.q_row0) return size_t(a.q_row0[b]);
    if (a.chunks > 1) return size_t(b / a.chunks) * a.nq_total + size_t(b % a.chunks) * a.n_q;
    return size_t(b) * a.n_q;
}

// Valid query rows (group * tokens) of (virtual) request b of a decode plan.
__host__ __device__ inline int valid_rows(const DecodeArgs& a, int b) {
    const int G = a.n_q_heads / a.n_kv_heads;
    if (a.chunks > 1) {
        const int left = a.nq_total - (b % a.chunks) * a.n_q;
        return G * (left < a.n_q ? left : a.n_q);
    }
    return G * a.n_q;
}

// TMA tensor maps over bf16 row-major matrices (capi.cpp).
int encode_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint32_t box_inner, uint32_t box_outer);
int encode_kv_map(CUtensorMap* map, const void* base, int64_t rows);
bool force_tc();

// Cascade (shared-prefix) merge: per row, LSE-merge the shared-pass partial
// (part 0, only where has_shared[request]) with the private-pass partial.
cudaError_t launch_cascade_merge(int rows, int d, int row_per_req, const float* o_parts,
                                 const float* lse_parts, const uint8_t* has_shared, void* o,
                                 int o_dtype, float* lse, cudaStream_t s);

// R = rows per (request, kv-head) = group * n_q; K1 pads it to a power of two.
bool decode_supported(int kv_dtype, int d_head, int rows);
// Any f32 / bf16 shape with d_head <= 256 (the generic kernel behind K1 / K3).
bool generic_supported(int kv_dtype, int d_head);
cudaError_t launch_generic_decode(int kv_dtype, int d_head, int batch, int n_q, const DecodeArgs& a,
                                  cudaStream_t s);
int decode_ctas_per_sm(int kv_dtype, int d_head, int rows);
cudaError_t launch_spliced_decode(int kv_dtype, int d_head, int rows, int n_ctas,
                                  const DecodeArgs& a, cudaStream_t s);
cudaError_t launch_empty_units(int d_head, int rows, const DecodeArgs& a, cudaStream_t s);

// K3: tcgen05 multi-row (verify) attention; bf16 KV, d_head 128, rows <= 64.
bool verify_supported(int kv_dtype, int d_head, int rows);
cudaError_t launch_verify_attention(int n_ctas, const DecodeArgs& a, const CUtensorMap& tk,
                                    const CUtensorMap& tv, int rows, cudaStream_t s);

// K4: score GEMM (tcgen05) + LN-folded argmax + greedy accept.
cudaError_t launch_colsum(const void* wt, int width, int vocab, float* colsum, float* wmax2, cudaStream_t s);
// fp32 attention rows: hi-only GEMM + exact refinement of the candidates
// within the per-row error bound (kern_score.cu).
constexpr int kScoreTileNMax = 256;    // vocabulary columns per K4 score tile, at most (one TMEM accumulator)
constexpr int kScoreCandPerTile = 16;  // candidate slots per (row, vocab tile)
// K4 tile width for `rows` score rows: one wave of CTAs (or CTA pairs) over
// n_sms SMs; rows of the W tensor-map box for that width.
constexpr int kScoreStreamK = 0, kScorePair = 1, kScoreOneSm = 2;
int score_mode();
int score_tile_n(int rows, int vocab, int n_sms);
int score_w_box_rows(int tn);
int score_cand_tiles(int vocab, int tn);
size_t score_streamk_ws_bytes(int n_sms);
struct RefineArgs {
    const void* wt = nullptr;      // W^T bf16 [vocab][width]
    const float* wmax2 = nullptr;  // max_n ||W^T[n]||_2
    float* ebound = nullptr;       // [rows]
    int32_t* cand_cnt = nullptr;   // [rows][vocab / 256]
    int32_t* cand_n = nullptr;     // [rows][vocab tiles][kScoreCandPerTile]
    float* cand_z = nullptr;       // [rows][vocab tiles][kScoreCandPerTile]
    int32_t* req_count = nullptr;  // [batch] row arrivals of the fused accept, zero between launches
    float* sk_ws = nullptr;        // stream-K GEMM: [sk_ctas] fp32 partial tiles (score_streamk_ws_bytes)
    unsigned int* sk_flags = nullptr;  // [sk_ctas], zero between launches
    int sk_ctas = 0;
};
cudaError_t launch_score_accept(int rows, int width, int vocab, int tn, const void* attn_out, void* split,
                                const CUtensorMap& tmap_a, const CUtensorMap& tmap_w,
                                const float* colsum, float* mean, float* rstd,
                                unsigned long long* best, float* logits, int batch, int n_q,
                                const int32_t* drafts, int32_t* target, int32_t* n_accepted,
                                const RefineArgs& rf, cudaStream_t s);

}  // namespace ep
