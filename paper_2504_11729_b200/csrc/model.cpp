// model.cpp — include/ep/ep_model.h: the decoder around the spliced attention
// on the GPU.
//
// The reference (/root/reference/proj/core/src/model.cpp) keeps fp64 weights
// in host Matrix objects and runs, per new token row, embed -> L x
// transformer_layer -> unembed_logits -> argmax_token, with the attention of
// each layer as one partial_attention per cached segment (+ the new tokens)
// fused by merge_partials. Here:
//   * weights live in one device allocation in generation order, each tensor
//     256-byte aligned and filled from its own range of the one SplitMix64
//     stream (init_model's draw order);
//   * every layer has a KV page pool with the same page numbering, so one
//     host splice table addresses all layers;
//   * a forward pass is a fixed launch sequence per layer — QKV (LN fused,
//     K/V rows scattered into their pages), spliced attention (the K1/K3 plans
//     of plan.cpp, or the generic paged kernel for fp64 / other head sizes),
//     Wo + residual, LN + W1 + ReLU, W2 + residual — then the unembedding of
//     each request's last row and argmax.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "ep/ep_model.h"
#include "model_internal.h"

using namespace ep;

namespace {

struct LayerOffsets {
    size_t wq, wk, wv, wo, w1, b1, w2, b2;
};

}  // namespace

struct ep_model_s {
    ep_handle h = nullptr;
    ep_model_config cfg{};
    int dt = EP_F64, kv_dtype = EP_F64, P = 64;
    int64_t num_pages = 0;
    int D = 0, H = 0, dh = 0, V = 0, L = 0, F = 0;
    size_t n_weights = 0, off_unembed = 0;
    std::vector<LayerOffsets> lw;
    DeviceBuffer weights;
    DeviceBuffer pe;      // sinusoid table [max_positions][d_model] fp64 (model.cpp:121-126)
    DeviceBuffer persist_layers, persist_scratch, persist_counters;  // K9 persistent rollout (fp32 models)
    DeviceBuffer persist_image;  // K9 resident weight images (persist_image_ctas CTAs)
    int persist_image_ctas = 0;
    DeviceBuffer arrive;  // fused-argmax arrival counter (zero between launches)
    std::vector<std::unique_ptr<DeviceBuffer>> kpages, vpages;
    // per-forward workspace
    DeviceBuffer hid, xbuf, qbuf, attn, h1, logits_ws, next_ws, meta;
    void* stage = nullptr;
    size_t stage_bytes = 0;
    cudaEvent_t staged = nullptr;
    ep_plan decode_plan = nullptr;
    int32_t decode_plan_batch = -1;
    ep_plan prefill_plan = nullptr;
    int last_path = 0;

    size_t esz() const { return dt == EP_F64 ? 8 : 4; }
    char* wptr(size_t off) const { return static_cast<char*>(weights.ptr) + off * esz(); }
    ep_kv_pool pool(int l) const {
        ep_kv_pool p{};
        p.dtype = kv_dtype;
        p.n_kv_heads = H;
        p.d_head = dh;
        p.page_tokens = P;
        p.num_pages = num_pages;
        p.k_pages = kpages[l]->ptr;
        p.v_pages = vpages[l]->ptr;
        return p;
    }
    ~ep_model_s() {
        if (decode_plan) ep_plan_destroy(decode_plan);
        if (prefill_plan) ep_plan_destroy(prefill_plan);
        if (stage) cudaFreeHost(stage);
        if (staged) cudaEventDestroy(staged);
    }
};

namespace {

size_t kv_elem_bytes(int kv) { return kv == EP_F64 ? 8 : kv == EP_F32 ? 4 : 2; }

// Host-side row metadata of one forward (or rollout), uploaded in one copy.
struct Meta {
    std::vector<int32_t> tokens, pos, dst_page, dst_slot, row_req, last_row, step;
    std::vector<int64_t> req_page_off, q_pos;
    std::vector<PageDesc> pdesc;
};

// One request of a forward: its validated page descriptors and the page
// slots of its last nn positions (the new tokens).
struct Req {
    std::vector<PageDesc> pages;
    int64_t start = 0, end = 0;
    int nn = 0;
    std::vector<std::pair<int32_t, int32_t>> slots;
};

template <typename T>
size_t append_bytes(std::vector<char>& blob, const std::vector<T>& v) {
    const size_t off = (blob.size() + 255) & ~size_t(255);
    blob.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
}

}  // namespace

namespace {

bool uses_plans(ep_model m) {
    return m->dt == EP_F32 && (m->dh == 64 || m->dh == 128) && m->P % 64 == 0;
}

// Validates every request's splice table (SegmentedCache invariants via
// collect_request_pages) and locates the page slot of each new position.
int collect_requests(ep_model m, int batch, const int64_t* seg_indptr, const ep_segment* segs,
                     const int32_t* page_table, const int32_t* n_new, std::vector<Req>& reqs, bool* all_decode) {
    if (seg_indptr[0] != 0) return fail(EP_EINVAL, "ep_model: seg_indptr[0] must be 0");
    reqs.assign(batch, Req{});
    *all_decode = true;
    for (int b = 0; b < batch; ++b) {
        Req& r = reqs[b];
        int64_t first = 0;
        if (int rc = collect_request_pages(m->P, m->num_pages, b, seg_indptr, segs, page_table, r.pages, &first))
            return rc;
        r.start = r.pages.empty() ? 0 : r.pages.front().pos;
        r.end = r.pages.empty() ? 0 : r.pages.back().pos + r.pages.back().n_tok;
        r.nn = n_new[b];
        if (r.nn <= 0 || r.nn > r.end - r.start)
            return fail(EP_EINVAL, "ep_model: request " + std::to_string(b) + " has " +
                                       std::to_string(r.end - r.start) + " tokens, n_new = " + std::to_string(r.nn));
        if (r.end > m->cfg.max_positions)  // embed's std::out_of_range (model.cpp:107-112)
            return fail(EP_EINVAL, "embed: positions " + std::to_string(r.end - r.nn) + ".." +
                                       std::to_string(r.end) + " overflow max_positions " +
                                       std::to_string(m->cfg.max_positions));
        *all_decode = *all_decode && r.nn == 1;
        // new positions [end - nn, end): walk the descriptors from the back
        r.slots.resize(r.nn);
        size_t di = r.pages.size();
        for (int64_t p = r.end - 1; p >= r.end - r.nn; --p) {
            while (di > 0 && r.pages[di - 1].pos > p) --di;
            const PageDesc& d = r.pages[di - 1];
            r.slots[p - (r.end - r.nn)] = {d.page, int32_t(p - d.pos)};
        }
    }
    return EP_OK;
}

int reserve_ws(ep_model m, int n, int batch) {
    const size_t es = m->esz();
    EP_CUDA_TRY(m->hid.reserve(size_t(n) * m->D * es), "ep_model ws");
    EP_CUDA_TRY(m->xbuf.reserve(size_t(n) * m->D * es), "ep_model ws");
    EP_CUDA_TRY(m->qbuf.reserve(size_t(n) * m->D * es), "ep_model ws");
    EP_CUDA_TRY(m->attn.reserve(size_t(n) * m->D * es), "ep_model ws");
    EP_CUDA_TRY(m->h1.reserve(size_t(n) * m->F * es), "ep_model ws");
    // (verify unembeds every row: n >= batch rows of logits / next ids)
    EP_CUDA_TRY(m->logits_ws.reserve(size_t(std::max(n, batch)) * m->V * es), "ep_model ws");
    EP_CUDA_TRY(m->next_ws.reserve(size_t(std::max(n, batch)) * sizeof(int32_t)), "ep_model ws");
    return EP_OK;
}

// forward declaration (defined below)
struct Pass;
int upload_meta(ep_model m, const Meta& md, Pass& ps, cudaStream_t s);

// One forward pass over n token rows of `batch` requests (device metadata
// already uploaded). step != null: a rollout step — row metadata is indexed
// by the device step counter and the step's tokens come from the previous
// step's argmax (see ep_model_generate).
struct Pass {
    int n = 0, batch = 0;
    const int32_t *tok = nullptr, *prev = nullptr, *step = nullptr, *pos = nullptr;
    const int32_t *dst_page = nullptr, *dst_slot = nullptr, *row_req = nullptr, *last_row = nullptr;
    const int64_t* req_page_off = nullptr;
    const PageDesc* pdesc = nullptr;
    ep_plan plan = nullptr;
    void* logits = nullptr;
    int32_t* next = nullptr;
    bool advance = false;       // rollout: step += 1, adv_qpos[0..batch) += 1 after the argmax
    int64_t* adv_qpos = nullptr;
    bool all_rows = false;      // verify: unembed + argmax every new row (logits [n][V], next [n])
};

// Metadata upload: one pinned staging buffer, one async copy; fills the
// device pointers of ps.
int upload_meta(ep_model m, const Meta& md, Pass& ps, cudaStream_t s) {
    std::vector<char> blob;
    const size_t o_tok = append_bytes(blob, md.tokens), o_pos = append_bytes(blob, md.pos),
                 o_pg = append_bytes(blob, md.dst_page), o_sl = append_bytes(blob, md.dst_slot),
                 o_rq = append_bytes(blob, md.row_req), o_last = append_bytes(blob, md.last_row),
                 o_rpo = append_bytes(blob, md.req_page_off), o_pd = append_bytes(blob, md.pdesc),
                 o_st = append_bytes(blob, md.step);
    EP_CUDA_TRY(m->meta.reserve(blob.size()), "ep_model meta");
    EP_CUDA_TRY(cudaEventSynchronize(m->staged), "ep_model staging");
    if (blob.size() > m->stage_bytes) {
        if (m->stage) cudaFreeHost(m->stage);
        m->stage = nullptr;
        EP_CUDA_TRY(cudaMallocHost(&m->stage, blob.size()), "ep_model pinned");
        m->stage_bytes = blob.size();
    }
    std::memcpy(m->stage, blob.data(), blob.size());
    EP_CUDA_TRY(cudaMemcpyAsync(m->meta.ptr, m->stage, blob.size(), cudaMemcpyHostToDevice, s), "ep_model meta copy");
    EP_CUDA_TRY(cudaEventRecord(m->staged, s), "ep_model event");
    char* mb = static_cast<char*>(m->meta.ptr);
    ps.tok = reinterpret_cast<const int32_t*>(mb + o_tok);
    ps.pos = reinterpret_cast<const int32_t*>(mb + o_pos);
    ps.dst_page = reinterpret_cast<const int32_t*>(mb + o_pg);
    ps.dst_slot = reinterpret_cast<const int32_t*>(mb + o_sl);
    ps.row_req = reinterpret_cast<const int32_t*>(mb + o_rq);
    ps.last_row = reinterpret_cast<const int32_t*>(mb + o_last);
    ps.req_page_off = reinterpret_cast<const int64_t*>(mb + o_rpo);
    ps.pdesc = reinterpret_cast<const PageDesc*>(mb + o_pd);
    ps.step = md.step.empty() ? nullptr : reinterpret_cast<const int32_t*>(mb + o_st);
    return EP_OK;
}

int enqueue_pass(ep_model m, const Pass& ps, cudaStream_t s) {
    ep_handle h = m->h;
    const int dt = m->dt, n = ps.n;
    bool embed_fused = false;
    for (int l = 0; l < m->L; ++l) {
        const LayerOffsets& o = m->lw[l];
        const ep_kv_pool pool = m->pool(l);
        // LN -> Q | K | V; K/V rows scattered into their page slots
        DenseArgs a{};
        a.x = m->hid.ptr;
        a.n = n;
        a.K = m->D;
        a.N = 3 * m->D;
        a.w[0] = m->wptr(o.wq);
        a.w[1] = m->wptr(o.wk);
        a.w[2] = m->wptr(o.wv);
        a.n_wblk = 3;
        a.q_out = m->qbuf.ptr;
        a.k_pages = pool.k_pages;
        a.v_pages = pool.v_pages;
        a.kv_dtype = m->kv_dtype;
        a.H = m->H;
        a.P = m->P;
        a.dh = m->dh;
        a.dst_page = ps.dst_page;
        a.dst_slot = ps.dst_slot;
        a.step = ps.step;
        if (l == 0) {
            // embed (model.cpp:104-129) fused into the first projection's
            // LayerNorm prologue, which also stores the embedded rows
            embed_fused = dense_uses_gemv(a, true);
            if (embed_fused) {
                a.emb = m->wptr(0);
                a.pe = static_cast<const double*>(m->pe.ptr);
                a.tok = ps.tok;
                a.tok_prev = ps.prev;
                a.pos = ps.pos;
                a.x_store = m->hid.ptr;
            } else {
                EP_CUDA_TRY(launch_embed(dt, m->wptr(0), static_cast<const double*>(m->pe.ptr), ps.tok, ps.prev,
                                         ps.step, ps.pos, n, m->D, m->hid.ptr, s),
                            "embed launch");
                h->launches++;
            }
        }
        EP_CUDA_TRY(launch_dense(dt, kEpiQKV, true, a, s), "qkv launch");
        h->launches++;
        // spliced causal attention over the request's pages
        if (ps.plan) {
            if (int rc = ep_spliced_attention(h, ps.plan, &pool, EP_F32, m->qbuf.ptr, EP_F32, m->attn.ptr,
                                              nullptr, s))
                return rc;
        } else {
            EP_CUDA_TRY(launch_attention_generic(dt, m->kv_dtype, m->qbuf.ptr, n, m->H, m->dh, ps.pdesc,
                                                 ps.req_page_off, ps.row_req, ps.pos, ps.step, pool.k_pages,
                                                 pool.v_pages, m->P, m->attn.ptr, s),
                        "attention launch");
            h->launches++;
        }
        // x = hidden + attn @ Wo
        DenseArgs b{};
        b.x = m->attn.ptr;
        b.n = n;
        b.K = m->D;
        b.N = m->D;
        b.w[0] = m->wptr(o.wo);
        b.n_wblk = 1;
        b.resid = m->hid.ptr;
        b.out = m->xbuf.ptr;
        EP_CUDA_TRY(launch_dense(dt, kEpiResid, false, b, s), "wo launch");
        h->launches++;
        // h1 = relu(LN(x) @ W1 + b1)
        DenseArgs c{};
        c.x = m->xbuf.ptr;
        c.n = n;
        c.K = m->D;
        c.N = m->F;
        c.w[0] = m->wptr(o.w1);
        c.n_wblk = 1;
        c.bias = m->wptr(o.b1);
        c.out = m->h1.ptr;
        EP_CUDA_TRY(launch_dense(dt, kEpiRelu, true, c, s), "w1 launch");
        h->launches++;
        // hidden = x + h1 @ W2 + b2
        DenseArgs d{};
        d.x = m->h1.ptr;
        d.n = n;
        d.K = m->F;
        d.N = m->D;
        d.w[0] = m->wptr(o.w2);
        d.n_wblk = 1;
        d.bias = m->wptr(o.b2);
        d.resid = m->xbuf.ptr;
        d.out = m->hid.ptr;
        EP_CUDA_TRY(launch_dense(dt, kEpiResid, false, d, s), "w2 launch");
        h->launches++;
    }
    // unembed_logits of each request's last row (model.cpp:238-246) + argmax
    DenseArgs u{};
    u.x = m->hid.ptr;
    u.row_map = ps.all_rows ? nullptr : ps.last_row;
    u.n = ps.all_rows ? ps.n : ps.batch;
    u.K = m->D;
    u.N = m->V;
    u.w[0] = m->wptr(m->off_unembed);
    u.n_wblk = 1;
    u.out = ps.logits;
    u.step = ps.step;
    if (dense_uses_gemv(u, true)) {
        // argmax_token (+ the rollout's position advance) in the last CTA
        u.next = ps.next;
        u.arrive = static_cast<int32_t*>(m->arrive.ptr);
        if (ps.advance) {
            u.adv_step = const_cast<int32_t*>(ps.step);
            u.adv_qpos = ps.adv_qpos;
        }
        EP_CUDA_TRY(launch_dense(dt, kEpiStore, true, u, s), "unembed launch");
        h->launches++;
        return EP_OK;
    }
    EP_CUDA_TRY(launch_dense(dt, kEpiStore, true, u, s), "unembed launch");
    h->launches++;
    EP_CUDA_TRY(launch_argmax_rows(dt, ps.logits, u.n, m->V, ps.step, ps.next, s), "argmax launch");
    h->launches++;
    if (ps.advance) {
        EP_CUDA_TRY(launch_advance(const_cast<int32_t*>(ps.step), ps.adv_qpos, ps.batch, s), "advance launch");
        h->launches++;
    }
    return EP_OK;
}

}  // namespace

extern "C" {

int ep_model_create(ep_handle h, const ep_model_config* cfg, int32_t kv_dtype, int32_t page_tokens,
                    int64_t num_pages, ep_model* out) {
    if (!h || !cfg || !out) return fail(EP_EINVAL, "ep_model_create: null argument");
    *out = nullptr;
    const ep_model_config& c = *cfg;
    // ModelConfig::validate (model.cpp:42-50)
    if (c.n_layers <= 0 || c.n_heads <= 0 || c.d_model <= 0 || c.vocab_size <= 0 || c.max_positions <= 0)
        return fail(EP_EINVAL, "ModelConfig: all dimensions must be positive");
    if (c.d_model % c.n_heads != 0)
        return fail(EP_EINVAL, "ModelConfig: d_model " + std::to_string(c.d_model) +
                                   " not divisible by n_heads " + std::to_string(c.n_heads));
    if (c.dtype != EP_F64 && c.dtype != EP_F32)
        return fail(EP_EUNSUPPORTED, "ep_model_create: model dtype must be EP_F64 or EP_F32");
    if (c.dtype == EP_F64 ? kv_dtype != EP_F64 : (kv_dtype != EP_F32 && kv_dtype != EP_BF16))
        return fail(EP_EUNSUPPORTED, "ep_model_create: kv dtype must be EP_F64 for an fp64 model, "
                                     "EP_F32 or EP_BF16 for an fp32 model");
    if (c.d_model / c.n_heads > 256)
        return fail(EP_EUNSUPPORTED, "ep_model_create: d_head > 256");
    if (page_tokens <= 0 || num_pages <= 0) return fail(EP_EINVAL, "ep_model_create: page_tokens / num_pages");

    std::unique_ptr<ep_model_s> m(new (std::nothrow) ep_model_s());
    if (!m) return fail(EP_ENOMEM, "ep_model_create");
    m->h = h;
    m->cfg = c;
    m->dt = c.dtype;
    m->kv_dtype = kv_dtype;
    m->P = page_tokens;
    m->num_pages = num_pages;
    m->D = c.d_model;
    m->H = c.n_heads;
    m->dh = c.d_model / c.n_heads;
    m->V = c.vocab_size;
    m->L = c.n_layers;
    m->F = 4 * c.d_model;
    // Tensors in generation order of init_model (model.cpp:82-102); each
    // starts 256-byte aligned (16-byte vector loads) and is filled with its
    // own range of the single SplitMix64 stream (draw index != storage index).
    const size_t D = size_t(m->D), V = size_t(m->V), F = size_t(m->F);
    struct Fill {
        size_t store, draw, count;
    };
    std::vector<Fill> fills;
    size_t store = 0, draw = 0;
    auto place = [&](size_t count) {
        const size_t at = store;
        fills.push_back({at, draw, count});
        draw += count;
        store = (store + count + 31) & ~size_t(31);
        return at;
    };
    place(V * D);  // embedding [V][D] at 0
    m->lw.resize(m->L);
    for (LayerOffsets& o : m->lw) {
        o.wq = place(D * D);
        o.wk = place(D * D);
        o.wv = place(D * D);
        o.wo = place(D * D);
        o.w1 = place(D * F);
        o.b1 = place(F);
        o.w2 = place(F * D);
        o.b2 = place(D);
    }
    m->off_unembed = place(D * V);
    m->n_weights = draw;

    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_model_create");
    EP_CUDA_TRY(m->weights.reserve(store * m->esz()), "ep_model_create weights");
    for (const Fill& f : fills) {
        EP_CUDA_TRY(launch_fill_uniform_at(m->dt, m->wptr(f.store), f.count, c.init_seed, f.draw, -0.1, 0.1,
                                           nullptr),
                    "ep_model_create init");
        h->launches++;
    }
    EP_CUDA_TRY(m->pe.reserve(size_t(c.max_positions) * D * sizeof(double)), "ep_model_create pe");
    EP_CUDA_TRY(launch_posenc(static_cast<double*>(m->pe.ptr), c.max_positions, m->D, nullptr), "posenc launch");
    h->launches++;
    EP_CUDA_TRY(m->arrive.reserve(sizeof(int32_t)), "ep_model_create");
    EP_CUDA_TRY(cudaMemset(m->arrive.ptr, 0, sizeof(int32_t)), "ep_model_create");
    const size_t pool_bytes = size_t(num_pages) * m->H * size_t(page_tokens) * m->dh * kv_elem_bytes(kv_dtype);
    for (int l = 0; l < m->L; ++l) {
        m->kpages.emplace_back(new DeviceBuffer());
        m->vpages.emplace_back(new DeviceBuffer());
        EP_CUDA_TRY(m->kpages.back()->reserve(pool_bytes), "ep_model_create kv pool");
        EP_CUDA_TRY(m->vpages.back()->reserve(pool_bytes), "ep_model_create kv pool");
        EP_CUDA_TRY(cudaMemset(m->kpages.back()->ptr, 0, pool_bytes), "ep_model_create kv pool");
        EP_CUDA_TRY(cudaMemset(m->vpages.back()->ptr, 0, pool_bytes), "ep_model_create kv pool");
    }
    EP_CUDA_TRY(cudaEventCreateWithFlags(&m->staged, cudaEventDisableTiming), "ep_model_create event");
    EP_CUDA_TRY(cudaDeviceSynchronize(), "ep_model_create");
    *out = m.release();
    return EP_OK;
}

int ep_model_destroy(ep_model m) {
    if (m) {
        cudaSetDevice(m->h->device);
        cudaDeviceSynchronize();
        delete m;
    }
    return EP_OK;
}

int ep_model_weight_sum(ep_model m, double* out) {
    if (!m || !out) return fail(EP_EINVAL, "ep_model_weight_sum: null argument");
    EP_CUDA_TRY(cudaSetDevice(m->h->device), "ep_model_weight_sum");
    // the fp64 draws of the whole stream, contiguous in generation order
    DeviceBuffer tmp;
    EP_CUDA_TRY(tmp.reserve(m->n_weights * sizeof(double)), "ep_model_weight_sum");
    EP_CUDA_TRY(launch_fill_uniform_at(EP_F64, tmp.ptr, m->n_weights, m->cfg.init_seed, 0, -0.1, 0.1, nullptr),
                "ep_model_weight_sum");
    m->h->launches++;
    std::vector<double> w(m->n_weights);
    EP_CUDA_TRY(cudaMemcpy(w.data(), tmp.ptr, w.size() * sizeof(double), cudaMemcpyDeviceToHost),
                "ep_model_weight_sum copy");
    // Model::weight_sum (model.cpp:52-67) adds in generation order
    double sum = 0.0;
    for (double v : w) sum += v;
    *out = sum;
    return EP_OK;
}

int ep_model_kv_pool(ep_model m, int32_t layer, ep_kv_pool* out) {
    if (!m || !out) return fail(EP_EINVAL, "ep_model_kv_pool: null argument");
    if (layer < 0 || layer >= m->L) return fail(EP_EINVAL, "ep_model_kv_pool: bad layer index");
    *out = m->pool(layer);
    return EP_OK;
}

int ep_model_weight(ep_model m, const char* name, int32_t layer, void** ptr, size_t* count) {
    if (!m || !name || !ptr || !count) return fail(EP_EINVAL, "ep_model_weight: null argument");
    const size_t D = size_t(m->D), V = size_t(m->V), F = size_t(m->F);
    const std::string n(name);
    if (n == "embedding") {
        *ptr = m->wptr(0);
        *count = V * D;
        return EP_OK;
    }
    if (n == "unembed") {
        *ptr = m->wptr(m->off_unembed);
        *count = D * V;
        return EP_OK;
    }
    if (layer < 0 || layer >= m->L) return fail(EP_EINVAL, "ep_model_weight: bad layer index");
    const LayerOffsets& o = m->lw[layer];
    struct {
        const char* name;
        size_t off, count;
    } table[] = {{"wq", o.wq, D * D}, {"wk", o.wk, D * D}, {"wv", o.wv, D * D}, {"wo", o.wo, D * D},
                 {"w1", o.w1, D * F}, {"b1", o.b1, F},     {"w2", o.w2, F * D}, {"b2", o.b2, D}};
    for (const auto& t : table) {
        if (n == t.name) {
            *ptr = m->wptr(t.off);
            *count = t.count;
            return EP_OK;
        }
    }
    return fail(EP_EINVAL, "ep_model_weight: unknown tensor " + n);
}

int ep_model_last_attention_path(ep_model m) { return m ? m->last_path : 0; }

// K9: whether decode rows of this batch run in the persistent cooperative
// kernel — every decode of up to 8 sessions of a small fp32 model (config 1
// rollout: 47 / 55 / 64 us per step at batch 1 / 4 / 8 vs 64 / 64 / 70 on the
// CUDA-graph path). EP_MODEL_PERSIST=0 keeps the layer-by-layer path.
bool use_persist(ep_model m, int batch, int* n_ctas) {
    const char* e = std::getenv("EP_MODEL_PERSIST");
    if (e && e[0] == '0') return false;
    if (m->dt != EP_F32 || m->kv_dtype != EP_F32) return false;
    int c = m->h->n_sms;  // one CTA per SM (EP_PERSIST_CTAS: fewer)
    if (const char* ec = std::getenv("EP_PERSIST_CTAS")) c = std::max(1, std::min(m->h->n_sms, std::atoi(ec)));
    *n_ctas = c;
    return persist_supported(m->L, batch, m->D, m->H, m->F, m->V, m->P, c);
}

// n_steps greedy steps of `batch` decode rows in one K9 launch: ps holds the
// uploaded step-major metadata (token of step 0, pos / dst_page / dst_slot
// [n_steps][batch]) and every request's final page table; tokens -> out
// [n_steps][batch] (device), the last step's logits -> logits_out (device
// fp32 [batch][V], may be null).
int run_persist(ep_model m, const std::vector<Req>& reqs, const Pass& ps, int batch, int n_steps,
                int persist_ctas, int32_t* out, void* logits_out, cudaStream_t s) {
    if (!m->persist_layers.ptr) {
        std::vector<PersistLayer> tab(m->L);
        for (int l = 0; l < m->L; ++l) {
            const LayerOffsets& o = m->lw[l];
            tab[l] = {reinterpret_cast<const float*>(m->wptr(o.wq)), reinterpret_cast<const float*>(m->wptr(o.wk)),
                      reinterpret_cast<const float*>(m->wptr(o.wv)), reinterpret_cast<const float*>(m->wptr(o.wo)),
                      reinterpret_cast<const float*>(m->wptr(o.w1)), reinterpret_cast<const float*>(m->wptr(o.b1)),
                      reinterpret_cast<const float*>(m->wptr(o.w2)), reinterpret_cast<const float*>(m->wptr(o.b2)),
                      static_cast<float*>(m->kpages[l]->ptr), static_cast<float*>(m->vpages[l]->ptr)};
        }
        EP_CUDA_TRY(m->persist_layers.reserve(tab.size() * sizeof(PersistLayer)), "ep_model_generate");
        EP_CUDA_TRY(cudaMemcpy(m->persist_layers.ptr, tab.data(), tab.size() * sizeof(PersistLayer),
                               cudaMemcpyHostToDevice),
                    "ep_model_generate");
    }
    int max_chunks = 1;
    for (const Req& r : reqs) max_chunks = std::max<int>(max_chunks, int(r.pages.size()));
    const size_t B = size_t(batch), D = size_t(m->D), F = size_t(m->F), V = size_t(m->V);
    const size_t part = B * m->H * size_t(2 * max_chunks) * (m->dh + 2);  // 32-key halves
    // scratch blocks x | x2 | q | h1 | logits | part | att, each 256-byte
    // aligned (the kernel reads rows with 16-byte loads)
    auto al = [](size_t n) { return (n + 63) & ~size_t(63); };
    const size_t o_x2 = al(B * D), o_q = o_x2 + al(B * D), o_h1 = o_q + al(B * D), o_lg = o_h1 + al(B * F),
                 o_part = o_lg + al(B * V), o_att = o_part + al(part);
    const size_t o_keys = o_att + al(B * D);
    const size_t floats = o_keys + al(2 * B * size_t(persist_ctas));
    EP_CUDA_TRY(m->persist_scratch.reserve(floats * sizeof(float)), "ep_model_generate scratch");
    EP_CUDA_TRY(m->persist_counters.reserve((2 + B * m->H) * sizeof(int32_t)), "ep_model_generate counters");
    float* f0 = static_cast<float*>(m->persist_scratch.ptr);
    PersistArgs pa{};
    pa.layers = static_cast<const PersistLayer*>(m->persist_layers.ptr);
    pa.L = m->L;
    pa.B = batch;
    pa.D = m->D;
    pa.H = m->H;
    pa.dh = m->dh;
    pa.F = m->F;
    pa.V = m->V;
    pa.P = m->P;
    pa.n_steps = n_steps;
    pa.max_chunks = max_chunks;
    pa.emb = reinterpret_cast<const float*>(m->wptr(0));
    pa.pe = static_cast<const double*>(m->pe.ptr);
    pa.unembed = reinterpret_cast<const float*>(m->wptr(m->off_unembed));
    pa.first = ps.tok;
    pa.pos = ps.pos;
    pa.dst_page = ps.dst_page;
    pa.dst_slot = ps.dst_slot;
    pa.pdesc = ps.pdesc;
    pa.req_page_off = ps.req_page_off;
    pa.x = f0;
    pa.x2 = f0 + o_x2;
    pa.q = f0 + o_q;
    pa.h1 = f0 + o_h1;
    pa.logits = logits_out ? static_cast<float*>(logits_out) : f0 + o_lg;
    pa.part = f0 + o_part;
    pa.att = f0 + o_att;
    pa.keys = reinterpret_cast<unsigned long long*>(f0 + o_keys);
    pa.counters = static_cast<int32_t*>(m->persist_counters.ptr);
    pa.out = out;
    static unsigned long long* trace = [] {
        unsigned long long* b = nullptr;
        const char* e = std::getenv("EP_TRACE");
        if (e && e[0] == '1' && cudaMalloc(&b, 256 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(b, 0, 256 * sizeof(unsigned long long));
        return b;
    }();
    pa.trace = trace;
    if (m->persist_image_ctas != persist_ctas) {  // weight images, once per model and grid size
        EP_CUDA_TRY(m->persist_image.reserve(persist_image_floats(m->L, m->D, m->F, m->V, persist_ctas) * sizeof(float)),
                    "ep_model persist image");
        pa.image_out = static_cast<float*>(m->persist_image.ptr);
        EP_CUDA_TRY(launch_persist_image(pa, persist_ctas, s), "ep_model persist image");
        m->persist_image_ctas = persist_ctas;
    }
    pa.image = static_cast<const float*>(m->persist_image.ptr);
    EP_CUDA_TRY(launch_decode_persist(pa, persist_ctas, s), "ep_model_generate persistent launch");
    if (trace) {  // debug: EP_TRACE=1 dumps the barrier timestamps to EP_TRACE_FILE
        std::vector<unsigned long long> hb(256);
        cudaStreamSynchronize(s);
        cudaMemcpy(hb.data(), trace, hb.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        const char* f = std::getenv("EP_TRACE_FILE");
        if (FILE* fp = std::fopen(f ? f : "ep_trace_persist.bin", "wb")) {
            std::fwrite(hb.data(), sizeof(unsigned long long), hb.size(), fp);
            std::fclose(fp);
        }
    }
    m->h->launches++;
    m->last_path = 3;
    return EP_OK;
}

}  // extern "C"

namespace {

// ep_model_forward, and with all_rows the verify pass of ep_model_verify
// (every new row unembedded, the acceptance rule per request).
int forward_impl(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                 const int32_t* page_table, const int32_t* n_new, const int32_t* tokens, void* hidden,
                 void* logits, int32_t* next, bool all_rows, int32_t* n_accepted, ep_stream stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EP_CUDA_TRY(cudaSetDevice(m->h->device), "ep_model_forward");

    std::vector<Req> reqs;
    bool all_decode = true;
    if (int rc = collect_requests(m, batch, seg_indptr, segs, page_table, n_new, reqs, &all_decode)) return rc;
    // request-major rows: request b's new tokens are consecutive
    Meta md;
    md.req_page_off.push_back(0);
    for (int b = 0; b < batch; ++b) {
        const Req& r = reqs[b];
        for (int i = 0; i < r.nn; ++i) {
            const int32_t tok = tokens[md.tokens.size()];
            if (tok < 0 || tok >= m->V) return fail(EP_EINVAL, "embed: unknown token id " + std::to_string(tok));
            md.tokens.push_back(tok);
            md.pos.push_back(int32_t(r.end - r.nn + i));
            md.dst_page.push_back(r.slots[i].first);
            md.dst_slot.push_back(r.slots[i].second);
            md.row_req.push_back(b);
        }
        md.last_row.push_back(int32_t(md.tokens.size() - 1));
        md.q_pos.push_back(r.end - 1);
        md.pdesc.insert(md.pdesc.end(), r.pages.begin(), r.pages.end());
        md.req_page_off.push_back(int64_t(md.pdesc.size()));
    }
    const int n = int(md.tokens.size());
    if (int rc = reserve_ws(m, n, batch)) return rc;
    Pass ps{};
    if (int rc = upload_meta(m, md, ps, s)) return rc;
    ps.n = n;
    ps.batch = batch;

    // decode_step of one session of a small fp32 model: the K9 persistent
    // kernel (one launch for the whole forward)
    int persist_ctas = 0;
    if (all_decode && !hidden && !all_rows && use_persist(m, batch, &persist_ctas))
        return run_persist(m, reqs, ps, batch, 1, persist_ctas,
                           next ? next : static_cast<int32_t*>(m->next_ws.ptr), logits, s);

    // attention: the spliced decode / prefill plans where a kernel instance
    // exists, otherwise the generic paged kernel
    if (uses_plans(m)) {
        const ep_kv_pool pool0 = m->pool(0);
        if (all_decode) {
            if (m->decode_plan && m->decode_plan_batch == batch) {
                if (int rc = ep_plan_update(m->decode_plan, seg_indptr, segs, page_table, md.q_pos.data(), stream))
                    return rc;
            } else {
                if (m->decode_plan) {
                    EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_model_forward");
                    ep_plan_destroy(m->decode_plan);
                    m->decode_plan = nullptr;
                }
                if (int rc = ep_plan_create(m->h, &pool0, m->H, 1, batch, seg_indptr, segs, page_table,
                                            md.q_pos.data(), 0, &m->decode_plan))
                    return rc;
                m->decode_plan_batch = batch;
            }
            ps.plan = m->decode_plan;
        } else {
            if (m->prefill_plan) {
                EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_model_forward");
                ep_plan_destroy(m->prefill_plan);
                m->prefill_plan = nullptr;
            }
            if (int rc = ep_plan_create_prefill(m->h, &pool0, m->H, batch, seg_indptr, segs, page_table, n_new,
                                                &m->prefill_plan))
                return rc;
            ps.plan = m->prefill_plan;
        }
    }
    m->last_path = ps.plan ? 1 : 2;
    ps.logits = logits ? logits : m->logits_ws.ptr;
    ps.next = next ? next : static_cast<int32_t*>(m->next_ws.ptr);
    ps.all_rows = all_rows;
    if (int rc = enqueue_pass(m, ps, s)) return rc;
    if (all_rows) {
        // the acceptance rule per request over its rows' targets (fused
        // accept of speculative verify)
        EP_CUDA_TRY(launch_accept_rows(ps.tok, ps.next, ps.last_row, batch, n_accepted, s), "accept launch");
        m->h->launches++;
    }
    if (hidden)
        EP_CUDA_TRY(cudaMemcpyAsync(hidden, m->hid.ptr, size_t(n) * m->D * m->esz(), cudaMemcpyDeviceToDevice, s),
                    "ep_model_forward hidden copy");
    return EP_OK;
}

}  // namespace

extern "C" {

int ep_model_forward(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                     const int32_t* page_table, const int32_t* n_new, const int32_t* tokens, void* hidden,
                     void* logits, int32_t* next, ep_stream stream) {
    if (!m || !seg_indptr || !n_new || !tokens || (batch > 0 && (!segs || !page_table)))
        return fail(EP_EINVAL, "ep_model_forward: null argument");
    if (batch < 0) return fail(EP_EINVAL, "ep_model_forward: batch");
    if (batch == 0) return EP_OK;
    return forward_impl(m, batch, seg_indptr, segs, page_table, n_new, tokens, hidden, logits, next, false,
                        nullptr, stream);
}

int ep_model_verify(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                    const int32_t* page_table, const int32_t* n_new, const int32_t* tokens, void* logits,
                    int32_t* targets, int32_t* n_accepted, ep_stream stream) {
    if (!m || !seg_indptr || !n_new || !tokens || !targets || !n_accepted ||
        (batch > 0 && (!segs || !page_table)))
        return fail(EP_EINVAL, "ep_model_verify: null argument");
    if (batch < 0) return fail(EP_EINVAL, "ep_model_verify: batch");
    if (batch == 0) return EP_OK;
    return forward_impl(m, batch, seg_indptr, segs, page_table, n_new, tokens, nullptr, logits, targets, true,
                        n_accepted, stream);
}

int ep_model_generate(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                      const int32_t* page_table, int32_t n_steps, const int32_t* first_tokens,
                      int32_t* out_tokens, ep_stream stream) {
    if (!m || !seg_indptr || !first_tokens || !out_tokens || (batch > 0 && (!segs || !page_table)))
        return fail(EP_EINVAL, "ep_model_generate: null argument");
    if (batch < 0 || n_steps < 0) return fail(EP_EINVAL, "ep_model_generate: batch / n_steps");
    if (batch == 0 || n_steps == 0) return EP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EP_CUDA_TRY(cudaSetDevice(m->h->device), "ep_model_generate");

    std::vector<int32_t> nn(batch, n_steps);
    std::vector<Req> reqs;
    bool all_decode = true;
    if (int rc = collect_requests(m, batch, seg_indptr, segs, page_table, nn.data(), reqs, &all_decode)) return rc;
    Meta md;
    md.req_page_off.push_back(0);
    for (int b = 0; b < batch; ++b) {
        const Req& r = reqs[b];
        if (r.end - r.nn <= r.start)  // decode_step on an empty cache (model.cpp:258)
            return fail(EP_EINVAL, "decode_step: empty cache");
        const int32_t tok = first_tokens[b];
        if (tok < 0 || tok >= m->V) return fail(EP_EINVAL, "embed: unknown token id " + std::to_string(tok));
        md.tokens.push_back(tok);
        md.row_req.push_back(b);
        md.last_row.push_back(b);
        md.q_pos.push_back(r.end - r.nn);  // advanced on the device after every step
        md.pdesc.insert(md.pdesc.end(), r.pages.begin(), r.pages.end());
        md.req_page_off.push_back(int64_t(md.pdesc.size()));
    }
    // step-major rows: entry t * batch + b
    for (int t = 0; t < n_steps; ++t)
        for (int b = 0; b < batch; ++b) {
            const Req& r = reqs[b];
            md.pos.push_back(int32_t(r.end - r.nn + t));
            md.dst_page.push_back(r.slots[t].first);
            md.dst_slot.push_back(r.slots[t].second);
        }
    md.step.assign(1, 0);
    if (int rc = reserve_ws(m, batch, batch)) return rc;
    DeviceBuffer out_dev;
    EP_CUDA_TRY(out_dev.reserve(size_t(n_steps) * batch * sizeof(int32_t)), "ep_model_generate out");
    Pass ps{};
    if (int rc = upload_meta(m, md, ps, s)) return rc;
    ps.n = batch;
    ps.batch = batch;
    ps.prev = static_cast<const int32_t*>(out_dev.ptr);
    ps.next = static_cast<int32_t*>(out_dev.ptr);
    ps.logits = m->logits_ws.ptr;

    int persist_ctas = 0;
    if (use_persist(m, batch, &persist_ctas)) {
        if (int rc = run_persist(m, reqs, ps, batch, n_steps, persist_ctas, static_cast<int32_t*>(out_dev.ptr),
                                 nullptr, s))
            return rc;
        std::vector<int32_t> host(size_t(n_steps) * batch);
        EP_CUDA_TRY(cudaMemcpyAsync(host.data(), out_dev.ptr, host.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s),
                    "ep_model_generate tokens");
        EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_model_generate");
        for (int b = 0; b < batch; ++b)
            for (int t = 0; t < n_steps; ++t) out_tokens[size_t(b) * n_steps + t] = host[size_t(t) * batch + b];
        return EP_OK;
    }

    // the decode plan is built once for the FINAL table; the causal rule
    // masks the keys past each step's query position, which advances on the
    // device (launch_advance), so every step replays the same launches
    ep_plan plan = nullptr;
    int64_t* qpos_dev = nullptr;
    if (uses_plans(m)) {
        const ep_kv_pool pool0 = m->pool(0);
        if (int rc = ep_plan_create(m->h, &pool0, m->H, 1, batch, seg_indptr, segs, page_table, md.q_pos.data(), 0,
                                    &plan))
            return rc;
        qpos_dev = plan_qpos_dev(plan);
    }
    std::unique_ptr<ep_plan_s, int (*)(ep_plan)> plan_guard(plan, ep_plan_destroy);
    ps.plan = plan;
    m->last_path = plan ? 1 : 2;

    // capture one step into a CUDA graph, replay it n_steps times
    cudaStream_t cap = nullptr;
    EP_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "ep_model_generate stream");
    std::unique_ptr<CUstream_st, cudaError_t (*)(cudaStream_t)> cap_guard(cap, cudaStreamDestroy);
    EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_model_generate");  // metadata + plan uploads landed
    const int64_t launches0 = m->h->launches.load();
    EP_CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "ep_model_generate capture");
    ps.advance = true;
    ps.adv_qpos = qpos_dev;
    int rc = enqueue_pass(m, ps, cap);
    cudaError_t e = cudaSuccess;
    cudaGraph_t graph = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap, &graph);
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    EP_CUDA_TRY(e, "ep_model_generate advance");
    EP_CUDA_TRY(e2, "ep_model_generate end capture");
    const int64_t per_step = m->h->launches.load() - launches0;
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    EP_CUDA_TRY(e, "ep_model_generate instantiate");
    for (int t = 0; t < n_steps && e == cudaSuccess; ++t) e = cudaGraphLaunch(exec, s);
    std::vector<int32_t> host(size_t(n_steps) * batch);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(host.data(), out_dev.ptr, host.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaGraphExecDestroy(exec);
    EP_CUDA_TRY(e, "ep_model_generate replay");
    m->h->launches += per_step * (n_steps - 1);  // replays run; the capture counted one step
    for (int b = 0; b < batch; ++b)
        for (int t = 0; t < n_steps; ++t) out_tokens[size_t(b) * n_steps + t] = host[size_t(t) * batch + b];
    return EP_OK;
}

}  // extern "C"
