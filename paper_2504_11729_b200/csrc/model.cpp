// model.cpp — include/ep/ep_model.h: the decoder around the spliced attention
// on the GPU.
//
// The reference (/root/reference/proj/core/src/model.cpp) keeps fp64 weights
// in host Matrix objects and runs, per new token row, embed -> L x
// transformer_layer -> unembed_logits -> argmax_token, with the attention of
// each layer as one partial_attention per cached segment (+ the new tokens)
// fused by merge_partials. Here:
//   * weights live in one device allocation in generation order, so
//     init_model is a single SplitMix64 fill (draw i -> element i);
//   * every layer has a KV page pool with the same page numbering, so one
//     host splice table addresses all layers;
//   * a forward pass is a fixed launch sequence per layer — QKV (LN fused,
//     K/V rows scattered into their pages), spliced attention (the K1/K3 plans
//     of plan.cpp, or the generic paged kernel for fp64 / other head sizes),
//     Wo + residual, LN + W1 + ReLU, W2 + residual — then the unembedding of
//     each request's last row and argmax.
#include <algorithm>
#include <cmath>
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

// Host-side row metadata of one forward, uploaded in one copy.
struct Meta {
    std::vector<int32_t> tokens, pos, dst_page, dst_slot, row_req, last_row;
    std::vector<int64_t> req_page_off, q_pos;
    std::vector<PageDesc> pdesc;
};

template <typename T>
size_t append_bytes(std::vector<char>& blob, const std::vector<T>& v) {
    const size_t off = (blob.size() + 255) & ~size_t(255);
    blob.resize(off + v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(T));
    return off;
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
    // generation order of init_model (model.cpp:82-102) = storage order
    const size_t D = size_t(m->D), V = size_t(m->V), F = size_t(m->F);
    size_t off = D * V;  // embedding [V][D]
    m->lw.resize(m->L);
    for (LayerOffsets& o : m->lw) {
        o.wq = off; off += D * D;
        o.wk = off; off += D * D;
        o.wv = off; off += D * D;
        o.wo = off; off += D * D;
        o.w1 = off; off += D * F;
        o.b1 = off; off += F;
        o.w2 = off; off += F * D;
        o.b2 = off; off += D;
    }
    m->off_unembed = off;
    off += D * V;
    m->n_weights = off;

    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_model_create");
    EP_CUDA_TRY(m->weights.reserve(m->n_weights * m->esz()), "ep_model_create weights");
    EP_CUDA_TRY(launch_fill_uniform_at(m->dt, m->weights.ptr, m->n_weights, c.init_seed, 0, -0.1, 0.1, nullptr),
                "ep_model_create init");
    h->launches++;
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
    // the fp64 draws (re-drawn when the weights are stored in fp32)
    DeviceBuffer tmp;
    const void* src = m->weights.ptr;
    if (m->dt != EP_F64) {
        EP_CUDA_TRY(tmp.reserve(m->n_weights * sizeof(double)), "ep_model_weight_sum");
        EP_CUDA_TRY(launch_fill_uniform_at(EP_F64, tmp.ptr, m->n_weights, m->cfg.init_seed, 0, -0.1, 0.1, nullptr),
                    "ep_model_weight_sum");
        m->h->launches++;
        src = tmp.ptr;
    }
    std::vector<double> w(m->n_weights);
    EP_CUDA_TRY(cudaMemcpy(w.data(), src, w.size() * sizeof(double), cudaMemcpyDeviceToHost),
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

int ep_model_forward(ep_model m, int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                     const int32_t* page_table, const int32_t* n_new, const int32_t* tokens, void* hidden,
                     void* logits, int32_t* next, ep_stream stream) {
    if (!m || !seg_indptr || !n_new || !tokens || (batch > 0 && (!segs || !page_table)))
        return fail(EP_EINVAL, "ep_model_forward: null argument");
    if (batch < 0) return fail(EP_EINVAL, "ep_model_forward: batch");
    if (batch == 0) return EP_OK;
    if (seg_indptr[0] != 0) return fail(EP_EINVAL, "ep_model_forward: seg_indptr[0] must be 0");
    ep_handle h = m->h;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_model_forward");

    // ---- host: validate, locate every new token's page slot ----
    Meta md;
    md.req_page_off.push_back(0);
    bool all_decode = true;
    for (int b = 0; b < batch; ++b) {
        std::vector<PageDesc> pages;
        int64_t first = 0;
        if (int rc = collect_request_pages(m->P, m->num_pages, b, seg_indptr, segs, page_table, pages, &first))
            return rc;
        const int64_t start = pages.empty() ? 0 : pages.front().pos;
        const int64_t end = pages.empty() ? 0 : pages.back().pos + pages.back().n_tok;
        const int nn = n_new[b];
        if (nn <= 0 || nn > end - start)
            return fail(EP_EINVAL, "ep_model_forward: request " + std::to_string(b) + " has " +
                                       std::to_string(end - start) + " tokens, n_new = " + std::to_string(nn));
        if (end > m->cfg.max_positions)
            return fail(EP_EINVAL, "embed: positions " + std::to_string(end - nn) + ".." + std::to_string(end) +
                                       " overflow max_positions " + std::to_string(m->cfg.max_positions));
        all_decode = all_decode && nn == 1;
        // new positions [end - nn, end): walk the descriptors from the back
        size_t di = pages.size();
        std::vector<std::pair<int32_t, int32_t>> slots(nn);
        for (int64_t p = end - 1; p >= end - nn; --p) {
            while (di > 0 && pages[di - 1].pos > p) --di;
            const PageDesc& d = pages[di - 1];
            slots[p - (end - nn)] = {d.page, int32_t(p - d.pos)};
        }
        for (int i = 0; i < nn; ++i) {
            const int32_t tok = tokens[md.tokens.size()];
            if (tok < 0 || tok >= m->V)
                return fail(EP_EINVAL, "embed: unknown token id " + std::to_string(tok));
            md.tokens.push_back(tok);
            md.pos.push_back(int32_t(end - nn + i));
            md.dst_page.push_back(slots[i].first);
            md.dst_slot.push_back(slots[i].second);
            md.row_req.push_back(b);
        }
        md.last_row.push_back(int32_t(md.tokens.size() - 1));
        md.q_pos.push_back(end - 1);
        md.pdesc.insert(md.pdesc.end(), pages.begin(), pages.end());
        md.req_page_off.push_back(int64_t(md.pdesc.size()));
    }
    const int n = int(md.tokens.size());

    // ---- workspace ----
    const size_t es = m->esz();
    EP_CUDA_TRY(m->hid.reserve(size_t(n) * m->D * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->xbuf.reserve(size_t(n) * m->D * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->qbuf.reserve(size_t(n) * m->D * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->attn.reserve(size_t(n) * m->D * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->h1.reserve(size_t(n) * m->F * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->logits_ws.reserve(size_t(batch) * m->V * es), "ep_model_forward ws");
    EP_CUDA_TRY(m->next_ws.reserve(size_t(batch) * sizeof(int32_t)), "ep_model_forward ws");

    // ---- metadata upload (pinned staging, one copy) ----
    std::vector<char> blob;
    const size_t o_tok = append_bytes(blob, md.tokens), o_pos = append_bytes(blob, md.pos),
                 o_pg = append_bytes(blob, md.dst_page), o_sl = append_bytes(blob, md.dst_slot),
                 o_rq = append_bytes(blob, md.row_req), o_last = append_bytes(blob, md.last_row),
                 o_rpo = append_bytes(blob, md.req_page_off), o_pd = append_bytes(blob, md.pdesc);
    EP_CUDA_TRY(m->meta.reserve(blob.size()), "ep_model_forward meta");
    EP_CUDA_TRY(cudaEventSynchronize(m->staged), "ep_model_forward staging");
    if (blob.size() > m->stage_bytes) {
        if (m->stage) cudaFreeHost(m->stage);
        m->stage = nullptr;
        EP_CUDA_TRY(cudaMallocHost(&m->stage, blob.size()), "ep_model_forward pinned");
        m->stage_bytes = blob.size();
    }
    std::memcpy(m->stage, blob.data(), blob.size());
    EP_CUDA_TRY(cudaMemcpyAsync(m->meta.ptr, m->stage, blob.size(), cudaMemcpyHostToDevice, s),
                "ep_model_forward meta copy");
    EP_CUDA_TRY(cudaEventRecord(m->staged, s), "ep_model_forward event");
    char* mb = static_cast<char*>(m->meta.ptr);
    const int32_t* d_tok = reinterpret_cast<const int32_t*>(mb + o_tok);
    const int32_t* d_pos = reinterpret_cast<const int32_t*>(mb + o_pos);
    const int32_t* d_pg = reinterpret_cast<const int32_t*>(mb + o_pg);
    const int32_t* d_sl = reinterpret_cast<const int32_t*>(mb + o_sl);
    const int32_t* d_rq = reinterpret_cast<const int32_t*>(mb + o_rq);
    const int32_t* d_last = reinterpret_cast<const int32_t*>(mb + o_last);
    const int64_t* d_rpo = reinterpret_cast<const int64_t*>(mb + o_rpo);
    const PageDesc* d_pd = reinterpret_cast<const PageDesc*>(mb + o_pd);

    // ---- attention path: the spliced decode / prefill plans where a kernel
    // instance exists, otherwise the generic paged kernel ----
    const bool fast = m->dt == EP_F32 && (m->dh == 64 || m->dh == 128) && m->P % 64 == 0;
    ep_plan plan = nullptr;
    if (fast) {
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
                if (int rc = ep_plan_create(h, &pool0, m->H, 1, batch, seg_indptr, segs, page_table,
                                            md.q_pos.data(), 0, &m->decode_plan))
                    return rc;
                m->decode_plan_batch = batch;
            }
            plan = m->decode_plan;
        } else {
            if (m->prefill_plan) {
                EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_model_forward");
                ep_plan_destroy(m->prefill_plan);
                m->prefill_plan = nullptr;
            }
            if (int rc = ep_plan_create_prefill(h, &pool0, m->H, batch, seg_indptr, segs, page_table, n_new,
                                                &m->prefill_plan))
                return rc;
            plan = m->prefill_plan;
        }
    }
    m->last_path = plan ? 1 : 2;

    // ---- launches ----
    const int dt = m->dt;
    EP_CUDA_TRY(launch_embed(dt, m->wptr(0), d_tok, d_pos, n, m->D, m->hid.ptr, s), "embed launch");
    h->launches++;
    for (int l = 0; l < m->L; ++l) {
        const LayerOffsets& o = m->lw[l];
        const ep_kv_pool pool = m->pool(l);
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
        a.dst_page = d_pg;
        a.dst_slot = d_sl;
        EP_CUDA_TRY(launch_dense(dt, kEpiQKV, true, a, s), "qkv launch");
        h->launches++;

        if (plan) {
            if (int rc = ep_spliced_attention(h, plan, &pool, EP_F32, m->qbuf.ptr, EP_F32, m->attn.ptr, nullptr,
                                              stream))
                return rc;
        } else {
            EP_CUDA_TRY(launch_attention_generic(dt, m->kv_dtype, m->qbuf.ptr, n, m->H, m->dh, d_pd, d_rpo, d_rq,
                                                 d_pos, pool.k_pages, pool.v_pages, m->P, m->attn.ptr, s),
                        "attention launch");
            h->launches++;
        }

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
    void* lg = logits ? logits : m->logits_ws.ptr;
    int32_t* nx = next ? next : static_cast<int32_t*>(m->next_ws.ptr);
    DenseArgs u{};
    u.x = m->hid.ptr;
    u.row_map = d_last;
    u.n = batch;
    u.K = m->D;
    u.N = m->V;
    u.w[0] = m->wptr(m->off_unembed);
    u.n_wblk = 1;
    u.out = lg;
    EP_CUDA_TRY(launch_dense(dt, kEpiStore, true, u, s), "unembed launch");
    h->launches++;
    EP_CUDA_TRY(launch_argmax_rows(dt, lg, batch, m->V, nx, s), "argmax launch");
    h->launches++;
    if (hidden)
        EP_CUDA_TRY(cudaMemcpyAsync(hidden, m->hid.ptr, size_t(n) * m->D * es, cudaMemcpyDeviceToDevice, s),
                    "ep_model_forward hidden copy");
    return EP_OK;
}

}  // extern "C"
