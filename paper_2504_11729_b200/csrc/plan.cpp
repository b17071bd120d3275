// plan.cpp — the device-resident splice-table plan (ep_plan_*) and the
// spliced-attention launch (ep_spliced_attention).
//
// The reference walks, per session, per layer and per head, an ordered list
// of KVSegments and calls partial_attention per segment (model.cpp:161-182,
// cache.cpp:25-103). Here the host turns the whole batch's splice table into
// device work lists once (and again only when it changes):
//
//   * every request's segments become a list of page descriptors
//     {page, valid tokens, absolute position} (validated with the reference's
//     invariants: gapless positions, origin order — cache.cpp:25-53);
//   * "virtual requests" (a page list + the query rows that attend to it) are
//     cut into work items so every CTA (one per SM) streams the same number of
//     64-token blocks ("stream-K" over pages, crossing (request, kv-head)
//     boundaries; split units merge by LSE inside the kernels);
//   * cascade: when consecutive requests share an identical first segment
//     (the same cloud-prompt pages, config 5), that prefix is attended ONCE per
//     kv-head for tiles of up to 128 query rows spanning 128/(G n_q) requests
//     on the tensor cores (K3), the private remainder per request by K1/K3,
//     and a 2-way LSE merge combines them.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "ep_internal.h"

using namespace ep;

namespace ep {

// Validates request b's segments with the SegmentedCache invariants
// (cache.cpp:25-53: gapless positions, origin order, pages in the pool) and
// appends its page descriptors; *first_pages = pages of its first segment.
int collect_request_pages(int page_tokens, int64_t num_pages, int b, const int64_t* seg_indptr,
                          const ep_segment* segs, const int32_t* page_table, std::vector<PageDesc>& out,
                          int64_t* first_pages) {
    const int P = page_tokens;
    if (seg_indptr[b + 1] < seg_indptr[b]) return fail(EP_EINVAL, "ep_plan: seg_indptr not monotone");
    int64_t expect_pos = -1;
    int last_origin = -1;
    *first_pages = 0;
    for (int64_t si = seg_indptr[b]; si < seg_indptr[b + 1]; ++si) {
        const ep_segment& s = segs[si];
        if (s.len < 0 || s.pos_offset < 0 || s.page_off < 0)
            return fail(EP_EINVAL, "ep_plan: negative segment field");
        if (expect_pos >= 0 && s.pos_offset != expect_pos)
            return fail(EP_EINVAL, "ep_plan: request " + std::to_string(b) + " segment starts at " +
                                       std::to_string(s.pos_offset) + ", previous ends at " +
                                       std::to_string(expect_pos));
        if (s.origin < last_origin)
            return fail(EP_EINVAL, "ep_plan: origin order must be (cloud, edge, generated)");
        expect_pos = s.pos_offset + s.len;
        last_origin = s.origin;
        const int64_t npg = (int64_t(s.len) + P - 1) / P;
        for (int64_t i = 0; i < npg; ++i) {
            const int32_t page = page_table[s.page_off + i];
            if (page < 0 || page >= num_pages)
                return fail(EP_EINVAL, "ep_plan: page id " + std::to_string(page) + " outside pool");
            PageDesc d;
            d.page = page;
            d.n_tok = int32_t(std::min<int64_t>(P, s.len - i * P));
            d.pos = s.pos_offset + i * P;
            out.push_back(d);
        }
        if (si == seg_indptr[b]) *first_pages = int64_t(out.size());
    }
    return EP_OK;
}

}  // namespace ep

namespace {

constexpr int kBlockTokens = 64;
constexpr int64_t kTcItemWeight = 10;  // K3 work-item overhead in blocks (see build_subplan)
// Overhead of a full 128-row K3 tile item (shared-prefix / prefill): the Q
// load, the two-group epilogue over 128 rows and, when the unit is split,
// the partial store + merge — measured by the per-CTA trace (tools/trace_k3.py).
int64_t tc_item_weight(int rows) {
    static const int64_t env = [] {
        const char* e = std::getenv("EP_TC_ITEM_WEIGHT");
        return e ? std::atoll(e) : -1;
    }();
    if (env >= 0) return env;
    return rows > 64 ? 14 : kTcItemWeight;
}
// K1 (CUDA-core decode) item overhead in blocks. Item ends run on K1's
// epilogue warp behind the streaming, so an item costs the consumers little:
// sweeping 0/1/2/4 blocks on config 2 gave 101.7 / 102.0 / 102.1 / 103.6 us
// (config 5 flat at 0.265 ms). (Before the epilogue warp the 8-warp item end
// stalled the ring and 4 was best: cfg5 0.321 -> 0.296 ms.)
// K1 tail penalty in blocks (see build_subplan)
int64_t k1_tail_pen() {
    static const int64_t w = [] {
        const char* e = std::getenv("EP_K1_TAIL_PEN");
        return e ? std::atoll(e) : int64_t(5);  // config 2 sweep 0/3/5/8: 100.4 / 99.0 / 97.8 / 98.7 us
    }();
    return w;
}
int64_t k1_item_weight() {
    static const int64_t w = [] {
        const char* e = std::getenv("EP_K1_ITEM_WEIGHT");
        return e ? std::atoll(e) : int64_t(0);
    }();
    return w;
}

// One query-row set attending to one page list.
struct VReq {
    std::vector<PageDesc> pages;
    int32_t rq0;     // first real request of the rows
    int64_t q0min;   // smallest query position among the rows
    int32_t n_rows;  // valid rows (<= the sub-plan's row stride)
};

struct SubPlan {
    int rows = 0;  // row stride per unit
    bool tc = false;
    int64_t n_ctas = 0, n_items = 0, n_pages = 0, n_units = 0;
    bool has_empty_unit = false;
    std::vector<PageDesc> pdesc;
    std::vector<int64_t> req_page_off;
    std::vector<WorkItem> items;
    std::vector<int32_t> cta_item_ptr, unit_item_ptr, cta_item_idx;
    std::vector<int32_t> cta_unit_ptr;  // fused split-KV: units whose final merge CTA c owns (its last item's CTA)
    DeviceBuffer d_pdesc, d_req_off, d_items, d_cta_ptr, d_unit_ptr, d_opart, d_lsepart, d_counter, d_cta_idx,
        d_cta_unit;
    size_t counter_units = 0;
};

// item_weight: fixed cost of one work item (Q load, epilogue, output) in
// 64-token-block units, so CTAs that get many short units (prefill chunks near
// the start of a prompt) are not overloaded. Measured for K3 (clock64 item
// trace): ~12-13K cycles per item vs ~1.0-1.4K per block -> 10.
//
// tail_pen (K1): a CTA whose items are all pieces of split units ends with
// one of them, and that final item end (partial store, arrival and usually
// the unit's merge) is not overlapped by streaming (~4 us vs ~1 us for a
// whole unit's store, per-CTA trace on config 2); such CTAs get tail_pen
// fewer blocks and the others share them (one re-cut).
void build_subplan(SubPlan& sp, const std::vector<VReq>& vr, int Hkv, int64_t cap_ctas,
                   int64_t item_weight = 0, int64_t tail_pen = 0) {
    sp.pdesc.clear();
    sp.req_page_off.assign(vr.size() + 1, 0);
    std::vector<int64_t> blocks(vr.size(), 0);
    for (size_t b = 0; b < vr.size(); ++b) {
        for (const PageDesc& d : vr[b].pages) {
            sp.pdesc.push_back(d);
            blocks[b] += (d.n_tok + kBlockTokens - 1) / kBlockTokens;
        }
        sp.req_page_off[b + 1] = int64_t(sp.pdesc.size());
    }
    sp.n_pages = int64_t(sp.pdesc.size());
    sp.n_units = int64_t(vr.size()) * Hkv;
    int64_t total = 0, total_blocks = 0;
    for (int64_t x : blocks) {
        total += (x + (x > 0 ? item_weight : 0)) * Hkv;
        total_blocks += x * Hkv;
    }
    sp.n_ctas = std::max<int64_t>(1, std::min<int64_t>(cap_ctas, total_blocks));
    std::vector<int32_t> item_cta;
    // cumulative capacity ends of the CTAs (equal shares first)
    std::vector<int64_t> bnd(sp.n_ctas);
    for (int64_t c = 0; c < sp.n_ctas; ++c) bnd[c] = (total * (c + 1) + sp.n_ctas - 1) / sp.n_ctas;
    // (the re-cut only where a CTA's share is much larger than the penalty)
    const bool recut = tail_pen > 0 && sp.n_ctas > 1 && total > 4 * tail_pen * sp.n_ctas;
    for (int pass = 0; pass < (recut ? 2 : 1); ++pass) {
    if (pass == 1) {
        // CTAs without a whole unit: shorter shares
        std::vector<int> whole(sp.n_ctas, 0);
        std::vector<int32_t> n_it(sp.n_units, 0);
        for (const WorkItem& w : sp.items) n_it[int64_t(w.b) * Hkv + w.g]++;
        for (size_t i = 0; i < sp.items.size(); ++i)
            if (n_it[int64_t(sp.items[i].b) * Hkv + sp.items[i].g] == 1) whole[item_cta[i]] = 1;
        int64_t n_flag = 0;
        for (int64_t c = 0; c < sp.n_ctas; ++c) n_flag += whole[c] ? 0 : 1;
        if (n_flag == 0 || n_flag == sp.n_ctas) break;
        const double base = double(total) / double(sp.n_ctas);
        const double lo = base - double(tail_pen);
        const double hi = base + double(tail_pen) * double(n_flag) / double(sp.n_ctas - n_flag);
        double run = 0.0;
        for (int64_t c = 0; c < sp.n_ctas; ++c) {
            run += whole[c] ? hi : lo;
            bnd[c] = int64_t(run + 0.5);
        }
        bnd[sp.n_ctas - 1] = total;
    }
    sp.items.clear();
    item_cta.clear();
    sp.cta_item_ptr.assign(sp.n_ctas + 1, 0);
    sp.unit_item_ptr.assign(sp.n_units + 1, 0);
    int64_t acc = 0, cta = 0;
    auto boundary = [&](int64_t c) { return bnd[c]; };
    for (size_t b = 0; b < vr.size(); ++b) {
        const int64_t npg = sp.req_page_off[b + 1] - sp.req_page_off[b];
        for (int g = 0; g < Hkv; ++g) {
            const int64_t unit = int64_t(b) * Hkv + g;
            bool open = false;
            if (npg > 0) acc += item_weight;
            for (int64_t lp = 0; lp < npg; ++lp) {
                while (cta < sp.n_ctas - 1 && acc >= boundary(cta)) {
                    ++cta;
                    open = false;
                }
                if (!open) {
                    WorkItem w{};
                    w.b = int32_t(b);
                    w.g = g;
                    w.lp0 = w.lp1 = int32_t(lp);
                    w.nblk = 0;
                    w.rq0 = vr[b].rq0;
                    w.q0min = int32_t(vr[b].q0min);
                    w.pad = vr[b].n_rows;
                    sp.items.push_back(w);
                    item_cta.push_back(int32_t(cta));
                    sp.unit_item_ptr[unit + 1]++;
                    open = true;
                }
                sp.items.back().lp1 = int32_t(lp + 1);
                const PageDesc& d = sp.pdesc[sp.req_page_off[b] + lp];
                const int nb = (d.n_tok + kBlockTokens - 1) / kBlockTokens;
                sp.items.back().nblk += nb;
                acc += nb;
            }
        }
    }
    }  // passes
    sp.n_items = int64_t(sp.items.size());
    for (int32_t c : item_cta) sp.cta_item_ptr[c + 1]++;
    for (int64_t c = 0; c < sp.n_ctas; ++c) sp.cta_item_ptr[c + 1] += sp.cta_item_ptr[c];
    sp.has_empty_unit = false;
    for (int64_t u = 0; u < sp.n_units; ++u) {
        if (sp.unit_item_ptr[u + 1] == 0) sp.has_empty_unit = true;
        sp.unit_item_ptr[u + 1] += sp.unit_item_ptr[u];
    }
    // owner of each unit = the CTA of its last item (monotonic in the unit)
    sp.cta_unit_ptr.assign(sp.n_ctas + 1, 0);
    for (int64_t u = 0; u < sp.n_units; ++u)
        if (sp.unit_item_ptr[u + 1] > sp.unit_item_ptr[u]) sp.cta_unit_ptr[item_cta[sp.unit_item_ptr[u + 1] - 1] + 1]++;
    for (int64_t c = 0; c < sp.n_ctas; ++c) sp.cta_unit_ptr[c + 1] += sp.cta_unit_ptr[c];
    // K1 order within a CTA: items of split units first, whole units last.
    // A split item's end (partial store, arrival, maybe the merge) then runs
    // on the epilogue warp while the CTA streams on, and the CTA's final item
    // end — the one nothing overlaps — is a plain output store where possible.
    sp.cta_item_idx.resize(sp.items.size());
    for (int64_t c = 0; c < sp.n_ctas; ++c) {
        int32_t o = sp.cta_item_ptr[c];
        for (int pass = 0; pass < 2; ++pass)
            for (int32_t it = sp.cta_item_ptr[c]; it < sp.cta_item_ptr[c + 1]; ++it) {
                const int64_t unit = int64_t(sp.items[it].b) * Hkv + sp.items[it].g;
                const bool split = sp.unit_item_ptr[unit + 1] - sp.unit_item_ptr[unit] > 1;
                if (split == (pass == 0)) sp.cta_item_idx[o++] = it;
            }
    }
}

template <typename T>
size_t bytes_of(const std::vector<T>& v) {
    return v.size() * sizeof(T);
}

}  // namespace

struct ep_plan_s {
    ep_handle h = nullptr;
    int32_t kv_dtype = 0, n_kv_heads = 0, d_head = 0, page_tokens = 0;
    int64_t num_pages = 0;
    int32_t n_q_heads = 0, n_q = 0, batch = 0, rows = 0;
    bool cascade = false;
    bool concurrent = false;          // cascade passes on disjoint SM sets, side by side
    cudaStream_t side = nullptr;      // the shared-prefix pass's stream (concurrent cascade)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool prefill = false;             // prefill plan: virtual requests = query chunks
    int32_t chunks = 1;               // decode plan cut into query chunks (K1 takes <= 8 rows): per request
    int32_t chunk_q = 0;              //   `chunks` virtual requests of chunk_q tokens
    bool generic = false;             // no K1 / K3 instance: the generic kernel (any d_head <= 256, any group)
    std::vector<int32_t> q_row0;      // prefill: first q/o token row per virtual request
    int64_t n_q_rows = 0;             // prefill: query token rows (sum n_new)
    SubPlan main;    // whole table (non-cascade) or the private remainders (cascade)
    SubPlan shared;  // cascade: shared prefixes, row-group tiles on K3
    std::vector<int64_t> q_pos;
    std::vector<uint8_t> has_shared;  // per request (cascade)
    DeviceBuffer d_qpos, d_has_shared, d_parts_o, d_parts_lse, d_qrow0;
    // every uploaded plan array lives in ONE device arena (views above and in
    // the sub-plans), each part with some capacity slack: an update is one
    // pinned-staged H2D copy, and the views stay put (captured CUDA graphs
    // stay valid) until a part outgrows its capacity
    DeviceBuffer arena;
    std::vector<size_t> arena_cap;
    // ep_cache the plan was last fully built from (ep_plan_create_cache / a
    // full ep_plan_update_cache): identity, structure version, layer
    const void* built_cache = nullptr;
    uint64_t built_version = 0;
    int built_layer = -1;
    // staging for stream-ordered updates: a ring of pinned buffers, so an
    // update waits only for the upload kStageRing updates back (the host
    // stays ahead of the GPU in a serving loop)
    static constexpr int kStageRing = 4;
    void* h_stage[kStageRing] = {};
    size_t h_stage_bytes[kStageRing] = {};
    cudaEvent_t staged[kStageRing] = {};
    int stage_idx = 0;
    CUtensorMap tmap_k{}, tmap_v{};
    const void* tm_k = nullptr;
    const void* tm_v = nullptr;
    int64_t tm_pages = -1;
    ~ep_plan_s() {
        for (int i = 0; i < kStageRing; ++i) {
            if (staged[i]) {
                cudaEventSynchronize(staged[i]);
                cudaEventDestroy(staged[i]);
            }
            if (h_stage[i]) cudaFreeHost(h_stage[i]);
        }
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
    }
};

namespace {

// EP_CASCADE_SERIAL=1 runs the two cascade passes one after the other on
// all SMs (the pre-overlap schedule, kept for comparison).
bool concurrent_cascade() {
    static const bool serial = [] {
        const char* e = std::getenv("EP_CASCADE_SERIAL");
        return e && e[0] == '1';
    }();
    return !serial;
}

bool cascade_allowed(const ep_plan_s& p) {
    static const bool off = [] {
        const char* e = std::getenv("EP_NO_CASCADE");
        return e && e[0] == '1';
    }();
    const int rpr = (p.n_q_heads / p.n_kv_heads) * p.n_q;
    return !off && verify_supported(p.kv_dtype, p.d_head, rpr) && rpr <= 128 && 128 / rpr >= 2;
}

// Validates request b's segments with the SegmentedCache invariants and
// appends its page descriptors (see ep::collect_request_pages).
int collect_pages(const ep_plan_s& p, int b, const int64_t* seg_indptr, const ep_segment* segs,
                  const int32_t* page_table, std::vector<PageDesc>& out, int64_t* first_pages) {
    return collect_request_pages(p.page_tokens, p.num_pages, b, seg_indptr, segs, page_table, out,
                                 first_pages);
}

int pow2ceil_rows(int r) { return r <= 1 ? 1 : r <= 2 ? 2 : r <= 4 ? 4 : 8; }

int build_plan_host(ep_plan_s& p, const int64_t* seg_indptr, const ep_segment* segs,
                    const int32_t* page_table, const int64_t* q_pos) {
    const int B = p.batch, Hkv = p.n_kv_heads, G = p.n_q_heads / Hkv;
    const int rpr = G * p.n_q;
    p.q_pos.assign(q_pos, q_pos + B);
    if (seg_indptr[0] != 0) return fail(EP_EINVAL, "ep_plan: seg_indptr[0] must be 0");
    // per request: page descriptors, and where its first segment's pages end
    std::vector<std::vector<PageDesc>> req_pages(B);
    std::vector<int64_t> first_seg_pages(B, 0);
    for (int b = 0; b < B; ++b) {
        if (q_pos[b] < 0 || q_pos[b] > INT32_MAX) return fail(EP_EINVAL, "ep_plan: query position out of range");
        if (int rc = collect_pages(p, b, seg_indptr, segs, page_table, req_pages[b], &first_seg_pages[b]))
            return rc;
    }
    const int64_t cap = int64_t(p.h->n_sms);

    // ---- kernel choice: K1 (CUDA cores, <= 8 rows per unit, padded to a
    // power of two), K3 (tcgen05, bf16 d 128, <= 64 rows), K1 on query
    // chunks of 8 / G tokens (more rows, G <= 8), else the generic kernel ----
    const bool k1_direct = decode_supported(p.kv_dtype, p.d_head, rpr);
    const bool k3 = verify_supported(p.kv_dtype, p.d_head, rpr) && rpr <= 64;
    const bool k1_chunk = !k1_direct && !k3 && G <= 8 && decode_supported(p.kv_dtype, p.d_head, G);
    p.generic = !k1_direct && !k3 && !k1_chunk;
    p.chunks = 1;
    p.chunk_q = p.n_q;
    if (p.generic) {
        std::vector<VReq> vr(B);
        for (int b = 0; b < B; ++b) {
            vr[b].pages = std::move(req_pages[b]);
            vr[b].rq0 = b;
            vr[b].q0min = q_pos[b];
            vr[b].n_rows = rpr;
        }
        p.cascade = false;
        p.has_shared.assign(B, 0);
        p.main.tc = false;
        build_subplan(p.main, vr, Hkv, cap, 0);  // page descriptors only
        p.main.rows = rpr;
        return EP_OK;
    }
    if (k1_chunk) {
        // virtual request v = b * chunks + c holds query tokens [c C, (c+1) C)
        // of request b at positions q_pos[b] + c C ..; its pages stop at its
        // last query (later keys are masked anyway)
        const int C = std::max(1, 8 / G);
        p.chunk_q = C;
        p.chunks = (p.n_q + C - 1) / C;
        std::vector<VReq> vr;
        std::vector<int64_t> vq;
        for (int b = 0; b < B; ++b)
            for (int c = 0; c < p.chunks; ++c) {
                const int nq = std::min(C, p.n_q - c * C);
                const int64_t q0 = q_pos[b] + int64_t(c) * C, vis = q0 + nq;
                VReq v;
                for (const PageDesc& d : req_pages[b]) {
                    if (d.pos >= vis) break;
                    PageDesc t = d;
                    t.n_tok = int32_t(std::min<int64_t>(d.n_tok, vis - d.pos));
                    v.pages.push_back(t);
                }
                v.rq0 = int32_t(vr.size());
                v.q0min = q0;
                v.n_rows = G * nq;
                vq.push_back(q0);
                vr.push_back(std::move(v));
            }
        p.q_pos = vq;
        p.cascade = false;
        p.has_shared.assign(B, 0);
        p.main.tc = false;
        build_subplan(p.main, vr, Hkv, cap, k1_item_weight(), k1_tail_pen());
        p.main.rows = pow2ceil_rows(G * C);
        return EP_OK;
    }

    // ---- cascade detection: runs of consecutive requests whose first segment
    // is the same page list (a shared cloud prompt) ----
    p.cascade = false;
    p.has_shared.assign(B, 0);
    std::vector<VReq> shared_vr;
    const int group_cap = cascade_allowed(p) ? 128 / rpr : 0;
    if (group_cap >= 2) {
        auto same_first = [&](int a, int b) {
            if (first_seg_pages[a] != first_seg_pages[b] || first_seg_pages[a] < 2) return false;
            for (int64_t i = 0; i < first_seg_pages[a]; ++i) {
                const PageDesc &x = req_pages[a][i], &y = req_pages[b][i];
                if (x.page != y.page || x.n_tok != y.n_tok || x.pos != y.pos) return false;
            }
            return true;
        };
        int b = 0;
        while (b < B) {
            int e = b + 1;
            while (e < B && same_first(b, e)) ++e;
            if (e - b >= 2) {
                for (int r0 = b; r0 < e; r0 += group_cap) {
                    const int r1 = std::min(e, r0 + group_cap);
                    VReq v;
                    v.pages.assign(req_pages[r0].begin(), req_pages[r0].begin() + first_seg_pages[r0]);
                    v.rq0 = r0;
                    v.q0min = q_pos[r0];
                    for (int r = r0; r < r1; ++r) {
                        v.q0min = std::min<int64_t>(v.q0min, q_pos[r]);
                        p.has_shared[r] = 1;
                    }
                    v.n_rows = (r1 - r0) * rpr;
                    shared_vr.push_back(std::move(v));
                }
            }
            b = e;
        }
        p.cascade = !shared_vr.empty();
    }
    std::vector<VReq> main_vr(B);
    for (int b = 0; b < B; ++b) {
        const int64_t skip = p.has_shared[b] ? first_seg_pages[b] : 0;
        main_vr[b].pages.assign(req_pages[b].begin() + skip, req_pages[b].end());
        main_vr[b].rq0 = b;
        main_vr[b].q0min = q_pos[b];
        main_vr[b].n_rows = rpr;
    }
    p.main.tc = !k1_direct || (force_tc() && k3);
    int64_t cap_main = cap, cap_shared = cap;
    if (p.cascade && !p.main.tc && concurrent_cascade()) {
        // The shared-prefix tiles (K3: tensor / MUFU bound, ~35 MB of K/V)
        // and the private remainders (K1: HBM bound) run side by side on
        // disjoint SMs; the SMs are split in proportion to their estimated
        // times (per 64-key block: K3 128-row tile ~0.70 us beside K1, K1
        // ~0.80 us — per-CTA trace, tools/trace_k3.py; an SM-count sweep on
        // config 5 puts the optimum at 24-25 of 148 SMs for the shared pass).
        int64_t sb = 0, mb = 0;
        for (const VReq& v : shared_vr)
            for (const PageDesc& d : v.pages) sb += (d.n_tok + kBlockTokens - 1) / kBlockTokens;
        for (const VReq& v : main_vr)
            for (const PageDesc& d : v.pages) mb += (d.n_tok + kBlockTokens - 1) / kBlockTokens;
        const double ts = 0.70 * double(sb), tm = 0.80 * double(mb);
        cap_shared = std::max<int64_t>(1, std::min<int64_t>(cap - 1, int64_t(double(cap) * ts / (ts + tm) + 0.5)));
        static const int64_t env_sh = [] {
            const char* e = std::getenv("EP_CASCADE_SHARED_CTAS");
            return e ? std::atoll(e) : int64_t(0);
        }();
        if (env_sh > 0 && env_sh < cap) cap_shared = env_sh;
        cap_main = cap - cap_shared;
        p.concurrent = true;
    } else {
        p.concurrent = false;
    }
    if (!p.main.tc) {
        static const int64_t env = [] {
            const char* e = std::getenv("EP_K1_CTAS");
            return e ? std::atoll(e) : int64_t(0);
        }();
        if (env > 0) cap_main = env;
    }
    build_subplan(p.main, main_vr, Hkv, cap_main, p.main.tc ? kTcItemWeight : k1_item_weight(),
                  p.main.tc ? 0 : k1_tail_pen());
    p.main.rows = p.main.tc ? rpr : pow2ceil_rows(rpr);
    if (p.cascade) {
        build_subplan(p.shared, shared_vr, Hkv, cap_shared, tc_item_weight(group_cap * rpr));
        p.shared.rows = group_cap * rpr;
        p.shared.tc = true;
    }
    return EP_OK;
}

// Prefill plan (cloud-prompt / edge prefill, model.cpp:211-236 ->
// transformer_layer's attention block): the last n_new[b] tokens of request b
// are queries; query t attends to every key at a position <= its own
// (attention.cpp:29-33). The queries are cut into chunks of C = 128 / G
// tokens, so one chunk x G heads fills the M = 128 rows of a K3 tile; each
// chunk is a virtual request whose page list stops at its last query (the
// diagonal blocks are masked per row inside K3).
int build_prefill_host(ep_plan_s& p, int n_req, const int64_t* seg_indptr, const ep_segment* segs,
                       const int32_t* page_table, const int32_t* n_new) {
    const int Hkv = p.n_kv_heads, G = p.n_q_heads / Hkv;
    const int C = p.n_q;  // query tokens per chunk
    if (seg_indptr[0] != 0) return fail(EP_EINVAL, "ep_plan: seg_indptr[0] must be 0");
    std::vector<VReq> vr;
    p.q_pos.clear();
    p.q_row0.clear();
    int64_t tok_base = 0;
    for (int b = 0; b < n_req; ++b) {
        std::vector<PageDesc> pages;
        int64_t first = 0;
        if (int rc = collect_pages(p, b, seg_indptr, segs, page_table, pages, &first)) return rc;
        const int64_t end = pages.empty() ? 0 : pages.back().pos + pages.back().n_tok;
        const int64_t start = pages.empty() ? 0 : pages.front().pos;
        if (n_new[b] < 0 || n_new[b] > end - start)
            return fail(EP_EINVAL, "ep_plan_create_prefill: request " + std::to_string(b) + " has " +
                                       std::to_string(end - start) + " tokens, n_new = " +
                                       std::to_string(n_new[b]));
        if (end > INT32_MAX) return fail(EP_EINVAL, "ep_plan_create_prefill: position out of range");
        for (int64_t q0 = end - n_new[b]; q0 < end; q0 += C) {
            const int64_t nq = std::min<int64_t>(C, end - q0), vis = q0 + nq;  // keys < vis
            VReq v;
            for (const PageDesc& d : pages) {
                if (d.pos >= vis) break;
                PageDesc t = d;
                t.n_tok = int32_t(std::min<int64_t>(d.n_tok, vis - d.pos));
                v.pages.push_back(t);
            }
            v.rq0 = int32_t(vr.size());
            v.q0min = q0;
            v.n_rows = int32_t(nq) * G;
            p.q_pos.push_back(q0);
            p.q_row0.push_back(int32_t(tok_base + (q0 - (end - n_new[b]))));
            vr.push_back(std::move(v));
        }
        tok_base += n_new[b];
        if (tok_base > INT32_MAX) return fail(EP_EINVAL, "ep_plan_create_prefill: too many query tokens");
    }
    p.batch = int32_t(vr.size());
    p.n_q_rows = tok_base;
    p.cascade = false;
    p.has_shared.assign(vr.size(), 0);
    build_subplan(p.main, vr, Hkv, int64_t(p.h->n_sms), p.main.tc ? tc_item_weight(G * C) : 1);
    p.main.rows = G * C;
    return EP_OK;
}

int upload_subplan(SubPlan& sp, int d_head, cudaStream_t s, std::vector<std::pair<DeviceBuffer*, std::pair<const void*, size_t>>>& parts) {
    parts.push_back({&sp.d_pdesc, {sp.pdesc.data(), bytes_of(sp.pdesc)}});
    parts.push_back({&sp.d_req_off, {sp.req_page_off.data(), bytes_of(sp.req_page_off)}});
    parts.push_back({&sp.d_items, {sp.items.data(), bytes_of(sp.items)}});
    parts.push_back({&sp.d_cta_ptr, {sp.cta_item_ptr.data(), bytes_of(sp.cta_item_ptr)}});
    parts.push_back({&sp.d_unit_ptr, {sp.unit_item_ptr.data(), bytes_of(sp.unit_item_ptr)}});
    parts.push_back({&sp.d_cta_idx, {sp.cta_item_idx.data(), bytes_of(sp.cta_item_idx)}});
    parts.push_back({&sp.d_cta_unit, {sp.cta_unit_ptr.data(), bytes_of(sp.cta_unit_ptr)}});
    const size_t ws = size_t(std::max<int64_t>(sp.n_items, 1)) * sp.rows;
    EP_CUDA_TRY(sp.d_opart.reserve(ws * d_head * sizeof(float)), "ep_plan workspace");
    EP_CUDA_TRY(sp.d_lsepart.reserve(ws * sizeof(float)), "ep_plan workspace");
    const size_t units = size_t(std::max<int64_t>(1, sp.n_units));
    if (units > sp.counter_units) {
        EP_CUDA_TRY(sp.d_counter.reserve(units * sizeof(int32_t)), "ep_plan counters");
        // on the launch stream (a non-blocking stream does not wait for the legacy one)
        EP_CUDA_TRY(cudaMemsetAsync(sp.d_counter.ptr, 0, units * sizeof(int32_t), s), "ep_plan counters");
        sp.counter_units = units;
    }
    return EP_OK;
}

using Parts = std::vector<std::pair<DeviceBuffer*, std::pair<const void*, size_t>>>;

// Stream-ordered upload of the plan arrays: (re)lays out the arena when a
// part does not fit its capacity, stages every part at its arena offset in
// one pinned slot of the ring and copies the used extent with ONE H2D copy
// (async), or synchronously at plan creation.
int stage_and_copy(ep_plan_s& p, const Parts& parts, cudaStream_t s, bool async) {
    bool relayout = p.arena_cap.size() != parts.size() || !p.arena.ptr;
    for (size_t i = 0; !relayout && i < parts.size(); ++i) relayout = parts[i].second.second > p.arena_cap[i];
    if (relayout) {
        p.arena_cap.resize(parts.size());
        size_t total = 0;
        for (size_t i = 0; i < parts.size(); ++i) {
            const size_t b = parts[i].second.second;
            p.arena_cap[i] = (std::max<size_t>(b + b / 4, 256) + 255) & ~size_t(255);
            total += p.arena_cap[i];
        }
        // (cudaFree of the old arena waits for kernels still reading it)
        if (p.arena.ptr) {
            cudaFree(p.arena.ptr);
            p.arena.ptr = nullptr;
            p.arena.bytes = 0;
        }
        EP_CUDA_TRY(p.arena.reserve(total), "ep_plan arena");
        size_t off = 0;
        for (size_t i = 0; i < parts.size(); ++i) {
            DeviceBuffer* v = parts[i].first;
            if (v->ptr && !v->view) cudaFree(v->ptr);
            v->ptr = static_cast<char*>(p.arena.ptr) + off;
            v->bytes = p.arena_cap[i];
            v->view = true;
            off += p.arena_cap[i];
        }
    }
    size_t extent = 0, off = 0;
    for (size_t i = 0; i < parts.size(); ++i) {
        if (parts[i].second.second) extent = off + parts[i].second.second;
        off += p.arena_cap[i];
    }
    if (!extent) return EP_OK;
    if (!async) {
        std::vector<char> blob(extent);
        off = 0;
        for (size_t i = 0; i < parts.size() && off < extent; ++i) {
            if (parts[i].second.second) std::memcpy(blob.data() + off, parts[i].second.first, parts[i].second.second);
            off += p.arena_cap[i];
        }
        EP_CUDA_TRY(cudaMemcpy(p.arena.ptr, blob.data(), extent, cudaMemcpyHostToDevice), "ep_plan upload");
        return EP_OK;
    }
    const int k = p.stage_idx;
    p.stage_idx = (p.stage_idx + 1) % ep_plan_s::kStageRing;
    if (p.staged[k]) EP_CUDA_TRY(cudaEventSynchronize(p.staged[k]), "ep_plan_update wait");
    if (extent > p.h_stage_bytes[k]) {
        if (p.h_stage[k]) cudaFreeHost(p.h_stage[k]);
        p.h_stage[k] = nullptr;
        EP_CUDA_TRY(cudaMallocHost(&p.h_stage[k], p.arena.bytes), "ep_plan_update pinned");
        p.h_stage_bytes[k] = p.arena.bytes;
    }
    if (!p.staged[k]) EP_CUDA_TRY(cudaEventCreateWithFlags(&p.staged[k], cudaEventDisableTiming), "event");
    off = 0;
    for (size_t i = 0; i < parts.size() && off < extent; ++i) {
        if (parts[i].second.second)
            std::memcpy(static_cast<char*>(p.h_stage[k]) + off, parts[i].second.first, parts[i].second.second);
        off += p.arena_cap[i];
    }
    EP_CUDA_TRY(cudaMemcpyAsync(p.arena.ptr, p.h_stage[k], extent, cudaMemcpyHostToDevice, s), "ep_plan_update copy");
    EP_CUDA_TRY(cudaEventRecord(p.staged[k], s), "ep_plan_update event");
    return EP_OK;
}

int upload_plan(ep_plan_s& p, cudaStream_t s, bool async);

// Per-token growth fast path of ep_plan_update: when every request keeps the
// same pages, in the same 64-token blocks, and only the token counts of its
// pages and its query position moved (a decode step appending into the last
// page's free slots), the work partition stays valid: the page descriptors
// and query positions are refreshed and re-uploaded, nothing is re-planned.
// Returns 1 when it applied, 0 when a full rebuild is needed, <0 on error.
int try_grow_in_place(ep_plan_s& p, const int64_t* seg_indptr, const ep_segment* segs, const int32_t* page_table,
                      const int64_t* q_pos, cudaStream_t s) {
    if (p.cascade || p.prefill || p.generic || p.chunks > 1 || p.main.tc || p.main.pdesc.empty()) return 0;
    SubPlan& sp = p.main;
    std::vector<PageDesc> pages;
    pages.reserve(sp.pdesc.size());
    for (int b = 0; b < p.batch; ++b) {
        if (q_pos[b] < 0 || q_pos[b] > INT32_MAX) return -fail(EP_EINVAL, "ep_plan: query position out of range");
        const size_t before = pages.size();
        int64_t first = 0;
        if (int rc = collect_pages(p, b, seg_indptr, segs, page_table, pages, &first)) return -rc;
        const int64_t n = int64_t(pages.size() - before);
        if (n != sp.req_page_off[b + 1] - sp.req_page_off[b]) return 0;
    }
    if (pages.size() != sp.pdesc.size()) return 0;
    for (size_t i = 0; i < pages.size(); ++i) {
        const PageDesc &a = pages[i], &o = sp.pdesc[i];
        if (a.page != o.page || a.pos != o.pos ||
            (a.n_tok + kBlockTokens - 1) / kBlockTokens != (o.n_tok + kBlockTokens - 1) / kBlockTokens)
            return 0;
    }
    sp.pdesc.swap(pages);
    p.q_pos.assign(q_pos, q_pos + p.batch);
    if (int rc = upload_plan(p, s, true)) return -rc;  // one staged copy of the (unchanged-layout) arena
    return 1;
}

int upload_plan(ep_plan_s& p, cudaStream_t s, bool async) {
    std::vector<std::pair<DeviceBuffer*, std::pair<const void*, size_t>>> parts;
    parts.push_back({&p.d_qpos, {p.q_pos.data(), bytes_of(p.q_pos)}});
    parts.push_back({&p.d_has_shared, {p.has_shared.data(), bytes_of(p.has_shared)}});
    if (p.prefill) parts.push_back({&p.d_qrow0, {p.q_row0.data(), bytes_of(p.q_row0)}});
    if (int rc = upload_subplan(p.main, p.d_head, s, parts)) return rc;
    if (p.cascade) {
        if (int rc = upload_subplan(p.shared, p.d_head, s, parts)) return rc;
        const size_t rows = size_t(p.batch) * p.n_q * p.n_q_heads;
        EP_CUDA_TRY(p.d_parts_o.reserve(2 * rows * p.d_head * sizeof(float)), "ep_plan cascade ws");
        EP_CUDA_TRY(p.d_parts_lse.reserve(2 * rows * sizeof(float)), "ep_plan cascade ws");
    }
    return stage_and_copy(p, parts, s, async);
}

bool valid_dt(int dt) { return dt == EP_F32 || dt == EP_BF16; }

// final_dtype: the dtype the caller asked for (fp32 output keeps P as bf16
// hi+lo in K3; bf16 output uses a single bf16 P).
DecodeArgs make_args(const ep_plan_s& p, const SubPlan& sp, const ep_kv_pool* pool, int32_t q_dtype,
                     const void* q, int32_t o_dtype, void* o, float* lse, int32_t final_dtype) {
    DecodeArgs a{};
    a.k_pages = pool->k_pages;
    a.v_pages = pool->v_pages;
    a.n_kv_heads = p.n_kv_heads;
    a.n_q_heads = p.n_q_heads;
    a.page_tokens = p.page_tokens;
    a.n_q = p.chunks > 1 ? p.chunk_q : p.n_q;
    a.num_pages = pool->num_pages;
    a.n_q_rows = p.prefill ? p.n_q_rows : int64_t(p.batch) * p.n_q;
    a.n_items = int32_t(sp.n_items);
    a.chunks = p.chunks;
    a.nq_total = p.n_q;
    a.pdesc = static_cast<const PageDesc*>(sp.d_pdesc.ptr);
    a.req_page_off = static_cast<const int64_t*>(sp.d_req_off.ptr);
    a.items = static_cast<const WorkItem*>(sp.d_items.ptr);
    a.cta_item_ptr = static_cast<const int32_t*>(sp.d_cta_ptr.ptr);
    a.cta_item_idx = sp.tc ? nullptr : static_cast<const int32_t*>(sp.d_cta_idx.ptr);
    a.unit_item_ptr = static_cast<const int32_t*>(sp.d_unit_ptr.ptr);
    a.q_pos = static_cast<const int64_t*>(p.d_qpos.ptr);
    a.q = q;
    a.q_dtype = q_dtype;
    a.o_part = static_cast<float*>(sp.d_opart.ptr);
    a.lse_part = static_cast<float*>(sp.d_lsepart.ptr);
    a.o = o;
    a.o_dtype = o_dtype;
    a.lse = lse;
    a.batch = int32_t(sp.n_units / std::max(1, p.n_kv_heads));
    a.q_scale = float(1.4426950408889634 / std::sqrt(double(p.d_head)));
    a.zero_rows = p.h->zero_rows.ptr;
    a.unit_counter = static_cast<int32_t*>(sp.d_counter.ptr);
    a.trace = nullptr;
    a.reqs_per_unit = 1;
    a.q_row0 = p.prefill ? static_cast<const int32_t*>(p.d_qrow0.ptr) : nullptr;
    a.pv_parts = final_dtype == EP_F32 ? 2 : 1;
    return a;
}

unsigned long long* trace_buffer() {
    static unsigned long long* t = [] {
        unsigned long long* b = nullptr;
        const char* e = std::getenv("EP_TRACE");
        if (e && e[0] == '1' && cudaMalloc(&b, 32 * 1024 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(b, 0, 32 * 1024 * sizeof(unsigned long long));
        return b;
    }();
    return t;
}

// debug: EP_TRACE=1 dumps the trace buffer (CTA 0 event clocks, per-CTA
// start / end / work) of the last launch to EP_TRACE_FILE
void dump_trace(unsigned long long* trace, cudaStream_t s) {
    std::vector<unsigned long long> host(32 * 1024);
    cudaStreamSynchronize(s);
    cudaMemcpy(host.data(), trace, host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    const char* f = std::getenv("EP_TRACE_FILE");
    if (FILE* fp = std::fopen(f ? f : "ep_trace.bin", "wb")) {
        std::fwrite(host.data(), sizeof(unsigned long long), host.size(), fp);
        std::fclose(fp);
    }
}

int launch_subplan(ep_plan_s& p, SubPlan& sp, const ep_kv_pool* pool, DecodeArgs a, cudaStream_t s) {
    ep_handle h = p.h;
    if (sp.n_items > 0 && sp.tc) {
        if (p.tm_k != pool->k_pages || p.tm_v != pool->v_pages || p.tm_pages != pool->num_pages) {
            const int64_t rows_total = pool->num_pages * pool->n_kv_heads * pool->page_tokens;
            if (int rc = encode_kv_map(&p.tmap_k, pool->k_pages, rows_total)) return rc;
            if (int rc = encode_kv_map(&p.tmap_v, pool->v_pages, rows_total)) return rc;
            p.tm_k = pool->k_pages;
            p.tm_v = pool->v_pages;
            p.tm_pages = pool->num_pages;
        }
        a.trace = trace_buffer();
        EP_CUDA_TRY(launch_verify_attention(int(sp.n_ctas), a, p.tmap_k, p.tmap_v, sp.rows, s),
                    "verify attention launch");
        h->launches++;
        if (a.trace) dump_trace(a.trace, s);
    } else if (p.generic) {
        EP_CUDA_TRY(launch_generic_decode(p.kv_dtype, p.d_head, p.batch, p.n_q, a, s), "generic decode launch");
        h->launches++;
        return EP_OK;
    } else if (sp.n_items > 0) {
        a.trace = trace_buffer();
        EP_CUDA_TRY(launch_spliced_decode(p.kv_dtype, p.d_head, sp.rows, int(sp.n_ctas), a, s),
                    "spliced decode launch");
        h->launches++;
        if (a.trace) dump_trace(a.trace, s);
    }
    if (sp.has_empty_unit) {
        EP_CUDA_TRY(launch_empty_units(p.d_head, sp.rows, a, s), "empty units launch");
        h->launches++;
    }
    return EP_OK;
}

}  // namespace

namespace ep {
void plan_mark_built(ep_plan p, const void* cache, uint64_t version, int layer) {
    if (!p) return;
    p->built_cache = cache;
    p->built_version = version;
    p->built_layer = layer;
}

int plan_grow_in_place(ep_plan p, const void* cache, uint64_t version, int layer, const int64_t* ends, int n_q,
                       cudaStream_t s) {
    if (!p || p->built_cache != cache || p->built_version != version || p->built_layer != layer) return 0;
    if (p->cascade || p->prefill || p->generic || p->chunks > 1 || p->main.tc || n_q != p->n_q) return 0;
    SubPlan& sp = p->main;
    // every request's last page takes its new end; block counts must not change
    for (int b = 0; b < p->batch; ++b) {
        const int64_t i = sp.req_page_off[b + 1] - 1;
        if (i < sp.req_page_off[b]) return 0;
        const PageDesc& d = sp.pdesc[size_t(i)];
        const int64_t n = ends[b] - d.pos;
        if (n < 1 || n > p->page_tokens ||
            (n + kBlockTokens - 1) / kBlockTokens != (d.n_tok + kBlockTokens - 1) / kBlockTokens)
            return 0;
    }
    // host mirror + device patch (one small kernel per 128 requests; the
    // arena, its views and any captured graph's pointers stay as they are)
    PlanPatch pp{};
    pp.pdesc = static_cast<PageDesc*>(sp.d_pdesc.ptr);
    pp.q_pos = static_cast<int64_t*>(p->d_qpos.ptr);
    for (int b = 0; b < p->batch; ++b) {
        const int32_t i = int32_t(sp.req_page_off[b + 1] - 1);
        PageDesc& d = sp.pdesc[size_t(i)];
        const int32_t nt = int32_t(ends[b] - d.pos);
        const int64_t qp = std::max<int64_t>(0, ends[b] - n_q);
        if (nt == d.n_tok && qp == p->q_pos[b]) continue;
        d.n_tok = nt;
        p->q_pos[b] = qp;
        pp.idx[pp.n] = i;
        pp.ntok[pp.n] = nt;
        pp.req[pp.n] = b;
        pp.qpos[pp.n] = qp;
        if (++pp.n == kPlanPatchMax) {
            EP_CUDA_TRY(launch_plan_patch(pp, s), "ep_plan_update_cache patch");
            pp.n = 0;
        }
    }
    EP_CUDA_TRY(launch_plan_patch(pp, s), "ep_plan_update_cache patch");
    return 1;
}

int64_t* plan_qpos_dev(ep_plan p) { return p ? static_cast<int64_t*>(p->d_qpos.ptr) : nullptr; }
}  // namespace ep

extern "C" {

int ep_plan_create(ep_handle h, const ep_kv_pool* pool, int32_t n_q_heads, int32_t n_q,
                   int32_t batch, const int64_t* seg_indptr, const ep_segment* segs,
                   const int32_t* page_table, const int64_t* q_pos, int32_t ctas_per_sm,
                   ep_plan* out) {
    if (!h || !pool || !out || !seg_indptr || !q_pos) return fail(EP_EINVAL, "ep_plan_create: null argument");
    *out = nullptr;
    if (!valid_dt(pool->dtype)) return fail(EP_EUNSUPPORTED, "ep_plan_create: kv dtype must be f32 or bf16");
    if (pool->n_kv_heads <= 0 || n_q_heads <= 0 || n_q_heads % pool->n_kv_heads)
        return fail(EP_EINVAL, "ep_plan_create: n_q_heads must be a multiple of n_kv_heads");
    if (pool->page_tokens <= 0 || pool->page_tokens % kBlockTokens)
        return fail(EP_EUNSUPPORTED, "ep_plan_create: page_tokens must be a multiple of 64");
    if (batch < 0 || n_q <= 0) return fail(EP_EINVAL, "ep_plan_create: batch/n_q");
    const int rows = (n_q_heads / pool->n_kv_heads) * n_q;
    if (!generic_supported(pool->dtype, pool->d_head))
        return fail(EP_EUNSUPPORTED, "ep_plan_create: no kernel for kv dtype " + std::to_string(pool->dtype) +
                                         ", d_head=" + std::to_string(pool->d_head) + " (d_head must be 1..256)");
    std::unique_ptr<ep_plan_s> p(new (std::nothrow) ep_plan_s());
    if (!p) return fail(EP_ENOMEM, "ep_plan_create");
    p->h = h;
    p->kv_dtype = pool->dtype;
    p->n_kv_heads = pool->n_kv_heads;
    p->d_head = pool->d_head;
    p->page_tokens = pool->page_tokens;
    p->num_pages = pool->num_pages;
    p->n_q_heads = n_q_heads;
    p->n_q = n_q;
    p->batch = batch;
    p->rows = rows;
    (void)ctas_per_sm;
    if (int rc = build_plan_host(*p, seg_indptr, segs, page_table, q_pos)) return rc;
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_plan_create");
    if (int rc = upload_plan(*p, nullptr, false)) return rc;
    *out = p.release();
    return EP_OK;
}

int ep_plan_create_prefill(ep_handle h, const ep_kv_pool* pool, int32_t n_q_heads, int32_t batch,
                           const int64_t* seg_indptr, const ep_segment* segs, const int32_t* page_table,
                           const int32_t* n_new, ep_plan* out) {
    if (!h || !pool || !out || !seg_indptr || !n_new) return fail(EP_EINVAL, "ep_plan_create_prefill: null argument");
    *out = nullptr;
    if (pool->n_kv_heads <= 0 || n_q_heads <= 0 || n_q_heads % pool->n_kv_heads)
        return fail(EP_EINVAL, "ep_plan_create_prefill: n_q_heads must be a multiple of n_kv_heads");
    if (pool->page_tokens <= 0 || pool->page_tokens % kBlockTokens)
        return fail(EP_EUNSUPPORTED, "ep_plan_create_prefill: page_tokens must be a multiple of 64");
    if (batch < 0) return fail(EP_EINVAL, "ep_plan_create_prefill: batch");
    // tcgen05 tiles (K3) of C = 128/G query tokens x G heads where K3 has an
    // instance (bf16 KV, d_head 128); otherwise CUDA-core chunks (K1) of
    // C = 8/G tokens (fp32 / bf16 KV, d_head 64 or 128, G <= 8) — the
    // reference's own MHA shapes (config 1: fp32, d_head 64).
    const int G = n_q_heads / pool->n_kv_heads;
    const bool tc = G <= 128 && verify_supported(pool->dtype, pool->d_head, 128 / G * G);
    const bool k1 = !tc && G <= 8 && decode_supported(pool->dtype, pool->d_head, 8 / G * G);
    if (!tc && !k1)
        return fail(EP_EUNSUPPORTED, "ep_plan_create_prefill: no prefill kernel for kv dtype " +
                                         std::to_string(pool->dtype) + ", d_head " + std::to_string(pool->d_head) +
                                         ", group " + std::to_string(G) +
                                         " (tcgen05: bf16, d_head 128; CUDA cores: f32/bf16, d_head 64/128, group <= 8)");
    const int C = tc ? 128 / G : 8 / G;
    std::unique_ptr<ep_plan_s> p(new (std::nothrow) ep_plan_s());
    if (!p) return fail(EP_ENOMEM, "ep_plan_create_prefill");
    p->h = h;
    p->kv_dtype = pool->dtype;
    p->n_kv_heads = pool->n_kv_heads;
    p->d_head = pool->d_head;
    p->page_tokens = pool->page_tokens;
    p->num_pages = pool->num_pages;
    p->n_q_heads = n_q_heads;
    p->n_q = C;
    p->rows = G * C;
    p->prefill = true;
    p->main.tc = tc;
    if (int rc = build_prefill_host(*p, batch, seg_indptr, segs, page_table, n_new)) return rc;
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_plan_create_prefill");
    if (int rc = upload_plan(*p, nullptr, false)) return rc;
    *out = p.release();
    return EP_OK;
}

int ep_plan_update(ep_plan p, const int64_t* seg_indptr, const ep_segment* segs,
                   const int32_t* page_table, const int64_t* q_pos, ep_stream stream) {
    if (!p) return fail(EP_EINVAL, "ep_plan_update: null plan");
    if (p->prefill) return fail(EP_EINVAL, "ep_plan_update: prefill plans are rebuilt with ep_plan_create_prefill");
    p->built_cache = nullptr;  // (ep_plan_update_cache re-marks after a full build)
    const int fast = try_grow_in_place(*p, seg_indptr, segs, page_table, q_pos, static_cast<cudaStream_t>(stream));
    if (fast < 0) return -fast;
    if (fast == 1) return EP_OK;
    if (int rc = build_plan_host(*p, seg_indptr, segs, page_table, q_pos)) return rc;
    return upload_plan(*p, static_cast<cudaStream_t>(stream), true);
}

int ep_plan_destroy(ep_plan p) {
    delete p;
    return EP_OK;
}

int ep_spliced_attention_splitkv(ep_handle h, ep_plan p, const ep_kv_pool* pool, int32_t q_dtype, const void* q,
                                 ep_peer_group g, int32_t o_dtype, void* o, float* lse, ep_stream stream) {
    if (!h || !p || !pool || !q || !g || !o) return fail(EP_EINVAL, "ep_spliced_attention_splitkv: null argument");
    if (pool->dtype != p->kv_dtype || pool->n_kv_heads != p->n_kv_heads || pool->d_head != p->d_head ||
        pool->page_tokens != p->page_tokens || pool->num_pages < p->num_pages)
        return fail(EP_EINVAL, "ep_spliced_attention_splitkv: pool does not match the plan");
    if (!valid_dt(q_dtype) || !valid_dt(o_dtype))
        return fail(EP_EUNSUPPORTED, "ep_spliced_attention_splitkv: q/o dtype must be f32 or bf16");
    if (p->cascade || p->main.tc || p->generic || p->prefill || p->chunks > 1)
        return fail(EP_EUNSUPPORTED, "ep_spliced_attention_splitkv: the fused combine runs on the K1 decode "
                                     "plans (f32/bf16 KV, d_head 64/128, <= 8 rows per unit, no shared prefix)");
    if (p->main.has_empty_unit)
        return fail(EP_EINVAL, "ep_spliced_attention_splitkv: every (request, kv-head) needs keys on every rank");
    const int64_t rows = int64_t(p->batch) * p->n_q * p->n_q_heads;
    DecodeArgs a = make_args(*p, p->main, pool, q_dtype, q, o_dtype, o, lse, o_dtype);
    if (int rc = peer_link_fill(g, p->main.n_units, rows, p->d_head,
                                static_cast<const int32_t*>(p->main.d_cta_unit.ptr), &a.peer))
        return rc;
    return launch_subplan(*p, p->main, pool, a, static_cast<cudaStream_t>(stream));
}

int ep_plan_info(ep_plan p, int64_t* n_ctas, int64_t* n_items, int64_t* n_pages) {
    if (!p) return fail(EP_EINVAL, "ep_plan_info: null plan");
    if (n_ctas) *n_ctas = p->main.n_ctas + (p->cascade ? p->shared.n_ctas : 0);
    if (n_items) *n_items = p->main.n_items + (p->cascade ? p->shared.n_items : 0);
    if (n_pages) *n_pages = p->main.n_pages + (p->cascade ? p->shared.n_pages : 0);
    return EP_OK;
}

int ep_spliced_attention(ep_handle h, ep_plan p, const ep_kv_pool* pool, int32_t q_dtype,
                         const void* q, int32_t o_dtype, void* o, float* lse, ep_stream stream) {
    if (!h || !p || !pool || !q || !o) return fail(EP_EINVAL, "ep_spliced_attention: null argument");
    if (pool->dtype != p->kv_dtype || pool->n_kv_heads != p->n_kv_heads ||
        pool->d_head != p->d_head || pool->page_tokens != p->page_tokens ||
        pool->num_pages < p->num_pages)
        return fail(EP_EINVAL, "ep_spliced_attention: pool does not match the plan");
    if (!valid_dt(q_dtype) || !valid_dt(o_dtype))
        return fail(EP_EUNSUPPORTED, "ep_spliced_attention: q/o dtype must be f32 or bf16");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!p->cascade) {
        DecodeArgs a = make_args(*p, p->main, pool, q_dtype, q, o_dtype, o, lse, o_dtype);
        return launch_subplan(*p, p->main, pool, a, s);
    }
    // cascade: shared prefixes (K3 row-group tiles) -> part 0, private
    // remainders (K1/K3) -> part 1, then the 2-way LSE merge into o / lse.
    const size_t rows = size_t(p->batch) * p->n_q * p->n_q_heads;
    float* po = static_cast<float*>(p->d_parts_o.ptr);
    float* pl = static_cast<float*>(p->d_parts_lse.ptr);
    DecodeArgs as = make_args(*p, p->shared, pool, q_dtype, q, EP_F32, po, pl, o_dtype);
    DecodeArgs am = make_args(*p, p->main, pool, q_dtype, q, EP_F32, po + rows * p->d_head, pl + rows, o_dtype);
    if (p->concurrent) {
        // fork: the shared pass on the side stream, the private pass here;
        // each kernel's grid is its SM share, so they run side by side
        if (!p->side) {
            EP_CUDA_TRY(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking), "cascade stream");
            EP_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "cascade event");
            EP_CUDA_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming), "cascade event");
        }
        EP_CUDA_TRY(cudaEventRecord(p->ev_fork, s), "cascade fork");
        EP_CUDA_TRY(cudaStreamWaitEvent(p->side, p->ev_fork, 0), "cascade fork");
        if (int rc = launch_subplan(*p, p->shared, pool, as, p->side)) return rc;
        if (int rc = launch_subplan(*p, p->main, pool, am, s)) return rc;
        EP_CUDA_TRY(cudaEventRecord(p->ev_join, p->side), "cascade join");
        EP_CUDA_TRY(cudaStreamWaitEvent(s, p->ev_join, 0), "cascade join");
    } else {
        if (int rc = launch_subplan(*p, p->shared, pool, as, s)) return rc;
        if (int rc = launch_subplan(*p, p->main, pool, am, s)) return rc;
    }
    EP_CUDA_TRY(launch_cascade_merge(int(rows), p->d_head, p->n_q * p->n_q_heads, po, pl,
                                     static_cast<const uint8_t*>(p->d_has_shared.ptr), o, o_dtype, lse, s),
                "cascade merge launch");
    h->launches++;
    return EP_OK;
}

}  // extern "C"
