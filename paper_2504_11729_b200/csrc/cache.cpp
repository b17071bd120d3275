// cache.cpp — ep_cache: the reference's SegmentedCache (cache.hpp:30-61,
// cache.cpp:16-103) for a batch of sessions whose K/V live in paged device
// pools, plus the plan builders that read it directly (no host arrays in
// between), so a serving loop grows every session by one token per step with
// a few microseconds of host work.
//
// State per (layer, request): an ordered list of segments {origin,
// pos_offset, len, pages}. Pages are ids in that layer's pool; the usual
// layout shares page ids across layers (one append for all layers), but
// per-layer appends exist for K/V that arrives layer by layer (kv frames,
// edge.cpp:177-209), which is what check_consistent guards.
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "ep_internal.h"

using ep::fail;

namespace {

struct Seg {
    int32_t origin;
    int64_t pos_offset;
    int64_t len;
    std::vector<int32_t> pages;
    int64_t end() const { return pos_offset + len; }
};

}  // namespace

struct ep_cache_s {
    int32_t n_layers = 0, batch = 0, page_tokens = 0;
    // bumped by every change other than tokens landing in already-listed
    // pages (append, a new page, truncation): a plan built at this version
    // can follow pure in-page growth without re-planning
    uint64_t structure_version = 1;
    std::vector<std::vector<std::vector<Seg>>> seg;  // [layer][request] -> segments
    // flattened arrays of one layer (rebuilt on demand for the plan builders)
    std::vector<int64_t> indptr;
    std::vector<ep_segment> flat;
    std::vector<int32_t> pt;

    int64_t end_position(int l, int b) const {
        const auto& s = seg[l][b];
        return s.empty() ? 0 : s.back().end();
    }
    void flatten(int l) {
        indptr.assign(batch + 1, 0);
        flat.clear();
        pt.clear();
        for (int b = 0; b < batch; ++b) {
            for (const Seg& s : seg[l][b]) {
                flat.push_back(ep_segment{s.origin, int32_t(s.len), s.pos_offset, int64_t(pt.size())});
                pt.insert(pt.end(), s.pages.begin(), s.pages.end());
            }
            indptr[b + 1] = int64_t(flat.size());
        }
        if (pt.empty()) pt.push_back(0);
    }
};

namespace {

int64_t pages_for(int64_t len, int P) { return (len + P - 1) / P; }

// cache.cpp:82-103 for one request: the reference's messages.
std::string check_request(const ep_cache_s& c, int b) {
    const auto& l0 = c.seg[0][b];
    for (int l = 0; l < c.n_layers; ++l) {
        const auto& segs = c.seg[l][b];
        if (segs.size() != l0.size()) return "layer segment counts differ";
        int64_t pos = segs.empty() ? 0 : segs.front().pos_offset;
        int last = -1;
        for (size_t i = 0; i < segs.size(); ++i) {
            const Seg& s = segs[i];
            if (s.pos_offset != pos) return "gap in position coverage";
            if (s.origin < last) return "origin order violated";
            if (s.pos_offset != l0[i].pos_offset || s.len != l0[i].len) return "layers cover different position ranges";
            if (int64_t(s.pages.size()) < pages_for(s.len, c.page_tokens)) return "segment has fewer pages than tokens";
            last = s.origin;
            pos = s.end();
        }
    }
    return {};
}

}  // namespace

extern "C" {

int ep_cache_create(int32_t n_layers, int32_t batch, int32_t page_tokens, ep_cache* out) {
    if (!out) return fail(EP_EINVAL, "ep_cache_create: null out");
    *out = nullptr;
    if (n_layers <= 0) return fail(EP_EINVAL, "SegmentedCache: zero layers");
    if (batch < 0 || page_tokens <= 0) return fail(EP_EINVAL, "ep_cache_create: batch / page_tokens");
    std::unique_ptr<ep_cache_s> c(new (std::nothrow) ep_cache_s());
    if (!c) return fail(EP_ENOMEM, "ep_cache_create");
    c->n_layers = n_layers;
    c->batch = batch;
    c->page_tokens = page_tokens;
    c->seg.assign(n_layers, std::vector<std::vector<Seg>>(batch));
    *out = c.release();
    return EP_OK;
}

int ep_cache_destroy(ep_cache c) {
    delete c;
    return EP_OK;
}

int64_t ep_cache_end_position(ep_cache c, int32_t b) {
    if (!c || b < 0 || b >= c->batch) return -1;
    return c->end_position(0, b);  // layers_.front() (cache.cpp:21-24)
}

int ep_cache_append(ep_cache c, int32_t layer, int32_t b, int32_t origin, int64_t pos_offset, int32_t len,
                    const int32_t* pages, int32_t n_pages) {
    if (!c || (!pages && n_pages > 0)) return fail(EP_EINVAL, "ep_cache_append: null argument");
    if (b < 0 || b >= c->batch) return fail(EP_EINVAL, "ep_cache_append: request out of range");
    if (layer < -1 || layer >= c->n_layers) return fail(EP_EINVAL, "SegmentedCache::append: segment layer mismatch");
    if (origin < 0 || origin > 2) return fail(EP_EINVAL, "ep_cache_append: origin must be 0 (cloud), 1 (edge), 2 (generated)");
    const int l0 = layer < 0 ? 0 : layer, l1 = layer < 0 ? c->n_layers : layer + 1;
    // validated for every layer first, then applied (cache.cpp:25-53: atomic)
    for (int l = l0; l < l1; ++l) {
        // all-layer appends continue the cache end (layer 0's); a per-layer
        // append continues its own layer (frames arrive layer by layer)
        const int64_t end = layer < 0 ? c->end_position(0, b) : c->end_position(l, b);
        const bool first = c->seg[l][b].empty();
        if (!first && pos_offset != end)
            return fail(EP_EINVAL, "SegmentedCache::append: segment starts at " + std::to_string(pos_offset) +
                                       ", cache ends at " + std::to_string(end));
        if (len <= 0) return fail(EP_EINVAL, "SegmentedCache::append: empty segment");
        if (!first && origin < c->seg[l][b].back().origin)
            return fail(EP_EINVAL, "SegmentedCache::append: origin order must be (cloud, edge, generated)");
    }
    if (pos_offset < 0) return fail(EP_EINVAL, "ep_cache_append: negative position");
    if (n_pages < pages_for(len, c->page_tokens))
        return fail(EP_EINVAL, "ep_cache_append: " + std::to_string(len) + " tokens need " +
                                   std::to_string(pages_for(len, c->page_tokens)) + " pages, got " +
                                   std::to_string(n_pages));
    for (int l = l0; l < l1; ++l)
        c->seg[l][b].push_back(Seg{origin, pos_offset, len,
                                   std::vector<int32_t>(pages, pages + pages_for(len, c->page_tokens))});
    c->structure_version++;
    return EP_OK;
}

int ep_cache_append_generated(ep_cache c, const int32_t* n_tokens, const int32_t* new_pages, int32_t max_new,
                              int32_t* dst_page, int32_t* dst_slot, int32_t* pages_used) {
    if (!c || !n_tokens || !dst_page || !dst_slot) return fail(EP_EINVAL, "ep_cache_append_generated: null argument");
    const int P = c->page_tokens;
    // validate: page supply and cross-layer agreement of the trailing generated segments
    for (int b = 0; b < c->batch; ++b) {
        const int32_t n = n_tokens[b];
        if (n < 0) return fail(EP_EINVAL, "ep_cache_append_generated: negative token count");
        if (n == 0) continue;
        const auto& s0 = c->seg[0][b];
        const bool has_gen = !s0.empty() && s0.back().origin == 2;
        const int64_t free = has_gen ? int64_t(s0.back().pages.size()) * P - s0.back().len : 0;
        const int64_t need = n > free ? pages_for(n - free, P) : 0;
        if (need > max_new || (need > 0 && !new_pages))
            return fail(EP_EINVAL, "ep_cache_append_generated: request " + std::to_string(b) + " needs " +
                                       std::to_string(need) + " new pages, max_new = " + std::to_string(max_new));
        for (int l = 1; l < c->n_layers; ++l) {
            const auto& s = c->seg[l][b];
            if (s.size() != s0.size() || (!s.empty() && (s.back().end() != s0.back().end() ||
                                                          s.back().origin != s0.back().origin)))
                return fail(EP_EINVAL, "ep_cache_append_generated: layers cover different position ranges");
        }
    }
    int64_t row = 0;
    for (int b = 0; b < c->batch; ++b) {
        const int32_t n = n_tokens[b];
        int32_t used = 0;
        if (n > 0) {
            const int64_t pos = c->end_position(0, b);
            for (int l = 0; l < c->n_layers; ++l) {
                auto& segs = c->seg[l][b];
                if (segs.empty() || segs.back().origin != 2) {
                    segs.push_back(Seg{2, pos, 0, {}});
                    c->structure_version++;
                }
                Seg& g = segs.back();
                int32_t u = 0;
                while (int64_t(g.pages.size()) * P < g.len + n) g.pages.push_back(new_pages[size_t(b) * max_new + u++]);
                if (u) c->structure_version++;
                used = u;
                if (l == 0)
                    for (int32_t i = 0; i < n; ++i) {
                        const int64_t t = g.len + i;  // token index inside the segment
                        dst_page[row + i] = g.pages[size_t(t / P)];
                        dst_slot[row + i] = int32_t(t % P);
                    }
                g.len += n;
            }
            row += n;
        }
        if (pages_used) pages_used[b] = used;
    }
    return EP_OK;
}

int ep_cache_truncate(ep_cache c, int32_t b, int32_t n_tokens, int32_t* released, int32_t* n_released) {
    if (!c || b < 0 || b >= c->batch) return fail(EP_EINVAL, "ep_cache_truncate: bad argument");
    if (n_released) *n_released = 0;
    if (n_tokens <= 0) return EP_OK;
    const auto& s0 = c->seg[0][b];
    if (s0.empty() || s0.back().origin != 2 || s0.back().len < n_tokens)
        return fail(EP_EINVAL, "ep_cache_truncate: request " + std::to_string(b) +
                                   " has fewer generated tokens than " + std::to_string(n_tokens));
    int32_t nr = 0;
    for (int l = 0; l < c->n_layers; ++l) {
        auto& segs = c->seg[l][b];
        if (segs.empty() || segs.back().origin != 2 || segs.back().len < n_tokens)
            return fail(EP_EINVAL, "ep_cache_truncate: layers cover different position ranges");
        Seg& g = segs.back();
        g.len -= n_tokens;
        const size_t keep = size_t(pages_for(g.len, c->page_tokens));
        if (l == 0) {
            for (size_t i = keep; i < g.pages.size(); ++i)
                if (released) released[nr++] = g.pages[i];
                else ++nr;
        }
        g.pages.resize(keep);
        if (g.len == 0) segs.pop_back();
    }
    c->structure_version++;
    if (n_released) *n_released = nr;
    return EP_OK;
}

int ep_cache_check_consistent(ep_cache c) {
    if (!c) return fail(EP_EINVAL, "ep_cache_check_consistent: null cache");
    for (int b = 0; b < c->batch; ++b) {
        const std::string why = check_request(*c, b);
        if (!why.empty()) return fail(EP_EINVAL, "request " + std::to_string(b) + ": " + why);
    }
    return EP_OK;
}

int ep_cache_layer_arrays(ep_cache c, int32_t layer, int64_t* seg_indptr, ep_segment* segs, int64_t segs_cap,
                          int32_t* page_table, int64_t pages_cap, int64_t* n_segs, int64_t* n_pages) {
    if (!c || layer < 0 || layer >= c->n_layers) return fail(EP_EINVAL, "ep_cache_layer_arrays: bad argument");
    c->flatten(layer);
    if (n_segs) *n_segs = int64_t(c->flat.size());
    if (n_pages) *n_pages = int64_t(c->pt.size());
    if (!seg_indptr) return EP_OK;  // size query
    if (!segs || !page_table || segs_cap < int64_t(c->flat.size()) || pages_cap < int64_t(c->pt.size()))
        return fail(EP_EINVAL, "ep_cache_layer_arrays: output arrays too small");
    std::memcpy(seg_indptr, c->indptr.data(), c->indptr.size() * sizeof(int64_t));
    if (!c->flat.empty()) std::memcpy(segs, c->flat.data(), c->flat.size() * sizeof(ep_segment));
    std::memcpy(page_table, c->pt.data(), c->pt.size() * sizeof(int32_t));
    return EP_OK;
}

// Decode / verify plans straight from the cache: the queries of request b
// are its last n_q positions (q_pos = end - n_q), as decode_step and the
// verify construction place them.
int ep_plan_create_cache(ep_handle h, const ep_kv_pool* pool, ep_cache c, int32_t layer, int32_t n_q_heads,
                         int32_t n_q, ep_plan* out) {
    if (!c || layer < 0 || layer >= c->n_layers) return fail(EP_EINVAL, "ep_plan_create_cache: bad cache / layer");
    if (pool && pool->page_tokens != c->page_tokens)
        return fail(EP_EINVAL, "ep_plan_create_cache: pool page_tokens != cache page_tokens");
    c->flatten(layer);
    std::vector<int64_t> qp(c->batch);
    for (int b = 0; b < c->batch; ++b) qp[b] = std::max<int64_t>(0, c->end_position(layer, b) - n_q);
    if (int rc = ep_plan_create(h, pool, n_q_heads, n_q, c->batch, c->indptr.data(), c->flat.data(), c->pt.data(),
                                qp.data(), 0, out))
        return rc;
    ep::plan_mark_built(*out, c, c->structure_version, layer);
    return EP_OK;
}

int ep_plan_update_cache(ep_plan p, ep_cache c, int32_t layer, int32_t n_q, ep_stream stream) {
    if (!c || layer < 0 || layer >= c->n_layers) return fail(EP_EINVAL, "ep_plan_update_cache: bad cache / layer");
    std::vector<int64_t> ends(c->batch);
    for (int b = 0; b < c->batch; ++b) ends[b] = c->end_position(layer, b);
    // pure in-page growth since the plan's last full build from this cache:
    // O(batch) page-descriptor refresh, no re-plan
    const int fast = ep::plan_grow_in_place(p, c, c->structure_version, layer, ends.data(), n_q,
                                            static_cast<cudaStream_t>(stream));
    if (fast < 0) return -fast;
    if (fast == 1) return EP_OK;
    c->flatten(layer);
    std::vector<int64_t> qp(c->batch);
    for (int b = 0; b < c->batch; ++b) qp[b] = std::max<int64_t>(0, ends[b] - n_q);
    if (int rc = ep_plan_update(p, c->indptr.data(), c->flat.data(), c->pt.data(), qp.data(), stream)) return rc;
    ep::plan_mark_built(p, c, c->structure_version, layer);
    return EP_OK;
}

}  // extern "C"
