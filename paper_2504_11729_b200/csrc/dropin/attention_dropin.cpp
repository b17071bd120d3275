// attention_dropin.cpp — link-level drop-in for the reference's attention.cpp.
//
// The reference builds src/attention.cpp into edgeprompt_core
// (proj/core/CMakeLists.txt:1-14). Linking THIS translation unit in its place
// gives every caller — transformer_layer (model.cpp:161-182), prefill,
// decode_step, the cloud server and the edge client — the same
// edgeprompt:: functions (attention.hpp:13-52), computed on the B200 by
// libep_b200.so through the C-ABI in include/ep/ep_attn.h.
//
// Semantics kept: value-semantics fp64 Matrix in/out, identity partials for
// fully masked rows, std::invalid_argument for shape errors and empty part
// lists, std::domain_error for rows masked everywhere. The math runs in fp64
// on the GPU, so the reference's own 1e-9 tolerances and golden tokens hold.
//
// Compiled against the reference headers (never copied into this repo) by
// oracle/Makefile's `dropin` target.
#include <cmath>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "edgeprompt/attention.hpp"
#include "ep/ep_attn.h"

namespace edgeprompt {

namespace {

constexpr double kNegInf = -std::numeric_limits<double>::infinity();

// One ep_handle per host thread (an ep_handle is single-thread, ep_attn.h);
// the functions stay reentrant like the reference's.
struct ThreadHandle {
    ep_handle h = nullptr;
    ~ThreadHandle() {
        if (h) ep_destroy(h);
    }
};

[[noreturn]] void rethrow(int rc, const char* where) {
    const std::string msg = std::string(where) + ": " + ep_last_error();
    switch (rc) {
    case EP_EINVAL: throw std::invalid_argument(msg);
    case EP_EMASKED: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
    }
}

ep_handle handle() {
    thread_local ThreadHandle th;
    if (!th.h) {
        const char* dev = std::getenv("EP_DEVICE");
        const int rc = ep_create(dev ? std::atoi(dev) : 0, &th.h);
        if (rc != EP_OK) rethrow(rc, "edgeprompt drop-in: ep_create");
    }
    return th.h;
}

// attention.cpp:14-25 — same checks and messages.
void check_qkv_shapes(const Matrix& q, const Matrix& k, const Matrix& v, const char* where) {
    if (q.cols() == 0) throw std::invalid_argument(std::string(where) + ": zero head width");
    if (k.cols() != q.cols()) {
        throw std::invalid_argument(std::string(where) + ": q is " + std::to_string(q.rows()) +
                                    "x" + std::to_string(q.cols()) + " but k is " +
                                    std::to_string(k.rows()) + "x" + std::to_string(k.cols()));
    }
    if (k.rows() != v.rows()) {
        throw std::invalid_argument(std::string(where) + ": k has " + std::to_string(k.rows()) +
                                    " rows but v has " + std::to_string(v.rows()));
    }
    // The C-ABI carries one head width for q, k and v (every reference caller
    // slices K and V to the same d_head, model.cpp:171-177).
    if (v.cols() != q.cols()) {
        throw std::invalid_argument(std::string(where) + ": v width " + std::to_string(v.cols()) +
                                    " differs from head width " + std::to_string(q.cols()));
    }
}

}  // namespace

PartialAttention PartialAttention::identity(std::size_t n_query, std::size_t d_head) {
    PartialAttention p;
    p.out = Matrix(n_query, d_head);
    p.lse.assign(n_query, kNegInf);
    p.n_keys = 0;
    return p;
}

Matrix full_attention(const Matrix& q, const Matrix& k, const Matrix& v, CausalSpan span) {
    check_qkv_shapes(q, k, v, "full_attention");
    Matrix out(q.rows(), v.cols());
    if (q.rows() == 0) return out;
    const int rc = ep_full_attention_f64(handle(), q.data().data(), q.rows(), k.data().data(),
                                         v.data().data(), k.rows(), q.cols(), span.query_offset,
                                         span.key_offset, out.data().data());
    if (rc != EP_OK) rethrow(rc, "full_attention");
    return out;
}

PartialAttention partial_attention(const Matrix& q, const Matrix& seg_k, const Matrix& seg_v,
                                   CausalSpan span) {
    check_qkv_shapes(q, seg_k, seg_v, "partial_attention");
    PartialAttention part;
    part.out = Matrix(q.rows(), seg_v.cols());
    part.lse.assign(q.rows(), kNegInf);
    part.n_keys = seg_k.rows();
    if (q.rows() == 0) return part;
    const int rc = ep_partial_attention_f64(handle(), q.data().data(), q.rows(),
                                            seg_k.data().data(), seg_v.data().data(),
                                            seg_k.rows(), q.cols(), span.query_offset,
                                            span.key_offset, part.out.data().data(),
                                            part.lse.data());
    if (rc != EP_OK) rethrow(rc, "partial_attention");
    return part;
}

PartialAttention merge_partials(const std::vector<PartialAttention>& parts) {
    if (parts.empty()) throw std::invalid_argument("merge_partials: no partials");
    const std::size_t n_query = parts.front().out.rows();
    const std::size_t d_head = parts.front().out.cols();
    std::size_t n_keys = 0;
    std::vector<const double*> outs, lses;
    for (const auto& p : parts) {
        if (p.out.rows() != n_query || p.out.cols() != d_head || p.lse.size() != n_query) {
            throw std::invalid_argument("merge_partials: partials disagree on shape");
        }
        n_keys += p.n_keys;
        outs.push_back(p.out.data().data());
        lses.push_back(p.lse.data());
    }
    PartialAttention merged;
    merged.out = Matrix(n_query, d_head);
    merged.lse.assign(n_query, kNegInf);
    merged.n_keys = n_keys;
    if (n_query == 0 || d_head == 0) return merged;
    const int rc = ep_merge_partials_f64(handle(), parts.size(), outs.data(), lses.data(), n_query,
                                         d_head, merged.out.data().data(), merged.lse.data());
    if (rc != EP_OK) rethrow(rc, "merge_partials");
    return merged;
}

Matrix fuse_partials(const std::vector<PartialAttention>& parts) {
    PartialAttention merged = merge_partials(parts);
    for (std::size_t i = 0; i < merged.lse.size(); ++i) {
        if (std::isinf(merged.lse[i]) && merged.lse[i] < 0) {
            throw std::domain_error("fuse_partials: query row " + std::to_string(i) +
                                    " is masked in every partial");
        }
    }
    return std::move(merged.out);
}

}  // namespace edgeprompt
