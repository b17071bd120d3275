// ref_capi.cpp — C entry points over the UNMODIFIED reference C++ API.
//
// TEST INFRASTRUCTURE ONLY. oracle/Makefile compiles this file together with
// the reference's own sources straight from /root/reference/proj/core (never
// copied) into oracle/_ref/libep_ref.so, so Python tests and bench.py's
// reference arm can call the real edgeprompt:: functions through ctypes.
//
// The same file is linked a second time against the B200 drop-in shim
// (paper_2504_11729_b200/csrc/dropin/attention_dropin.cpp) instead of the
// reference attention.cpp, giving oracle/_ref/libep_ref_dropin.so: the
// reference model/cache code driving the GPU attention through the C-ABI.
//
// Exceptions never cross this boundary; they map to status codes:
//   0 ok, 1 std::invalid_argument, 2 std::domain_error, 3 std::out_of_range,
//   4 any other exception.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <thread>
#include <atomic>
#include <memory>
#include <vector>

#include "edgeprompt/attention.hpp"
#include "edgeprompt/cache.hpp"
#include "edgeprompt/matrix.hpp"
#include "edgeprompt/model.hpp"
#include "edgeprompt/wire.hpp"
#include "ep_oracle.h"

using namespace edgeprompt;

namespace {

thread_local char g_err[512];

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 1;
    } catch (const std::domain_error& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 2;
    } catch (const std::out_of_range& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 4;
    }
}

Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
    return Matrix(rows, cols, std::vector<double>(p, p + rows * cols));
}

double load_elem(int dtype, const void* base, std::size_t idx) {
    if (dtype == EPO_DT_BF16) {
        std::uint32_t u = static_cast<std::uint32_t>(static_cast<const std::uint16_t*>(base)[idx]) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
    if (dtype == EPO_DT_F32) return static_cast<const float*>(base)[idx];
    return static_cast<const double*>(base)[idx];
}

struct Session {
    const Model* model;
    SegmentedCache cache;
    Matrix last_hidden;
};

} // namespace

extern "C" {

const char* epref_last_error(void) { return g_err; }

double epref_log_add_exp(double a, double b) { return log_add_exp(a, b); }

std::uint32_t epref_argmax(const double* logits, std::size_t n) {
    return argmax_token(std::span<const double>(logits, n));
}

int epref_partial_attention(const double* q, std::size_t n_q, const double* k, const double* v,
                            std::size_t n_keys, std::size_t d, std::size_t q_off,
                            std::size_t k_off, double* out, double* lse) {
    return guarded([&] {
        PartialAttention p = partial_attention(to_matrix(q, n_q, d), to_matrix(k, n_keys, d),
                                               to_matrix(v, n_keys, d), CausalSpan{q_off, k_off});
        std::copy(p.out.data().begin(), p.out.data().end(), out);
        std::copy(p.lse.begin(), p.lse.end(), lse);
    });
}

int epref_full_attention(const double* q, std::size_t n_q, const double* k, const double* v,
                         std::size_t n_keys, std::size_t d, std::size_t q_off, std::size_t k_off,
                         double* out) {
    return guarded([&] {
        Matrix o = full_attention(to_matrix(q, n_q, d), to_matrix(k, n_keys, d),
                                  to_matrix(v, n_keys, d), CausalSpan{q_off, k_off});
        std::copy(o.data().begin(), o.data().end(), out);
    });
}

static std::vector<PartialAttention> gather_parts(std::size_t n_parts, const double* const* outs,
                                                  const double* const* lses, std::size_t n_q,
                                                  std::size_t d) {
    std::vector<PartialAttention> parts(n_parts);
    for (std::size_t p = 0; p < n_parts; ++p) {
        parts[p].out = to_matrix(outs[p], n_q, d);
        parts[p].lse.assign(lses[p], lses[p] + n_q);
    }
    return parts;
}

int epref_merge_partials(std::size_t n_parts, const double* const* outs, const double* const* lses,
                         std::size_t n_q, std::size_t d, double* out, double* lse) {
    return guarded([&] {
        PartialAttention m = merge_partials(gather_parts(n_parts, outs, lses, n_q, d));
        std::copy(m.out.data().begin(), m.out.data().end(), out);
        std::copy(m.lse.begin(), m.lse.end(), lse);
    });
}

int epref_fuse_partials(std::size_t n_parts, const double* const* outs, const double* const* lses,
                        std::size_t n_q, std::size_t d, double* out) {
    return guarded([&] {
        Matrix m = fuse_partials(gather_parts(n_parts, outs, lses, n_q, d));
        std::copy(m.data().begin(), m.data().end(), out);
    });
}

// The attention block of transformer_layer (model.cpp:167-181) for a batch
// of (request, q-head) units over a paged splice table: per-head K/V copies
// of every segment, partial_attention per segment, merge in segment order.
// Units run on n_threads std::threads (the functions are pure).
int epref_spliced_attention(const epo_splice_batch* s, int n_threads, const std::int64_t* unit_list,
                            std::int64_t n_units, double* out, double* lse) {
    if (!s || s->n_kv_heads <= 0 || s->n_q_heads % s->n_kv_heads != 0) return 1;
    const std::int64_t total = unit_list ? n_units : std::int64_t(s->batch) * s->n_q_heads;
    std::atomic<std::int64_t> next{0};
    std::atomic<int> rc{0};
    auto work = [&] {
        for (;;) {
            const std::int64_t i = next.fetch_add(1);
            if (i >= total) return;
            const std::int64_t unit = unit_list ? unit_list[i] : i;
            const int r = guarded([&] {
                const int Hq = s->n_q_heads, Hkv = s->n_kv_heads, d = s->d_head, P = s->page_tokens;
                const std::int64_t b = unit / Hq;
                const int h = int(unit % Hq), g = h / (Hq / Hkv);
                Matrix q(s->n_q, d);
                for (int r = 0; r < s->n_q; ++r)
                    for (int c = 0; c < d; ++c)
                        q(r, c) = load_elem(s->q_dtype, s->q,
                                            ((std::size_t(b) * s->n_q + r) * Hq + h) * d + c);
                std::vector<PartialAttention> parts;
                for (std::int64_t si = s->seg_indptr[b]; si < s->seg_indptr[b + 1]; ++si) {
                    const epo_segment& seg = s->segs[si];
                    Matrix k(seg.len, d), v(seg.len, d);
                    for (int t = 0; t < seg.len; ++t) {
                        const std::int64_t page = s->page_table[seg.page_off + t / P];
                        const std::size_t base = ((std::size_t(page) * Hkv + g) * P + t % P) * d;
                        for (int c = 0; c < d; ++c) {
                            k(t, c) = load_elem(s->kv_dtype, s->k_pages, base + c);
                            v(t, c) = load_elem(s->kv_dtype, s->v_pages, base + c);
                        }
                    }
                    parts.push_back(partial_attention(
                        q, k, v,
                        CausalSpan{std::size_t(s->q_pos[b]), std::size_t(seg.pos_offset)}));
                }
                PartialAttention m = merge_partials(parts);
                for (int r = 0; r < s->n_q; ++r) {
                    const std::size_t row = (std::size_t(b) * s->n_q + r) * Hq + h;
                    std::copy(m.out.row_ptr(r), m.out.row_ptr(r) + d, out + row * d);
                    lse[row] = m.lse[r];
                }
            });
            if (r) rc = r;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < std::max(1, n_threads); ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    return rc;
}

// The reference's own data layout for a batch: per request, fp64 KVSegments
// of seq_len x (Hkv*d) with heads concatenated (cache.hpp:15-28), gathered once
// from the pages OUTSIDE any timed region. epref_cache_attention then runs the
// attention block exactly as transformer_layer does (model.cpp:167-181):
// per-head col_slice copies, partial_attention per segment, fuse in order.
struct RefCache {
    int Hq = 0, Hkv = 0, d = 0, n_q = 0;
    std::vector<std::vector<KVSegment>> req;
    std::vector<std::size_t> q_pos;
};

void* epref_cache_create(const epo_splice_batch* s) {
    RefCache* c = nullptr;
    const int rc = guarded([&] {
        auto cc = std::make_unique<RefCache>();
        cc->Hq = s->n_q_heads;
        cc->Hkv = s->n_kv_heads;
        cc->d = s->d_head;
        cc->n_q = s->n_q;
        const int P = s->page_tokens, W = s->n_kv_heads * s->d_head;
        cc->req.resize(s->batch);
        for (int b = 0; b < s->batch; ++b) {
            cc->q_pos.push_back(std::size_t(s->q_pos[b]));
            for (std::int64_t si = s->seg_indptr[b]; si < s->seg_indptr[b + 1]; ++si) {
                const epo_segment& seg = s->segs[si];
                KVSegment ks;
                ks.origin = static_cast<SegmentOrigin>(seg.origin);
                ks.pos_offset = std::size_t(seg.pos_offset);
                ks.k = Matrix(seg.len, W);
                ks.v = Matrix(seg.len, W);
                for (int t = 0; t < seg.len; ++t) {
                    const std::int64_t page = s->page_table[seg.page_off + t / P];
                    for (int g = 0; g < s->n_kv_heads; ++g) {
                        const std::size_t base = ((std::size_t(page) * s->n_kv_heads + g) * P + t % P) * s->d_head;
                        for (int e = 0; e < s->d_head; ++e) {
                            ks.k(t, g * s->d_head + e) = load_elem(s->kv_dtype, s->k_pages, base + e);
                            ks.v(t, g * s->d_head + e) = load_elem(s->kv_dtype, s->v_pages, base + e);
                        }
                    }
                }
                cc->req[b].push_back(std::move(ks));
            }
        }
        c = cc.release();
    });
    return rc ? nullptr : c;
}

void epref_cache_destroy(void* c) { delete static_cast<RefCache*>(c); }

int epref_cache_attention(const void* cv, const double* q, int n_threads, const std::int64_t* unit_list,
                          std::int64_t n_units, double* out, double* lse) {
    const RefCache& c = *static_cast<const RefCache*>(cv);
    const std::int64_t total = unit_list ? n_units : std::int64_t(c.req.size()) * c.Hq;
    std::atomic<std::int64_t> next{0};
    std::atomic<int> rc{0};
    auto work = [&] {
        std::vector<PartialAttention> parts;
        for (;;) {
            const std::int64_t i = next.fetch_add(1);
            if (i >= total) return;
            const std::int64_t unit = unit_list ? unit_list[i] : i;
            const int r = guarded([&] {
                const std::int64_t b = unit / c.Hq;
                const int h = int(unit % c.Hq), g = h / (c.Hq / c.Hkv), d = c.d;
                Matrix qh(c.n_q, d);
                for (int row = 0; row < c.n_q; ++row)
                    for (int e = 0; e < d; ++e)
                        qh(row, e) = q[((std::size_t(b) * c.n_q + row) * c.Hq + h) * d + e];
                parts.clear();
                for (const KVSegment& seg : c.req[b])
                    parts.push_back(partial_attention(qh, seg.k.col_slice(g * d, d),
                                                      seg.v.col_slice(g * d, d),
                                                      CausalSpan{c.q_pos[b], seg.pos_offset}));
                PartialAttention m = merge_partials(parts);
                for (int row = 0; row < c.n_q; ++row) {
                    const std::size_t orow = (std::size_t(b) * c.n_q + row) * c.Hq + h;
                    std::copy(m.out.row_ptr(row), m.out.row_ptr(row) + d, out + orow * d);
                    lse[orow] = m.lse[row];
                }
            });
            if (r) rc = r;
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < std::max(1, n_threads); ++t) th.emplace_back(work);
    work();
    for (auto& t : th) t.join();
    return rc;
}

// ---------------------------------------------------------------- model ---

void* epref_model_create(std::size_t n_layers, std::size_t n_heads, std::size_t d_model,
                         std::size_t vocab, std::size_t max_positions, std::uint64_t seed) {
    Model* m = nullptr;
    const int rc = guarded([&] {
        ModelConfig c;
        c.n_layers = n_layers;
        c.n_heads = n_heads;
        c.d_model = d_model;
        c.vocab_size = vocab;
        c.max_positions = max_positions;
        c.init_seed = seed;
        m = new Model(init_model(c));
    });
    return rc ? nullptr : m;
}

void epref_model_destroy(void* m) { delete static_cast<Model*>(m); }

double epref_model_weight_sum(const void* m) { return static_cast<const Model*>(m)->weight_sum(); }

int epref_generate_split(const void* m, const std::uint32_t* cloud, std::size_t n_cloud,
                         const std::uint32_t* edge, std::size_t n_edge, std::size_t n_steps,
                         std::uint32_t* out) {
    return guarded([&] {
        auto toks = generate_split(*static_cast<const Model*>(m),
                                   std::vector<TokenId>(cloud, cloud + n_cloud),
                                   std::vector<TokenId>(edge, edge + n_edge), n_steps);
        std::copy(toks.begin(), toks.end(), out);
    });
}

int epref_generate_monolithic(const void* m, const std::uint32_t* prompt, std::size_t n,
                              std::size_t n_steps, std::uint32_t* out) {
    return guarded([&] {
        auto toks = generate_monolithic(*static_cast<const Model*>(m),
                                        std::vector<TokenId>(prompt, prompt + n), n_steps);
        std::copy(toks.begin(), toks.end(), out);
    });
}

// A split session (cloud prefill, edge prefill against it — the in-process
// generate_split of model.cpp:307-316) kept alive so tests can read the real
// spliced cache and step decode_step one token at a time.
void* epref_session_create(const void* m, const std::uint32_t* cloud, std::size_t n_cloud,
                           const std::uint32_t* edge, std::size_t n_edge) {
    Session* s = nullptr;
    const int rc = guarded([&] {
        const Model& model = *static_cast<const Model*>(m);
        auto sess = new Session{&model, SegmentedCache(model.config.n_layers), Matrix()};
        PrefillResult c = prefill(model, std::vector<TokenId>(cloud, cloud + n_cloud),
                                  SegmentOrigin::cloud, 0, sess->cache);
        sess->cache.append(std::move(c.segments));
        PrefillResult e = prefill(model, std::vector<TokenId>(edge, edge + n_edge),
                                  SegmentOrigin::edge, n_cloud, sess->cache);
        sess->cache.append(std::move(e.segments));
        sess->last_hidden = std::move(e.hidden);
        s = sess;
    });
    return rc ? nullptr : s;
}

void epref_session_destroy(void* s) { delete static_cast<Session*>(s); }

std::size_t epref_session_n_segments(const void* s) {
    return static_cast<const Session*>(s)->cache.layer(0).size();
}

std::size_t epref_session_end_position(const void* s) {
    return static_cast<const Session*>(s)->cache.end_position();
}

// Copies segment seg of layer l (K and V, seq_len x d_model, heads concatenated).
int epref_session_segment(const void* s, std::size_t l, std::size_t seg, double* k, double* v,
                          std::size_t* seq_len, std::size_t* pos_offset, int* origin) {
    return guarded([&] {
        const KVSegment& g = static_cast<const Session*>(s)->cache.layer(l).at(seg);
        if (k) std::copy(g.k.data().begin(), g.k.data().end(), k);
        if (v) std::copy(g.v.data().begin(), g.v.data().end(), v);
        *seq_len = g.seq_len();
        *pos_offset = g.pos_offset;
        *origin = static_cast<int>(g.origin);
    });
}

// First greedy token from the prefill hidden row (decode_greedy, model.cpp:285-297).
int epref_session_first_token(const void* s, std::uint32_t* tok) {
    return guarded([&] {
        const Session* ss = static_cast<const Session*>(s);
        auto lg = unembed_logits(*ss->model, ss->last_hidden.row(ss->last_hidden.rows() - 1));
        *tok = argmax_token(lg);
    });
}

int epref_session_decode_step(void* s, std::uint32_t last, double* logits, std::uint32_t* next) {
    return guarded([&] {
        Session* ss = static_cast<Session*>(s);
        DecodeResult r = decode_step(*ss->model, ss->cache, last);
        if (logits) std::copy(r.logits.begin(), r.logits.end(), logits);
        *next = r.next_token;
    });
}

// Speculative verify as SURVEY §8a a16 constructs it from the reference's own
// functions: prefill (model.cpp:211-236) of [last, d1..dk] as a generated
// segment at the cache end, then unembed_logits + argmax_token per row
// (model.cpp:238-255). The session's cache is left unchanged (prefill returns
// its segment; it is dropped here).
int epref_session_verify(const void* s, const std::uint32_t* toks, std::size_t n, double* logits,
                         std::uint32_t* targets) {
    return guarded([&] {
        const Session* ss = static_cast<const Session*>(s);
        PrefillResult r = prefill(*ss->model, std::vector<TokenId>(toks, toks + n), SegmentOrigin::generated,
                                  ss->cache.end_position(), ss->cache);
        const std::size_t V = ss->model->config.vocab_size;
        for (std::size_t i = 0; i < n; ++i) {
            auto lg = unembed_logits(*ss->model, r.hidden.row(i));
            if (logits) std::copy(lg.begin(), lg.end(), logits + i * V);
            targets[i] = argmax_token(lg);
        }
    });
}

// ---------------------------------------------------------------- wire --
// The reference's own EPKV codec (wire.cpp): encode a kv frame, decode any
// frame and report its WireError kind (wire.hpp:94-104) + 1, or 6 when the
// frame is valid but not a kv frame.

std::size_t epref_kv_frame_encode(const epo_kv_frame_info* info, const double* k, const double* v,
                                  std::uint8_t* out, std::size_t cap) {
    wire::KVFrame f;
    f.session_id = info->session_id;
    f.layer = info->layer;
    f.seq_len = info->seq_len;
    f.n_heads = info->n_heads;
    f.d_head = info->d_head;
    const std::size_t n = f.values_per_matrix();
    f.k_data.assign(k, k + n);
    f.v_data.assign(v, v + n);
    const std::vector<std::uint8_t> bytes = wire::encode_frame(f);
    if (out && bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return bytes.size();
}

std::size_t epref_end_of_prefill_frame(std::uint8_t* out, std::size_t cap) {
    const std::vector<std::uint8_t> bytes = wire::encode_frame(wire::EndOfPrefill{});
    if (out && bytes.size() <= cap) std::memcpy(out, bytes.data(), bytes.size());
    return bytes.size();
}

int epref_kv_frame_decode(const std::uint8_t* frame, std::size_t n, epo_kv_frame_info* info,
                          double* k, double* v) {
    try {
        const wire::Message m = wire::decode_frame(std::span<const std::uint8_t>(frame, n));
        const auto* f = std::get_if<wire::KVFrame>(&m);
        if (!f) return 6;
        if (info) {
            info->session_id = f->session_id;
            info->layer = f->layer;
            info->seq_len = f->seq_len;
            info->n_heads = f->n_heads;
            info->d_head = f->d_head;
            info->pad = 0;
        }
        if (k) std::copy(f->k_data.begin(), f->k_data.end(), k);
        if (v) std::copy(f->v_data.begin(), f->v_data.end(), v);
        return 0;
    } catch (const wire::WireError& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 1 + static_cast<int>(e.kind());
    }
}

} // extern "C"
