// capi.cpp — implementation of include/ep/ep_attn.h (host side of libep_b200.so).
//
// Sections mirror the header: (1) the synchronous host-buffer drop-in entry
// points that replace attention.cpp's functions, (2) device-pointer variants,
// (3) the paged splice-table plan + K1/K2 launch, (4) utilities.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "ep_internal.h"

namespace ep {

namespace {
thread_local std::string g_err;
}

int fail(int rc, const std::string& msg) {
    g_err = msg;
    return rc;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(EP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

DeviceBuffer::~DeviceBuffer() {
    if (ptr && !view) cudaFree(ptr);
}

cudaError_t DeviceBuffer::reserve(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (view) return cudaErrorInvalidValue;  // views are sized by their owner
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&ptr, n);
    if (e == cudaSuccess) bytes = n;
    return e;
}

}  // namespace ep

using namespace ep;

namespace ep {
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
// A row-major bf16 matrix [outer][inner] with box [box_outer][box_inner],
// 128B swizzle (box_inner * 2 == 128).
int encode_bf16_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint32_t box_inner, uint32_t box_outer) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f)
            return fail(EP_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * 2};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(EP_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return EP_OK;
}

// The KV pool as a 2-D tensor of 128-element bf16 rows (one row per (page,
// head, slot)); 64 x 64 boxes with 128B swizzle are exactly the UMMA K-major
// (K tiles) / MN-major (V tiles) canonical layouts.
//
// As a 3-D tensor {64 d, rows, 2 d-halves} (strides 256 B, 128 B) one box
// {64, 64, 2} moves a whole 64-row block in the [d-half][row][64] layout K3
// uses: one TMA instruction per K or V block instead of two.
int encode_kv_map(CUtensorMap* map, const void* base, int64_t rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !f)
            return fail(EP_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    const cuuint64_t dims[3] = {64, uint64_t(rows), 2};
    const cuuint64_t strides[2] = {256, 128};
    const cuuint32_t box[3] = {64, 64, 2};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(EP_ECUDA, "cuTensorMapEncodeTiled (KV, 3-D) failed: " + std::to_string(int(r)));
    return EP_OK;
}

bool force_tc() {
    static const bool f = [] {
        const char* e = std::getenv("EP_FORCE_TC");
        return e && e[0] == '1';
    }();
    return f;
}

}  // namespace ep

namespace {

bool valid_dt(int dt) { return dt == EP_F32 || dt == EP_BF16; }

}  // namespace

extern "C" {

int ep_abi_version(void) { return EP_ABI_VERSION; }

const char* ep_last_error(void) { return ep::g_err.c_str(); }

int ep_create(int device, ep_handle* out) {
    if (!out) return fail(EP_EINVAL, "ep_create: null out");
    *out = nullptr;
    int n = 0;
    EP_CUDA_TRY(cudaGetDeviceCount(&n), "ep_create");
    if (device < 0 || device >= n) return fail(EP_EINVAL, "ep_create: no CUDA device " + std::to_string(device));
    EP_CUDA_TRY(cudaSetDevice(device), "ep_create");
    cudaDeviceProp prop;
    EP_CUDA_TRY(cudaGetDeviceProperties(&prop, device), "ep_create");
    if (prop.major != 10)
        return fail(EP_EUNSUPPORTED, std::string("ep_create: built for sm_100a (B200), device is ") + prop.name);
    auto* h = new (std::nothrow) ep_context();
    if (!h) return fail(EP_ENOMEM, "ep_create: host alloc");
    h->device = device;
    h->n_sms = prop.multiProcessorCount;
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = h->zero_rows.reserve(64 * 128 * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(h->zero_rows.ptr, 0, h->zero_rows.bytes);
    if (e != cudaSuccess) {
        if (h->stream) cudaStreamDestroy(h->stream);
        delete h;
        return cuda_fail(e, "ep_create");
    }
    *out = h;
    return EP_OK;
}

int ep_destroy(ep_handle h) {
    if (!h) return EP_OK;
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamDestroy(h->stream);
    if (h->hdr_pinned) cudaFreeHost(h->hdr_pinned);
    if (h->pin) cudaFreeHost(h->pin);
    if (h->ingest_status) cudaFreeHost(h->ingest_status);
    if (h->ingest_done) {
        cudaEventSynchronize(h->ingest_done);
        cudaEventDestroy(h->ingest_done);
    }
    delete h;
    return EP_OK;
}

int64_t ep_launch_count(ep_handle h) { return h ? h->launches.load() : 0; }

// ------------------------------------------------ (1) host-buffer drop-in --

namespace {

int check_head(size_t d, const char* where) {
    if (d == 0) return fail(EP_EINVAL, std::string(where) + ": zero head width");
    if (d > 256) return fail(EP_EUNSUPPORTED, std::string(where) + ": head width > 256");
    return EP_OK;
}

// Pinned staging area of the synchronous host-buffer calls: the inputs are
// packed into it and cross PCIe in one copy each way (pageable sources
// would cost the driver a staging copy per argument).
cudaError_t reserve_pin(ep_context* h, size_t n) {
    if (n <= h->pin_bytes) return cudaSuccess;
    if (h->pin) cudaFreeHost(h->pin);
    h->pin = nullptr;
    h->pin_bytes = 0;
    const size_t cap = std::max(n, size_t(1) << 20);
    cudaError_t e = cudaMallocHost(&h->pin, cap);
    if (e == cudaSuccess) h->pin_bytes = cap;
    return e;
}

size_t visible(size_t q_off, size_t k_off, size_t n_keys, size_t i) {
    const size_t qpos = q_off + i;
    if (qpos < k_off) return 0;
    return std::min(n_keys, qpos - k_off + 1);
}

}  // namespace

int ep_partial_attention_f64(ep_handle h, const double* q, size_t n_q, const double* k,
                             const double* v, size_t n_keys, size_t d, size_t query_offset,
                             size_t key_offset, double* out, double* lse) {
    if (!h) return fail(EP_EINVAL, "partial_attention: null handle");
    if (int rc = check_head(d, "partial_attention")) return rc;
    if (n_q == 0) return EP_OK;
    const size_t nq = n_q * d, nk = n_keys * d;
    const size_t total = (2 * nq + 2 * nk + n_q) * sizeof(double);
    EP_CUDA_TRY(cudaSetDevice(h->device), "partial_attention");
    EP_CUDA_TRY(h->scratch.reserve(total), "partial_attention scratch");
    double* dq = static_cast<double*>(h->scratch.ptr);
    double* dk = dq + nq;
    double* dv = dk + nk;
    double* dout = dv + nk;
    double* dlse = dout + nq;
    cudaStream_t s = h->stream;
    // q | k | v packed in pinned memory -> one H2D; out | lse (adjacent on
    // the device) -> one D2H
    EP_CUDA_TRY(reserve_pin(h, total), "partial_attention pinned staging");
    double* hp = static_cast<double*>(h->pin);
    std::memcpy(hp, q, nq * sizeof(double));
    if (nk) {
        std::memcpy(hp + nq, k, nk * sizeof(double));
        std::memcpy(hp + nq + nk, v, nk * sizeof(double));
    }
    EP_CUDA_TRY(cudaMemcpyAsync(dq, hp, (nq + 2 * nk) * sizeof(double), cudaMemcpyHostToDevice, s), "H2D q|k|v");
    EP_CUDA_TRY(launch_partial_generic(EP_F64, dq, d, n_q, dk, d, dv, d, n_keys, d, query_offset,
                                       key_offset, dout, d, dlse, s),
                "partial_attention launch");
    h->launches++;
    EP_CUDA_TRY(cudaMemcpyAsync(hp, dout, (nq + n_q) * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H out|lse");
    EP_CUDA_TRY(cudaStreamSynchronize(s), "partial_attention sync");
    std::memcpy(out, hp, nq * sizeof(double));
    std::memcpy(lse, hp + nq, n_q * sizeof(double));
    return EP_OK;
}

int ep_full_attention_f64(ep_handle h, const double* q, size_t n_q, const double* k,
                          const double* v, size_t n_keys, size_t d, size_t query_offset,
                          size_t key_offset, double* out) {
    if (!h) return fail(EP_EINVAL, "full_attention: null handle");
    if (int rc = check_head(d, "full_attention")) return rc;
    for (size_t i = 0; i < n_q; ++i)
        if (visible(query_offset, key_offset, n_keys, i) == 0)
            return fail(EP_EMASKED, "full_attention: query at position " +
                                        std::to_string(query_offset + i) + " has no visible key");
    std::vector<double> lse(n_q);
    return ep_partial_attention_f64(h, q, n_q, k, v, n_keys, d, query_offset, key_offset, out,
                                    lse.data());
}

int ep_merge_partials_f64(ep_handle h, size_t n_parts, const double* const* outs,
                          const double* const* lses, size_t n_q, size_t d, double* out,
                          double* lse) {
    if (!h) return fail(EP_EINVAL, "merge_partials: null handle");
    if (n_parts == 0) return fail(EP_EINVAL, "merge_partials: no partials");
    if (n_q == 0 || d == 0) return EP_OK;
    const size_t per = n_q * d;
    const size_t total = (n_parts * (per + n_q) + per + n_q) * sizeof(double);
    EP_CUDA_TRY(cudaSetDevice(h->device), "merge_partials");
    EP_CUDA_TRY(h->scratch.reserve(total), "merge_partials scratch");
    double* d_outs = static_cast<double*>(h->scratch.ptr);
    double* d_lses = d_outs + n_parts * per;
    double* d_out = d_lses + n_parts * n_q;
    double* d_lse = d_out + per;
    cudaStream_t s = h->stream;
    // every partial (outs, then lses) packed in pinned memory -> one H2D;
    // out | lse (adjacent on the device) -> one D2H
    EP_CUDA_TRY(reserve_pin(h, total), "merge_partials pinned staging");
    double* hp = static_cast<double*>(h->pin);
    for (size_t p = 0; p < n_parts; ++p) {
        std::memcpy(hp + p * per, outs[p], per * sizeof(double));
        std::memcpy(hp + n_parts * per + p * n_q, lses[p], n_q * sizeof(double));
    }
    EP_CUDA_TRY(cudaMemcpyAsync(d_outs, hp, n_parts * (per + n_q) * sizeof(double), cudaMemcpyHostToDevice, s),
                "H2D partials");
    EP_CUDA_TRY(launch_merge_generic(EP_F64, n_parts, d_outs, d_lses, n_q, d, d_out, d_lse, s),
                "merge_partials launch");
    h->launches++;
    EP_CUDA_TRY(cudaMemcpyAsync(hp, d_out, (per + n_q) * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H out|lse");
    EP_CUDA_TRY(cudaStreamSynchronize(s), "merge_partials sync");
    std::memcpy(out, hp, per * sizeof(double));
    std::memcpy(lse, hp + per, n_q * sizeof(double));
    return EP_OK;
}

int ep_fuse_partials_f64(ep_handle h, size_t n_parts, const double* const* outs,
                         const double* const* lses, size_t n_q, size_t d, double* out) {
    std::vector<double> lse(n_q);
    int rc = ep_merge_partials_f64(h, n_parts, outs, lses, n_q, d, out, lse.data());
    if (rc) return rc;
    for (size_t i = 0; i < n_q; ++i)
        if (std::isinf(lse[i]) && lse[i] < 0)
            return fail(EP_EMASKED, "fuse_partials: query row " + std::to_string(i) +
                                        " is masked in every partial");
    return EP_OK;
}

// -------------------------------------------------- (2) device pointers --

int ep_partial_attention_dev(ep_handle h, ep_dtype dt, const void* q, size_t ldq, size_t n_q,
                             const void* k, size_t ldk, const void* v, size_t ldv,
                             size_t n_keys, size_t d, size_t query_offset, size_t key_offset,
                             void* out, size_t ldo, void* lse, ep_stream stream) {
    if (!h) return fail(EP_EINVAL, "partial_attention_dev: null handle");
    if (dt != EP_F64 && dt != EP_F32) return fail(EP_EUNSUPPORTED, "partial_attention_dev: dtype");
    if (int rc = check_head(d, "partial_attention_dev")) return rc;
    if (ldq < d || ldk < d || ldv < d || ldo < d)
        return fail(EP_EINVAL, "partial_attention_dev: leading dimension < d");
    EP_CUDA_TRY(launch_partial_generic(dt, q, ldq, n_q, k, ldk, v, ldv, n_keys, d, query_offset,
                                       key_offset, out, ldo, lse, static_cast<cudaStream_t>(stream)),
                "partial_attention_dev launch");
    if (n_q) h->launches++;
    return EP_OK;
}

int ep_merge_partials_dev(ep_handle h, ep_dtype dt, size_t n_parts, const void* outs,
                          const void* lses, size_t rows, size_t d, void* out, void* lse,
                          ep_stream stream) {
    if (!h) return fail(EP_EINVAL, "merge_partials_dev: null handle");
    if (dt != EP_F64 && dt != EP_F32) return fail(EP_EUNSUPPORTED, "merge_partials_dev: dtype");
    if (n_parts == 0) return fail(EP_EINVAL, "merge_partials: no partials");
    EP_CUDA_TRY(launch_merge_generic(dt, n_parts, outs, lses, rows, d, out, lse,
                                     static_cast<cudaStream_t>(stream)),
                "merge_partials_dev launch");
    if (rows) h->launches++;
    return EP_OK;
}

int ep_merge_partials_packed_dev(ep_handle h, int32_t n_parts, const float* packed, int32_t rows,
                                 int32_t d, int32_t out_dtype, void* out, float* lse,
                                 ep_stream stream) {
    if (!h || !packed || !out) return fail(EP_EINVAL, "merge_partials_packed: null argument");
    if (n_parts <= 0) return fail(EP_EINVAL, "merge_partials: no partials");
    if (d <= 0 || d > 256) return fail(EP_EUNSUPPORTED, "merge_partials_packed: d must be 1..256");
    if (out_dtype != EP_F32 && out_dtype != EP_BF16) return fail(EP_EUNSUPPORTED, "merge_partials_packed: out dtype");
    EP_CUDA_TRY(launch_merge_packed(n_parts, packed, rows, d, out, out_dtype, lse,
                                    static_cast<cudaStream_t>(stream)),
                "merge_partials_packed launch");
    if (rows > 0) h->launches++;
    return EP_OK;
}

int ep_kv_append(ep_handle h, const ep_kv_pool* pool, int32_t n_rows, const int32_t* dst_page,
                 const int32_t* dst_slot, const void* k_new, const void* v_new,
                 ep_stream stream) {
    if (!h || !pool) return fail(EP_EINVAL, "ep_kv_append: null argument");
    if (!valid_dt(pool->dtype)) return fail(EP_EUNSUPPORTED, "ep_kv_append: kv dtype");
    const int row_bytes = pool->d_head * (pool->dtype == EP_BF16 ? 2 : 4);
    if (row_bytes % 16) return fail(EP_EUNSUPPORTED, "ep_kv_append: row must be a multiple of 16 bytes");
    EP_CUDA_TRY(launch_kv_append(row_bytes, pool->n_kv_heads, pool->page_tokens, n_rows, dst_page,
                                 dst_slot, k_new, v_new, pool->k_pages, pool->v_pages,
                                 static_cast<cudaStream_t>(stream), pool->num_pages),
                "ep_kv_append launch");
    if (n_rows > 0) h->launches++;
    return EP_OK;
}

// ------------------------------------------------------- verify (K4) --

struct ep_verifier_s {
    ep_handle h = nullptr;
    int32_t width = 0, vocab = 0;
    const void* w_t = nullptr;
    CUtensorMap tmap_w{};
    DeviceBuffer colsum, mean, rstd, best, split, wmax2, ebound, cand_cnt, cand_n, cand_z, req_count;
    size_t req_count_n = 0;
    DeviceBuffer sk_ws, sk_flags;  // stream-K score GEMM partial tiles and their flags
    bool sk_ready = false;
    CUtensorMap tmap_a{};
    const void* a_ptr = nullptr;
    int32_t a_rows = -1, a_dtype = -1;
    int32_t w_tn = -1;  // tile width tmap_w was encoded for (the W box is 64 x tn)
};

int ep_verifier_create(ep_handle h, int32_t width, int32_t vocab, const void* w_score_t,
                       ep_verifier* out) {
    if (!h || !out || !w_score_t) return fail(EP_EINVAL, "ep_verifier_create: null argument");
    *out = nullptr;
    if (width <= 0 || width % 64 || vocab <= 0 || vocab % 256)
        return fail(EP_EUNSUPPORTED, "ep_verifier_create: width must be a multiple of 64 and vocab of 256");
    std::unique_ptr<ep_verifier_s> v(new (std::nothrow) ep_verifier_s());
    if (!v) return fail(EP_ENOMEM, "ep_verifier_create");
    v->h = h;
    v->width = width;
    v->vocab = vocab;
    v->w_t = w_score_t;
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_verifier_create");
    EP_CUDA_TRY(v->colsum.reserve(size_t(vocab) * sizeof(float)), "ep_verifier_create colsum");
    EP_CUDA_TRY(v->wmax2.reserve(sizeof(float)), "ep_verifier_create colnorm");
    EP_CUDA_TRY(launch_colsum(w_score_t, width, vocab, static_cast<float*>(v->colsum.ptr),
                              static_cast<float*>(v->wmax2.ptr), h->stream),
                "colsum launch");
    h->launches += 2;
    EP_CUDA_TRY(cudaStreamSynchronize(h->stream), "ep_verifier_create sync");
    *out = v.release();
    return EP_OK;
}

int ep_verifier_destroy(ep_verifier v) {
    delete v;
    return EP_OK;
}

int ep_verify_greedy(ep_handle h, ep_verifier v, int32_t batch, int32_t n_q, int32_t attn_dtype,
                     const void* attn_out, const int32_t* drafts, int32_t* target_ids,
                     int32_t* n_accepted, float* logits, ep_stream stream) {
    if (!h || !v || !attn_out || !target_ids || !n_accepted || (n_q > 1 && !drafts))
        return fail(EP_EINVAL, "ep_verify_greedy: null argument");
    if (batch <= 0 || n_q <= 0) return fail(EP_EINVAL, "ep_verify_greedy: batch/n_q");
    if (attn_dtype != EP_F32 && attn_dtype != EP_BF16)
        return fail(EP_EUNSUPPORTED, "ep_verify_greedy: attn_out must be f32 or bf16");
    const int32_t rows = batch * n_q;
    const int tn = score_tile_n(rows, v->vocab, h->n_sms);
    if (v->w_tn != tn) {
        if (int rc = encode_bf16_2d(&v->tmap_w, v->w_t, uint64_t(v->width), uint64_t(v->vocab), 64,
                                    uint32_t(score_w_box_rows(tn))))
            return rc;
        v->w_tn = tn;
    }
    EP_CUDA_TRY(v->mean.reserve(size_t(rows) * sizeof(float)), "ep_verify_greedy ws");
    EP_CUDA_TRY(v->rstd.reserve(size_t(rows) * sizeof(float)), "ep_verify_greedy ws");
    EP_CUDA_TRY(v->best.reserve(size_t(rows) * sizeof(unsigned long long)), "ep_verify_greedy ws");
    void* split = nullptr;
    const void* a_src = attn_out;
    uint64_t a_inner = uint64_t(v->width);
    RefineArgs rf;
    if (attn_dtype == EP_F32 && v->width > 4096)
        return fail(EP_EUNSUPPORTED, "ep_verify_greedy: fp32 attention rows wider than 4096");
    if (attn_dtype == EP_F32) {
        // the bf16 hi part of the rows is the GEMM's A operand
        EP_CUDA_TRY(v->split.reserve(size_t(rows) * v->width * 2), "ep_verify_greedy ws");
        EP_CUDA_TRY(v->ebound.reserve(size_t(rows) * sizeof(float)), "ep_verify_greedy ws");
        const size_t n_tiles = size_t(score_cand_tiles(v->vocab, tn));
        const size_t slots = n_tiles * kScoreCandPerTile;  // [rows][vocab tiles][per tile]
        EP_CUDA_TRY(v->cand_cnt.reserve(size_t(rows) * n_tiles * sizeof(int32_t)), "ep_verify_greedy ws");
        EP_CUDA_TRY(v->cand_n.reserve(size_t(rows) * slots * sizeof(int32_t)), "ep_verify_greedy ws");
        EP_CUDA_TRY(v->cand_z.reserve(size_t(rows) * slots * sizeof(float)), "ep_verify_greedy ws");
        split = v->split.ptr;
        a_src = split;
        rf.wt = v->w_t;
        rf.wmax2 = static_cast<const float*>(v->wmax2.ptr);
        rf.ebound = static_cast<float*>(v->ebound.ptr);
        rf.cand_cnt = static_cast<int32_t*>(v->cand_cnt.ptr);
        rf.cand_n = static_cast<int32_t*>(v->cand_n.ptr);
        rf.cand_z = static_cast<float*>(v->cand_z.ptr);
        if (size_t(batch) > v->req_count_n) {  // arrival counters start at zero; the kernel re-zeroes them
            EP_CUDA_TRY(v->req_count.reserve(size_t(batch) * sizeof(int32_t)), "ep_verify_greedy ws");
            EP_CUDA_TRY(cudaMemsetAsync(v->req_count.ptr, 0, size_t(batch) * sizeof(int32_t),
                                        static_cast<cudaStream_t>(stream)),
                        "ep_verify_greedy ws");
            v->req_count_n = size_t(batch);
        }
        rf.req_count = static_cast<int32_t*>(v->req_count.ptr);
    }
    if (score_mode() == kScoreStreamK) {
        if (!v->sk_ready) {  // flags start at zero; every launch leaves them at zero
            EP_CUDA_TRY(v->sk_ws.reserve(score_streamk_ws_bytes(h->n_sms)), "ep_verify_greedy ws");
            EP_CUDA_TRY(v->sk_flags.reserve(size_t(h->n_sms) * sizeof(unsigned int)), "ep_verify_greedy ws");
            EP_CUDA_TRY(cudaMemsetAsync(v->sk_flags.ptr, 0, size_t(h->n_sms) * sizeof(unsigned int),
                                        static_cast<cudaStream_t>(stream)),
                        "ep_verify_greedy ws");
            v->sk_ready = true;
        }
        rf.sk_ws = static_cast<float*>(v->sk_ws.ptr);
        rf.sk_flags = static_cast<unsigned int*>(v->sk_flags.ptr);
        rf.sk_ctas = h->n_sms;
    }
    if (v->a_ptr != a_src || v->a_rows != rows || v->a_dtype != attn_dtype) {
        if (int rc = encode_bf16_2d(&v->tmap_a, a_src, a_inner, uint64_t(rows), 64, 128)) return rc;
        v->a_ptr = a_src;
        v->a_rows = rows;
        v->a_dtype = attn_dtype;
    }
    EP_CUDA_TRY(launch_score_accept(rows, v->width, v->vocab, tn, attn_out, split, v->tmap_a, v->tmap_w,
                                    static_cast<const float*>(v->colsum.ptr),
                                    static_cast<float*>(v->mean.ptr), static_cast<float*>(v->rstd.ptr),
                                    static_cast<unsigned long long*>(v->best.ptr), logits, batch, n_q,
                                    drafts, target_ids, n_accepted, rf, static_cast<cudaStream_t>(stream)),
                "score/accept launch");
    h->launches += 3;
    return EP_OK;
}

// --------------------------------------------------------- (4) utilities --

int ep_fill_uniform(ep_handle h, ep_dtype dt, void* dst, size_t n, uint64_t seed, double lo,
                    double hi, ep_stream stream) {
    if (!h) return fail(EP_EINVAL, "ep_fill_uniform: null handle");
    if (dt != EP_F32 && dt != EP_BF16 && dt != EP_F64) return fail(EP_EINVAL, "ep_fill_uniform: dtype");
    EP_CUDA_TRY(launch_fill_uniform(dt, dst, n, seed, lo, hi, static_cast<cudaStream_t>(stream)),
                "ep_fill_uniform launch");
    if (n) h->launches++;
    return EP_OK;
}

}  // extern "C"
