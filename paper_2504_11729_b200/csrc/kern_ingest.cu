// kern_ingest.cu — KV ingest: one EPKV kv_frame straight into the page pool
// (SURVEY §8f rank 2).
//
// The reference's edge receives each layer's cloud-prompt KV as a kv frame
// (wire.hpp:59-75; encode_frame / decode_frame, wire.cpp:70-221), decodes
// it into two fp64 Matrices and copies them into a KVSegment
// (segment_from_frame, edge.cpp:61-67). Here the frame's little-endian
// doubles are read where they lie — device memory, or pinned host memory
// read in place over the host link — and a single pass decodes, rounds to the
// pool dtype (f64 -> bf16 / f32, round to nearest even) and scatters token t,
// head h into page page_table[t / page_tokens], slot t % page_tokens: no fp64
// staging copy, no separate convert pass. Pageable frames are staged into a
// per-handle device buffer first.
//
// Byte work, bound by the host link (pinned frames) or HBM (device frames):
// per value 8 B read, 2 B (bf16) or 4 B (fp32) written.
#include <cstdint>
#include <cstring>
#include <string>

#include "ep_common.cuh"
#include "ep_internal.h"

namespace ep {
namespace {

// Correctly rounded f64 -> bf16 (RNE): f64 -> f32 rounded to odd (toward
// zero, sticky bit on inexact), then f32 -> bf16 RNE; the 16 guard bits make
// the double rounding exact. Same rule as oracle/ep_oracle.c epo_f64_to_bf16.
__device__ __forceinline__ uint16_t f64_to_bf16(double x) {
    if (x != x) return 0x7FC0;
    float f = __double2float_rz(x);
    if (double(f) != x) f = __uint_as_float(__float_as_uint(f) | 1u);
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// Two values at once: fp64 -> fp32 round-to-odd each (exact double rounding,
// as f64_to_bf16), then one packed RNE conversion; NaN -> 0x7FC0 like the
// scalar rule (checked on the fp32 value: an fp64 NaN stays NaN).
__device__ __forceinline__ uint32_t f64x2_to_bf16x2(double x0, double x1) {
    float f0 = __double2float_rz(x0), f1 = __double2float_rz(x1);
    if (double(f0) != x0) f0 = __uint_as_float(__float_as_uint(f0) | 1u);
    if (double(f1) != x1) f1 = __uint_as_float(__float_as_uint(f1) | 1u);
    const __nv_bfloat162 b = __floats2bfloat162_rn(f0, f1);
    uint32_t w = *reinterpret_cast<const uint32_t*>(&b);
    if (f0 != f0) w = (w & 0xFFFF0000u) | 0x7FC0u;
    if (f1 != f1) w = (w & 0x0000FFFFu) | 0x7FC00000u;
    return w;
}

__host__ __device__ inline uint32_t rd_u32(const uint8_t* b) {
    return uint32_t(b[0]) | (uint32_t(b[1]) << 8) | (uint32_t(b[2]) << 16) | (uint32_t(b[3]) << 24);
}
__host__ __device__ inline uint16_t rd_u16(const uint8_t* b) { return uint16_t(b[0] | (b[1] << 8)); }

const char* kWireKind[] = {"ok", "bad_magic", "bad_version", "truncated", "length_overflow", "malformed",
                           "not a kv frame"};

// Why a frame fails (selects the message; the kind is what the reference throws).
enum WhyCode : int {
    kWhyNone, kWhyShort, kWhyMagic, kWhyVersion, kWhyType, kWhyLenLimit, kWhyLenMismatch, kWhyOtherPayload,
    kWhyNotKv, kWhyKvTruncated, kWhyKvShape
};

// decode_header + decode_frame + the kv_frame payload header (wire.cpp:138-221)
// on min(24, n) leading bytes of an n-byte frame: returns the WireError kind
// + 1 (0 = a valid kv frame, 6 = a valid frame of another type) and the
// reason; fills f. Host (synchronous check) and device (deferred check).
__host__ __device__ inline int parse_kv_core(const uint8_t* hdr, size_t n, ep_kv_frame_info* f, int* why) {
    *why = kWhyNone;
    if (n < 10) { *why = kWhyShort; return 3; }
    if (hdr[0] != 'E' || hdr[1] != 'P' || hdr[2] != 'K' || hdr[3] != 'V') { *why = kWhyMagic; return 1; }
    if (hdr[4] != 0x01) { *why = kWhyVersion; return 2; }
    if (hdr[5] > 4) { *why = kWhyType; return 5; }
    const uint32_t len = rd_u32(hdr + 6);
    if (len > (1u << 30)) { *why = kWhyLenLimit; return 4; }
    if (n != 10 + size_t(len)) { *why = kWhyLenMismatch; return 3; }
    // the other message types decode (or fail) as decode_payload would
    // (wire.cpp:165-184, :202-208); a valid one is "not a kv frame"
    const uint32_t need = hdr[5] == 0 ? 20u : hdr[5] == 1 ? 6u : 0u;
    if ((hdr[5] == 0 || hdr[5] == 1) && len != need) { *why = kWhyOtherPayload; return len < need ? 3 : 5; }
    if (hdr[5] == 3 && len != 0) { *why = kWhyOtherPayload; return 5; }
    if (hdr[5] == 4 && len < 4) { *why = kWhyOtherPayload; return 3; }
    if (hdr[5] != 2) { *why = kWhyNotKv; return 6; }
    if (len < 14) { *why = kWhyKvTruncated; return 3; }
    const uint8_t* p = hdr + 10;
    f->session_id = rd_u32(p);
    f->layer = rd_u16(p + 4);
    f->seq_len = rd_u32(p + 6);
    f->n_heads = rd_u16(p + 10);
    f->d_head = rd_u16(p + 12);
    const uint64_t vals = uint64_t(f->seq_len) * f->n_heads * f->d_head;
    if (uint64_t(len) - 14 != 16 * vals) { *why = kWhyKvShape; return 5; }
    return 0;
}

int parse_kv_header(const uint8_t* hdr, size_t n, ep_kv_frame_info* f, std::string* why) {
    int w = 0;
    const int kind = parse_kv_core(hdr, n, f, &w);
    const uint32_t len = n >= 10 ? rd_u32(hdr + 6) : 0;
    switch (w) {
    case kWhyNone: break;
    case kWhyShort: *why = "frame header shorter than 10 bytes"; break;
    case kWhyMagic: *why = "frame magic is not EPKV"; break;
    case kWhyVersion: *why = "unsupported protocol version " + std::to_string(hdr[4]); break;
    case kWhyType: *why = "unknown message type " + std::to_string(hdr[5]); break;
    case kWhyLenLimit: *why = "declared payload length " + std::to_string(len) + " exceeds limit"; break;
    case kWhyLenMismatch:
        *why = "frame buffer holds " + std::to_string(n) + " bytes, header declares " + std::to_string(10 + size_t(len));
        break;
    case kWhyOtherPayload:
        *why = kind == 3 ? "frame payload truncated"
               : hdr[5] == 0 ? "session init payload has trailing bytes"
               : hdr[5] == 1 ? "ack payload has trailing bytes"
                             : "end-of-prefill payload must be empty";
        break;
    case kWhyNotKv: *why = "message type " + std::to_string(hdr[5]) + " is not a kv frame"; break;
    case kWhyKvTruncated: *why = "frame payload truncated"; break;
    case kWhyKvShape: {
        const uint64_t vals = uint64_t(f->seq_len) * f->n_heads * f->d_head;
        *why = "kv frame payload length " + std::to_string(len) + " does not match shape (expected " +
               std::to_string(14 + 16 * vals) + ")";
        break;
    }
    }
    return kind;
}

// Deferred header check of ep_kv_ingest_frame_async: every CTA re-parses the
// frame's 24 leading bytes (an L2 hit after the first) against the shape the
// host derived from the frame length and the pool; on any difference the CTA
// writes nothing and CTA 0 records the first failing kind in status[0] and
// the header fields in status[1..6] (read back by ep_kv_ingest_poll).
struct HdrCheck {
    const uint8_t* frame;  // null: checked on the host already
    uint64_t frame_bytes;
    uint32_t seq_len, n_pages, page_tokens;
    uint16_t n_heads, d_head;
    int32_t* status;  // device words
};

__device__ __forceinline__ bool header_ok(const HdrCheck& c) {
    if (!c.frame) return true;
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        uint8_t hb[24];
        for (int i = 0; i < 24; ++i) hb[i] = i < int(c.frame_bytes) ? c.frame[i] : 0;
        ep_kv_frame_info f{};
        int why = 0;
        int kind = parse_kv_core(hb, c.frame_bytes, &f, &why);
        // the pool-side checks of the synchronous path (EP_EINVAL there)
        if (!kind && (f.n_heads != c.n_heads || f.d_head != c.d_head)) kind = 7;
        if (!kind && f.seq_len == 0) kind = 8;
        if (!kind && (uint64_t(f.seq_len) + c.page_tokens - 1) / c.page_tokens > c.n_pages) kind = 9;
        if (!kind && f.seq_len != c.seq_len) kind = 5;
        s_ok = kind == 0;
        if (kind && blockIdx.x == 0 && atomicCAS(c.status, 0, kind) == 0) {
            c.status[1] = int32_t(f.session_id);
            c.status[2] = int32_t(f.seq_len);
            c.status[3] = f.layer;
            c.status[4] = f.n_heads;
            c.status[5] = f.d_head;
            c.status[6] = why;
        }
    }
    __syncthreads();
    return s_ok != 0;
}

template <bool BF16, bool A16>
__global__ void __launch_bounds__(256) kv_ingest_kernel(const uint8_t* __restrict__ src,
                                                        uint32_t n_pairs, uint32_t row_pairs,
                                                        uint32_t d_pairs, uint32_t P, uint32_t H,
                                                        const int32_t* __restrict__ page_table,
                                                        void* __restrict__ kp, void* __restrict__ vp,
                                                        const HdrCheck chk) {
    if (!header_ok(chk)) return;
    constexpr int U = 4;  // pairs in flight per thread
    const uint32_t total = 2 * n_pairs;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < total; base += U * stride) {
        double2 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = base + u * stride;
            if (q < total) {
                const uint8_t* p = src + size_t(q) * 16;  // K pairs, then V pairs
                if (A16) {
                    x[u] = __ldg(reinterpret_cast<const double2*>(p));
                } else {
                    x[u].x = __ldg(reinterpret_cast<const double*>(p));
                    x[u].y = __ldg(reinterpret_cast<const double*>(p + 8));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t q = base + u * stride;
            if (q >= total) continue;
            const bool is_v = q >= n_pairs;
            const uint32_t qq = is_v ? q - n_pairs : q;
            const uint32_t t = qq / row_pairs, r = qq - t * row_pairs;
            const uint32_t h = r / d_pairs, cp = r - h * d_pairs;
            const uint32_t page = uint32_t(page_table[t / P]), slot = t % P;
            const size_t dst = ((size_t(page) * H + h) * P + slot) * d_pairs + cp;
            if (BF16) {
                const uint32_t w = uint32_t(f64_to_bf16(x[u].x)) | (uint32_t(f64_to_bf16(x[u].y)) << 16);
                static_cast<uint32_t*>(is_v ? vp : kp)[dst] = w;
            } else {
                static_cast<float2*>(is_v ? vp : kp)[dst] =
                    make_float2(__double2float_rn(x[u].x), __double2float_rn(x[u].y));
            }
        }
    }
}

// d_head % 4 == 0: one CTA per frame row (token t of K or of V; the V rows
// follow the K rows, so row r of 2*seq is contiguous at r * H*d values) and
// one thread per 4-value quad of it (32 wire bytes -> one 8-byte bf16 / 16-byte
// fp32 store). Page and slot are row-uniform; the head split is one division
// per quad. MIS8: the payload starts 8 bytes past a 16-byte boundary (it is at
// frame+24, so a 256-aligned device frame lands here): every lane reads the
// two aligned double2 (v[4j-1], v[4j]) and (v[4j+1], v[4j+2]) and takes v[4j+3]
// from the next lane's first load; the last lane of the warp, or of the row,
// reads it itself. Loops are warp-uniform so the full-mask shuffle is valid.
// DQ: d_head / 4 at compile time (16 / 32; 0 = a runtime d_quads), so the
// head split of a quad is a shift and its store address one multiply-add
// from the row's base.
template <bool BF16, bool MIS8, int DQ>
__global__ void __launch_bounds__(256) kv_ingest_rows_kernel(const uint8_t* __restrict__ src, uint32_t rows,
                                                             uint32_t seq, uint32_t row_quads, uint32_t d_quads_rt,
                                                             uint32_t P, int p_shift, uint32_t H,
                                                             const int32_t* __restrict__ page_table,
                                                             void* __restrict__ kp, void* __restrict__ vp,
                                                             const HdrCheck chk) {
    if (!header_ok(chk)) return;
    const uint32_t d_quads = DQ > 0 ? uint32_t(DQ) : d_quads_rt;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t span = (row_quads + 31) & ~31u;
    for (uint32_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const bool is_v = row >= seq;
        const uint32_t t = is_v ? row - seq : row;
        // page / slot of token t (a shift for the usual power-of-two pages)
        const uint32_t pg = p_shift >= 0 ? t >> p_shift : t / P;
        const size_t page = size_t(page_table[pg]), slot = t - pg * P;
        const uint8_t* rp = src + size_t(row) * row_quads * 32;
        const size_t row_base = (page * H * P + slot) * d_quads;  // quad index of head 0
        const size_t head_step = size_t(P) * d_quads;
        for (uint32_t j0 = threadIdx.x & ~31u; j0 < span; j0 += blockDim.x) {
            const uint32_t j = j0 + lane;
            const bool live = j < row_quads;
            double v0 = 0, v1 = 0, v2 = 0, v3 = 0;
            if (MIS8) {
                const double2* a = reinterpret_cast<const double2*>(rp + size_t(j) * 32 - 8);
                double2 lo = make_double2(0, 0), hi = make_double2(0, 0);
                if (live) { lo = __ldg(a); hi = __ldg(a + 1); }
                double nx = __shfl_down_sync(0xffffffffu, lo.x, 1);
                if (live && (lane == 31 || j + 1 >= row_quads))
                    nx = __ldg(reinterpret_cast<const double*>(rp + size_t(j) * 32 + 24));
                v0 = lo.y; v1 = hi.x; v2 = hi.y; v3 = nx;
            } else if (live) {
                const double2* a = reinterpret_cast<const double2*>(rp + size_t(j) * 32);
                const double2 lo = __ldg(a), hi = __ldg(a + 1);
                v0 = lo.x; v1 = lo.y; v2 = hi.x; v3 = hi.y;
            }
            if (!live) continue;
            const uint32_t h = j / d_quads, cq = j - h * d_quads;
            const size_t dst = row_base + h * head_step + cq;  // in quads
            if (BF16) {
                const uint2 w = make_uint2(f64x2_to_bf16x2(v0, v1), f64x2_to_bf16x2(v2, v3));
                static_cast<uint2*>(is_v ? vp : kp)[dst] = w;
            } else {
                static_cast<float4*>(is_v ? vp : kp)[dst] = make_float4(
                    __double2float_rn(v0), __double2float_rn(v1), __double2float_rn(v2), __double2float_rn(v3));
            }
        }
    }
}

}  // namespace
}  // namespace ep


using ep::fail;

namespace {

// Copies a frame payload into the per-handle staging buffer, ordered after the
// previous launch that read it (which may be on another stream).
int stage_payload(ep_context* h, const void* src, size_t bytes, cudaStream_t s, const uint8_t** out) {
    if (h->ingest_pending && bytes > h->ingest_stage.bytes)
        EP_CUDA_TRY(cudaEventSynchronize(h->ingest_done), "ep_kv_ingest_frame staging");
    EP_CUDA_TRY(h->ingest_stage.reserve(bytes), "ep_kv_ingest_frame staging");
    if (h->ingest_pending) EP_CUDA_TRY(cudaStreamWaitEvent(s, h->ingest_done, 0), "ep_kv_ingest_frame staging");
    EP_CUDA_TRY(cudaMemcpyAsync(h->ingest_stage.ptr, src, bytes, cudaMemcpyDefault, s),
                "ep_kv_ingest_frame staging copy");
    *out = static_cast<const uint8_t*>(h->ingest_stage.ptr);
    return EP_OK;
}

// One decode + convert + scatter launch over the payload at src (8-byte aligned).
int launch_ingest(ep_context* h, const ep_kv_pool* pool, uint32_t seq_len, uint32_t n_heads, uint32_t d_head,
                  const uint8_t* src, bool staged, const int32_t* page_table, const ep::HdrCheck& chk,
                  cudaStream_t s) {
    const uint64_t vals = uint64_t(seq_len) * n_heads * d_head;
    const uint32_t n_pairs = uint32_t(vals / 2), d_pairs = d_head / 2;
    const uint32_t row_pairs = n_heads * d_pairs;
    const uintptr_t mis = reinterpret_cast<uintptr_t>(src) & 15;
    const bool pool_al = (reinterpret_cast<uintptr_t>(pool->k_pages) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(pool->v_pages) & 15) == 0;
    const uint32_t P = uint32_t(pool->page_tokens), H = n_heads;
    if (d_head % 4 == 0 && pool_al) {
        const uint32_t rows = 2 * seq_len, d_quads = d_head / 4;
        const uint32_t row_quads = n_heads * d_quads;
        const uint32_t tpb = row_quads >= 256 ? 256 : ((row_quads + 31) & ~31u);
        const uint32_t grid = std::min<uint32_t>(rows, uint32_t(h->n_sms) * (2048 / tpb));
        int p_shift = -1;
        if ((P & (P - 1)) == 0)
            for (p_shift = 0; (1u << p_shift) < P; ++p_shift) {
            }
#define EP_INGEST_ROWS(BF, M8, DQ)                                                                          \
    ep::kv_ingest_rows_kernel<BF, M8, DQ><<<grid, tpb, 0, s>>>(src, rows, seq_len, row_quads, d_quads, P, p_shift, H, \
                                                               page_table, pool->k_pages, pool->v_pages, chk)
#define EP_INGEST_ROWS_DQ(BF, M8)                                      \
    do {                                                               \
        if (d_quads == 32) EP_INGEST_ROWS(BF, M8, 32);                 \
        else if (d_quads == 16) EP_INGEST_ROWS(BF, M8, 16);            \
        else EP_INGEST_ROWS(BF, M8, 0);                                \
    } while (0)
        if (pool->dtype == EP_BF16) {
            if (mis) EP_INGEST_ROWS_DQ(true, true); else EP_INGEST_ROWS_DQ(true, false);
        } else {
            if (mis) EP_INGEST_ROWS_DQ(false, true); else EP_INGEST_ROWS_DQ(false, false);
        }
#undef EP_INGEST_ROWS_DQ
#undef EP_INGEST_ROWS
    } else {
        const uint32_t total = 2 * n_pairs;
        const uint32_t blocks = std::min<uint32_t>((total + 1023) / 1024, uint32_t(h->n_sms) * 8);
#define EP_INGEST(BF, AL)                                                                              \
    ep::kv_ingest_kernel<BF, AL><<<blocks, 256, 0, s>>>(src, n_pairs, row_pairs, d_pairs, P, H, page_table, \
                                                       pool->k_pages, pool->v_pages, chk)
        if (pool->dtype == EP_BF16) {
            if (mis == 0) EP_INGEST(true, true); else EP_INGEST(true, false);
        } else {
            if (mis == 0) EP_INGEST(false, true); else EP_INGEST(false, false);
        }
#undef EP_INGEST
    }
    EP_CUDA_TRY(cudaGetLastError(), "ep_kv_ingest_frame launch");
    if (staged) {
        if (!h->ingest_done)
            EP_CUDA_TRY(cudaEventCreateWithFlags(&h->ingest_done, cudaEventDisableTiming), "ep_kv_ingest_frame");
        EP_CUDA_TRY(cudaEventRecord(h->ingest_done, s), "ep_kv_ingest_frame");
        h->ingest_pending = true;
    }
    h->launches++;
    return EP_OK;
}

int check_pool(const ep_kv_pool* pool, const char* where) {
    if (pool->dtype != EP_F32 && pool->dtype != EP_BF16)
        return fail(EP_EUNSUPPORTED, std::string(where) + ": pool dtype must be f32 or bf16");
    if (pool->d_head % 2) return fail(EP_EUNSUPPORTED, std::string(where) + ": odd d_head");
    return EP_OK;
}

}  // namespace

extern "C" int ep_kv_ingest_frame(ep_handle h, const ep_kv_pool* pool, const void* frame,
                                  size_t frame_bytes, const int32_t* page_table, int32_t n_pages,
                                  ep_kv_frame_info* info, ep_stream stream) {
    if (!h || !pool || !frame || !page_table) return fail(EP_EINVAL, "ep_kv_ingest_frame: null argument");
    if (int rc = check_pool(pool, "ep_kv_ingest_frame")) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ep_kv_frame_info f{};
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_kv_ingest_frame");
    cudaPointerAttributes at{};
    EP_CUDA_TRY(cudaPointerGetAttributes(&at, frame), "ep_kv_ingest_frame pointer attributes");
    const bool on_device = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
    const bool pinned = at.type == cudaMemoryTypeHost;
    uint8_t hdr[24] = {};
    const size_t nh = frame_bytes < 24 ? frame_bytes : 24;
    if (on_device) {
        // the header is checked on the host before launch (decode_frame's
        // errors stay synchronous): one small DMA into a pinned slot
        if (!h->hdr_pinned)
            EP_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h->hdr_pinned), 64, cudaHostAllocDefault),
                        "ep_kv_ingest_frame header slot");
        EP_CUDA_TRY(cudaMemcpyAsync(h->hdr_pinned, frame, nh, cudaMemcpyDeviceToHost, s), "ep_kv_ingest_frame header");
        EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_kv_ingest_frame header");
        std::memcpy(hdr, h->hdr_pinned, nh);
    } else {
        std::memcpy(hdr, frame, nh);
    }
    std::string why;
    const int kind = ep::parse_kv_header(hdr, frame_bytes, &f, &why);
    f.wire_error = kind;
    if (info) *info = f;
    if (kind) return fail(EP_EWIRE, std::string("wire: ") + ep::kWireKind[kind] + ": " + why);
    if (f.n_heads != pool->n_kv_heads || f.d_head != pool->d_head)
        return fail(EP_EINVAL, "ep_kv_ingest_frame: kv frame head shape (" + std::to_string(f.n_heads) + " x " +
                                   std::to_string(f.d_head) + ") does not match the pool");
    if (f.seq_len == 0) return fail(EP_EINVAL, "ep_kv_ingest_frame: kv frame with empty sequence");
    const int64_t need = (int64_t(f.seq_len) + pool->page_tokens - 1) / pool->page_tokens;
    if (n_pages < need)
        return fail(EP_EINVAL, "ep_kv_ingest_frame: " + std::to_string(f.seq_len) + " tokens need " +
                                   std::to_string(need) + " pages, got " + std::to_string(n_pages));
    const uint64_t vals = uint64_t(f.seq_len) * f.n_heads * f.d_head;
    if (vals / 2 > 0x7FFFFFFFull) return fail(EP_EUNSUPPORTED, "ep_kv_ingest_frame: frame too large");
    const uint8_t* src = static_cast<const uint8_t*>(on_device || !pinned || !at.devicePointer ? frame
                                                                                             : at.devicePointer) + 24;
    bool staged = false;
    // pageable frames, and device / pinned payloads that are not 8-byte
    // aligned (a kv frame following a 30-byte session_init frame in one
    // receive buffer), are copied into the aligned per-handle staging buffer
    if ((!on_device && !pinned) || (reinterpret_cast<uintptr_t>(src) & 7)) {
        if (int rc = stage_payload(h, static_cast<const uint8_t*>(frame) + 24, 16 * vals, s, &src)) return rc;
        staged = true;
    }
    return launch_ingest(h, pool, f.seq_len, f.n_heads, f.d_head, src, staged, page_table, ep::HdrCheck{}, s);
}

extern "C" int ep_kv_ingest_frame_async(ep_handle h, const ep_kv_pool* pool, const void* frame,
                                        size_t frame_bytes, const int32_t* page_table, int32_t n_pages,
                                        ep_stream stream) {
    if (!h || !pool || !frame || !page_table) return fail(EP_EINVAL, "ep_kv_ingest_frame_async: null argument");
    if (int rc = check_pool(pool, "ep_kv_ingest_frame_async")) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_kv_ingest_frame_async");
    cudaPointerAttributes at{};
    EP_CUDA_TRY(cudaPointerGetAttributes(&at, frame), "ep_kv_ingest_frame_async pointer attributes");
    const bool on_device = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
    // host frames: the header is readable without a sync, so the check stays immediate
    const uint64_t row = 16ull * uint64_t(pool->n_kv_heads) * uint64_t(pool->d_head);
    if (!on_device || frame_bytes < 24 || row == 0 || (frame_bytes - 24) % row != 0 ||
        (frame_bytes - 24) / row == 0 || (frame_bytes - 24) / row > 0xFFFFFFFFull ||
        (uint64_t(frame_bytes - 24) / 16) / 2 > 0x7FFFFFFFull)
        return ep_kv_ingest_frame(h, pool, frame, frame_bytes, page_table, n_pages, nullptr, stream);
    // device frame whose length fits the pool's head shape: launch at once,
    // the kernels check the header against the shape derived here
    if (!h->ingest_status) {
        EP_CUDA_TRY(cudaHostAlloc(reinterpret_cast<void**>(&h->ingest_status), 64, cudaHostAllocDefault),
                    "ep_kv_ingest_frame_async status");
        std::memset(h->ingest_status, 0, 64);
        EP_CUDA_TRY(h->scratch_status.reserve(64), "ep_kv_ingest_frame_async status");
        h->ingest_status_dev = static_cast<int32_t*>(h->scratch_status.ptr);
        EP_CUDA_TRY(cudaMemsetAsync(h->ingest_status_dev, 0, 64, s), "ep_kv_ingest_frame_async status");
    }
    const uint32_t seq = uint32_t((frame_bytes - 24) / row);
    ep::HdrCheck chk{static_cast<const uint8_t*>(frame), uint64_t(frame_bytes), seq, uint32_t(n_pages > 0 ? n_pages : 0),
                     uint32_t(pool->page_tokens), uint16_t(pool->n_kv_heads), uint16_t(pool->d_head),
                     h->ingest_status_dev};
    const uint8_t* src = static_cast<const uint8_t*>(frame) + 24;
    bool staged = false;
    if (reinterpret_cast<uintptr_t>(src) & 7) {
        if (int rc = stage_payload(h, src, frame_bytes - 24, s, &src)) return rc;
        staged = true;
    }
    return launch_ingest(h, pool, seq, uint32_t(pool->n_kv_heads), uint32_t(pool->d_head), src, staged, page_table,
                         chk, s);
}

extern "C" int ep_kv_ingest_poll(ep_handle h, ep_stream stream, ep_kv_frame_info* info) {
    if (!h) return fail(EP_EINVAL, "ep_kv_ingest_poll: null handle");
    if (!h->ingest_status) return EP_OK;  // no deferred ingest issued yet
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_kv_ingest_poll");
    EP_CUDA_TRY(cudaMemcpyAsync(h->ingest_status, h->ingest_status_dev, 8 * sizeof(int32_t), cudaMemcpyDeviceToHost, s),
                "ep_kv_ingest_poll");
    EP_CUDA_TRY(cudaStreamSynchronize(s), "ep_kv_ingest_poll");
    const int32_t* st = h->ingest_status;
    const int kind = st[0];
    if (!kind) return EP_OK;
    ep_kv_frame_info f{};
    f.session_id = uint32_t(st[1]);
    f.seq_len = uint32_t(st[2]);
    f.layer = uint16_t(st[3]);
    f.n_heads = uint16_t(st[4]);
    f.d_head = uint16_t(st[5]);
    f.wire_error = kind <= 6 ? kind : 0;
    if (info) *info = f;
    EP_CUDA_TRY(cudaMemsetAsync(h->ingest_status_dev, 0, 64, s), "ep_kv_ingest_poll");
    if (kind <= 6)
        return fail(EP_EWIRE, std::string("wire: ") + ep::kWireKind[kind] + ": deferred kv frame check failed");
    return fail(EP_EINVAL, kind == 7   ? "ep_kv_ingest_frame_async: kv frame head shape (" + std::to_string(f.n_heads) +
                                             " x " + std::to_string(f.d_head) + ") does not match the pool"
                           : kind == 8 ? std::string("ep_kv_ingest_frame_async: kv frame with empty sequence")
                                       : "ep_kv_ingest_frame_async: " + std::to_string(f.seq_len) +
                                             " tokens need more pages than given");
}
