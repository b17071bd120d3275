// kern_decode.cu — K1 spliced flash-decode and K2 split merge (sm_100a).
//
// Replaces, for a whole batch at once, the per-head loop of transformer_layer's
// attention block (/root/reference/proj/core/src/model.cpp:161-182): one
// partial_attention per visible segment (attention.cpp:80-114) recombined by
// fuse_partials/merge_partials (attention.cpp:116-156). Here the segments of a
// request are walked page by page straight out of the paged pool, with one
// online-softmax state per (request, kv-head) — the same log-sum-exp algebra —
// so no spliced copy of the cache is ever materialised.
//
// CTA anatomy (persistent, one CTA per SM, work = contiguous page ranges from
// plan.cpp so every SM streams the same number of bytes):
//   * warp NCW, one elected lane: producer. Streams each 64-token block of K
//     and V for the CTA's kv-head into an S-stage shared-memory ring with 1-D
//     bulk-async copies (TMA, SASS UBLKCP), completion on `full` mbarriers.
//   * warps 0..NCW-1: consumers. Each warp owns KPW keys of every block; each
//     half-warp owns J = 16/R keys; lane l16 of a half owns E = D/16 contiguous
//     elements of d. Per block: QK^T as packed-fp32 FFMA2 partial dots, a
//     16-lane butterfly reduce-scatter (every lane ends with exactly one
//     (row, key) score), warp-shuffle row max, exp2 online softmax, PV with
//     FFMA2. The R = group * n_q query rows of one kv-head share every K/V
//     element loaded (GQA reuse).
//   * end of a work item: halves, then warps combine in shared memory by
//     LSE; the result goes straight to the output when the item covers the
//     whole (request, kv-head), else to an fp32 partial slot for K2.
#include <cmath>
#include <cstdint>

#include "ep_common.cuh"
#include "ep_internal.h"

namespace ep {
namespace {

template <typename KV, int D, int R, int S>
struct DecodeCfg {
    static constexpr int BT = 64;          // tokens per pipeline block
    static constexpr int E = D / 16;       // d-elements per lane
    static constexpr int J = 16 / R;       // keys per half-warp per block
    static constexpr int KPW = 2 * J;      // keys per warp per block
    static constexpr int NCW = BT / KPW;   // consumer warps
    static constexpr int THREADS = (NCW + 1) * 32;
    static constexpr int ROW_BYTES = D * int(sizeof(KV));
    static constexpr int BLK_BYTES = BT * ROW_BYTES;
    static constexpr int PW_FLOATS = 2 * J * R + R;  // per-warp p and corr slots
    static constexpr int OFF_V = S * BLK_BYTES;
    static constexpr int OFF_BAR = 2 * S * BLK_BYTES;
    static constexpr int OFF_P = OFF_BAR + 2 * S * 8;
    static constexpr int OFF_CO = OFF_P + NCW * PW_FLOATS * 4;
    static constexpr int OFF_CM = OFF_CO + NCW * R * D * 4;
    static constexpr int OFF_CL = OFF_CM + NCW * R * 4;
    static constexpr int SMEM = OFF_CL + NCW * R * 4;
    static_assert(R * J == 16, "one score per lane after the reduce-scatter");
    static_assert(E % 4 == 0, "vector width");
};

// Loads the E elements lane l16 owns of one K/V row as E/2 float2 pairs.
template <typename KV, int E>
struct RowLoader;

template <int E>
struct RowLoader<__nv_bfloat16, E> {
    static_assert(E % 4 == 0, "bf16 rows are read 8 or 16 bytes at a time");
    // E/2 packed bf16 pairs, loaded as 8- or 16-byte vectors.
    __device__ __forceinline__ static void load(const uint8_t* row, int l16, uint32_t (&raw)[E / 2]) {
        if constexpr (E % 8 == 0) {
            const uint4* p = reinterpret_cast<const uint4*>(row) + l16 * (E / 8);
#pragma unroll
            for (int i = 0; i < E / 8; ++i) {
                const uint4 w = p[i];
                raw[4 * i] = w.x;
                raw[4 * i + 1] = w.y;
                raw[4 * i + 2] = w.z;
                raw[4 * i + 3] = w.w;
            }
        } else {
            const uint2* p = reinterpret_cast<const uint2*>(row) + l16 * (E / 4);
#pragma unroll
            for (int i = 0; i < E / 4; ++i) {
                const uint2 w = p[i];
                raw[2 * i] = w.x;
                raw[2 * i + 1] = w.y;
            }
        }
    }
    __device__ __forceinline__ static float2 pair(const uint32_t (&raw)[E / 2], int i) {
        return bf16x2_to_float2(raw[i]);
    }
    using Raw = uint32_t[E / 2];
};

template <int E>
struct RowLoader<float, E> {
    static_assert(E % 4 == 0, "fp32 rows are read 16 bytes at a time");
    __device__ __forceinline__ static void load(const uint8_t* row, int l16, float4 (&raw)[E / 4]) {
        const float4* p = reinterpret_cast<const float4*>(row) + l16 * (E / 4);
#pragma unroll
        for (int i = 0; i < E / 4; ++i) raw[i] = p[i];
    }
    __device__ __forceinline__ static float2 pair(const float4 (&raw)[E / 4], int i) {
        const float4 w = raw[i / 2];
        return (i % 2 == 0) ? make_float2(w.x, w.y) : make_float2(w.z, w.w);
    }
    using Raw = float4[E / 4];
};

template <typename T>
__device__ __forceinline__ float load_q(const void* q, size_t idx) {
    return to_f32<T>(static_cast<const T*>(q)[idx]);
}

template <typename KV, int D, int R, int S>
__global__ void __launch_bounds__(DecodeCfg<KV, D, R, S>::THREADS, 1)
    spliced_decode_kernel(const DecodeArgs a) {
    using C = DecodeCfg<KV, D, R, S>;
    constexpr int BT = C::BT, E = C::E, J = C::J, KPW = C::KPW, NCW = C::NCW;
    using L = RowLoader<KV, E>;

    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* sK = smem;
    uint8_t* sV = smem + C::OFF_V;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* empty = full + S;
    float* s_pw = reinterpret_cast<float*>(smem + C::OFF_P);
    float* c_o = reinterpret_cast<float*>(smem + C::OFF_CO);
    float* c_m = reinterpret_cast<float*>(smem + C::OFF_CM);
    float* c_l = reinterpret_cast<float*>(smem + C::OFF_CL);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it0 = a.cta_item_ptr[blockIdx.x], it1 = a.cta_item_ptr[blockIdx.x + 1];
    const int P = a.page_tokens, Hkv = a.n_kv_heads;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NCW) {
        // ============================ producer ============================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int it = it0; it < it1; ++it) {
                const WorkItem w = a.items[it];
                const PageDesc* pd = a.pdesc + a.req_page_off[w.b];
                for (int lp = w.lp0; lp < w.lp1; ++lp) {
                    const PageDesc d = pd[lp];
                    const size_t tile = (size_t(d.page) * Hkv + w.g) * size_t(P);
                    for (int t0 = 0; t0 < d.n_tok; t0 += BT) {
                        const int nv = min(BT, d.n_tok - t0);
                        const uint32_t bytes = uint32_t(nv) * C::ROW_BYTES;
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx(&full[stage], 2 * bytes);
                        const size_t off = (tile + t0) * C::ROW_BYTES;
                        bulk_g2s(sK + stage * C::BLK_BYTES,
                                 static_cast<const uint8_t*>(a.k_pages) + off, bytes, &full[stage]);
                        bulk_g2s(sV + stage * C::BLK_BYTES,
                                 static_cast<const uint8_t*>(a.v_pages) + off, bytes, &full[stage]);
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
        return;
    }

    // ============================== consumers ==============================
    const int hh = lane >> 4, l16 = lane & 15;
    const int my_r = l16 / J, my_j = l16 % J;  // (row, key) slot after reduce-scatter
    const int G = a.n_q_heads / Hkv;
    float* pw = s_pw + warp * C::PW_FLOATS;  // [2][J][R] p, then [R] corr
    int stage = 0;
    uint32_t phase = 0;

    for (int it = it0; it < it1; ++it) {
        const WorkItem w = a.items[it];
        const PageDesc* pd = a.pdesc + a.req_page_off[w.b];
        const int64_t q0 = a.q_pos[w.b];

        // q rows of this kv-head, pre-scaled by log2(e)/sqrt(d): row r is
        // (query row r / G, head g*G + r % G).
        float2 q2[R][E / 2];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int qi = r / G, h = w.g * G + r % G;
            const size_t base = ((size_t(w.b) * a.n_q + qi) * a.n_q_heads + h) * D + l16 * E;
#pragma unroll
            for (int e = 0; e < E / 2; ++e) {
                float x0, x1;
                if (a.q_dtype == EP_BF16) {
                    x0 = load_q<__nv_bfloat16>(a.q, base + 2 * e);
                    x1 = load_q<__nv_bfloat16>(a.q, base + 2 * e + 1);
                } else {
                    x0 = load_q<float>(a.q, base + 2 * e);
                    x1 = load_q<float>(a.q, base + 2 * e + 1);
                }
                q2[r][e] = make_float2(x0 * a.q_scale, x1 * a.q_scale);
            }
        }
        const int64_t my_qpos = q0 + my_r / G;

        float m_run = -INFINITY, l_run = 0.f;
        float2 o2[R][E / 2];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < E / 2; ++e) o2[r][e] = make_float2(0.f, 0.f);

        for (int lp = w.lp0; lp < w.lp1; ++lp) {
            const PageDesc d = pd[lp];
            for (int t0 = 0; t0 < d.n_tok; t0 += BT) {
                const int nv = min(BT, d.n_tok - t0);
                const int64_t blk_pos = d.pos + t0;
                const bool fast = (nv == BT) && (blk_pos + BT - 1 <= q0);
                mbar_wait(&full[stage], phase);
                const uint8_t* kb = sK + stage * C::BLK_BYTES;
                const uint8_t* vb = sV + stage * C::BLK_BYTES;
                const int key0 = warp * KPW + hh * J;

                // ---- S = Q K^T (partial dots over this lane's E elements) ----
                float sc[16];
                {
                    typename L::Raw kr[J];
#pragma unroll
                    for (int j = 0; j < J; ++j) L::load(kb + (key0 + j) * C::ROW_BYTES, l16, kr[j]);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
#pragma unroll
                        for (int j = 0; j < J; ++j) {
                            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                            for (int e = 0; e < E / 2; ++e) acc = ffma2(q2[r][e], L::pair(kr[j], e), acc);
                            sc[r * J + j] = acc.x + acc.y;
                        }
                    }
                }
                // ---- 16-lane butterfly reduce-scatter: lane l16 keeps sc index l16 ----
#pragma unroll
                for (int step = 0; step < 4; ++step) {
                    const int half = 8 >> step;  // 8,4,2,1 values exchanged
                    const bool upper = (l16 & half) != 0;
#pragma unroll
                    for (int i = 0; i < half; ++i) {
                        const float send = upper ? sc[i] : sc[i + half];
                        const float keep = upper ? sc[i + half] : sc[i];
                        sc[i] = keep + __shfl_xor_sync(0xffffffffu, send, half);
                    }
                }
                float s = sc[0];
                if (!fast) {
                    const int kk = key0 + my_j;
                    const bool ok = kk < nv && blk_pos + kk <= my_qpos;
                    s = ok ? s : -INFINITY;
                }
                // ---- online softmax (rows are lane groups: j bits and the half bit) ----
                float bm = s;
#pragma unroll
                for (int msk = 1; msk < J; msk <<= 1) bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, msk));
                bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, 16));
                const float m_new = fmaxf(m_run, bm);
                const float m_use = m_new == -INFINITY ? 0.f : m_new;
                const float p = fast_exp2(s - m_use);
                const float corr = fast_exp2(m_run - m_use);
                m_run = m_new;
                l_run = l_run * corr + p;
                pw[(hh * J + my_j) * R + my_r] = p;
                if (lane < 16 && my_j == 0) pw[2 * J * R + my_r] = corr;
                __syncwarp();

                // ---- rescale and O += P V ----
                float cr[R];
#pragma unroll
                for (int r = 0; r < R; ++r) cr[r] = pw[2 * J * R + r];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float2 c2 = make_float2(cr[r], cr[r]);
#pragma unroll
                    for (int e = 0; e < E / 2; ++e) o2[r][e] = fmul2(o2[r][e], c2);
                }
                {
                    typename L::Raw vr[J];
#pragma unroll
                    for (int j = 0; j < J; ++j) L::load(vb + (key0 + j) * C::ROW_BYTES, l16, vr[j]);
#pragma unroll
                    for (int j = 0; j < J; ++j) {
                        if (!fast && key0 + j >= nv) continue;  // stale smem beyond the page tail
                        float pj[R];
#pragma unroll
                        for (int r = 0; r < R; ++r) pj[r] = pw[(hh * J + j) * R + r];
#pragma unroll
                        for (int r = 0; r < R; ++r) {
                            const float2 p2 = make_float2(pj[r], pj[r]);
#pragma unroll
                            for (int e = 0; e < E / 2; ++e) o2[r][e] = ffma2(p2, L::pair(vr[j], e), o2[r][e]);
                        }
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);
                if (++stage == S) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }

        // ---- combine the two halves, then the NCW warps, by LSE ----
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < E / 2; ++e) {
                o2[r][e].x += __shfl_xor_sync(0xffffffffu, o2[r][e].x, 16);
                o2[r][e].y += __shfl_xor_sync(0xffffffffu, o2[r][e].y, 16);
            }
        float l_row = l_run;
#pragma unroll
        for (int msk = 1; msk < J; msk <<= 1) l_row += __shfl_xor_sync(0xffffffffu, l_row, msk);
        l_row += __shfl_xor_sync(0xffffffffu, l_row, 16);
        if (lane < 16) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < E / 2; ++e) {
                    float* dst = c_o + (warp * R + r) * D + l16 * E + 2 * e;
                    dst[0] = o2[r][e].x;
                    dst[1] = o2[r][e].y;
                }
            if (my_j == 0) {
                c_m[warp * R + my_r] = m_run;
                c_l[warp * R + my_r] = l_row;
            }
        }
        named_bar_sync(1, NCW * 32);

        const int unit = w.b * Hkv + w.g;
        const bool direct = (a.unit_item_ptr[unit + 1] - a.unit_item_ptr[unit]) == 1;
        for (int idx = threadIdx.x; idx < R * D; idx += NCW * 32) {
            const int r = idx / D, c = idx % D;
            float M = -INFINITY;
#pragma unroll
            for (int ww = 0; ww < NCW; ++ww) M = fmaxf(M, c_m[ww * R + r]);
            float Lsum = 0.f, acc = 0.f;
            if (M != -INFINITY) {
#pragma unroll
                for (int ww = 0; ww < NCW; ++ww) {
                    const float wt = fast_exp2(c_m[ww * R + r] - M);
                    Lsum += wt * c_l[ww * R + r];
                    acc += wt * c_o[(ww * R + r) * D + c];
                }
            }
            const bool empty_row = !(Lsum > 0.f);
            const float val = empty_row ? 0.f : acc / Lsum;
            const float lse2 = empty_row ? -INFINITY : M + fast_log2(Lsum);
            if (direct) {
                const int qi = r / G, h = w.g * G + r % G;
                const size_t orow = (size_t(w.b) * a.n_q + qi) * a.n_q_heads + h;
                if (a.o_dtype == EP_BF16)
                    static_cast<__nv_bfloat16*>(a.o)[orow * D + c] = __float2bfloat16_rn(val);
                else
                    static_cast<float*>(a.o)[orow * D + c] = val;
                if (c == 0 && a.lse) a.lse[orow] = lse2 * kLn2;
            } else {
                a.o_part[(size_t(it) * R + r) * D + c] = val;
                if (c == 0) a.lse_part[size_t(it) * R + r] = lse2;
            }
        }
        named_bar_sync(1, NCW * 32);
    }
}

// K2 for split (request, kv-head) units: LSE-merge the unit's partials in
// page (= segment) order, attention.cpp:116-145 in fp32/log2. Units with one
// item were written directly by K1; units with none are identity rows.
template <int D, int R>
__global__ void __launch_bounds__(128) split_merge_kernel(const DecodeArgs a) {
    const int unit = blockIdx.x;
    const int i0 = a.unit_item_ptr[unit], i1 = a.unit_item_ptr[unit + 1];
    if (i1 - i0 == 1) return;
    const int Hkv = a.n_kv_heads, G = a.n_q_heads / Hkv;
    const int b = unit / Hkv, g = unit % Hkv;
    for (int idx = threadIdx.x; idx < R * D; idx += blockDim.x) {
        const int r = idx / D, c = idx % D;
        float M = -INFINITY;
        for (int i = i0; i < i1; ++i) M = fmaxf(M, a.lse_part[size_t(i) * R + r]);
        float Lsum = 0.f, acc = 0.f;
        if (M != -INFINITY) {
            for (int i = i0; i < i1; ++i) {
                const float wt = exp2f(a.lse_part[size_t(i) * R + r] - M);
                if (wt == 0.f) continue;
                Lsum += wt;
                acc += wt * a.o_part[(size_t(i) * R + r) * D + c];
            }
        }
        const bool empty_row = !(Lsum > 0.f);
        const float val = empty_row ? 0.f : acc / Lsum;
        const int qi = r / G, h = g * G + r % G;
        const size_t orow = (size_t(b) * a.n_q + qi) * a.n_q_heads + h;
        if (a.o_dtype == EP_BF16)
            static_cast<__nv_bfloat16*>(a.o)[orow * D + c] = __float2bfloat16_rn(val);
        else
            static_cast<float*>(a.o)[orow * D + c] = val;
        if (c == 0 && a.lse) a.lse[orow] = empty_row ? -INFINITY : (M + log2f(Lsum)) * kLn2;
    }
}

// Pipeline depth: ~128 KB of K+V blocks in flight per SM (4 stages of a
// 64-token bf16 d=128 block; 2 for fp32 d=128 whose blocks are twice as big).
template <typename KV, int D>
constexpr int stages_for() {
    return (2 * 64 * D * int(sizeof(KV))) >= 65536 ? 2 : 4;
}

template <typename KV, int D, int R>
cudaError_t launch_decode_t(int n_ctas, const DecodeArgs& a, cudaStream_t s) {
    constexpr int S = stages_for<KV, D>();
    using C = DecodeCfg<KV, D, R, S>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    auto kern = spliced_decode_kernel<KV, D, R, S>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e =
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (n_ctas > 0) kern<<<n_ctas, C::THREADS, C::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <typename KV, int D>
cudaError_t dispatch_rows(int rows, int n_ctas, const DecodeArgs& a, cudaStream_t s) {
    switch (rows) {
    case 1: return launch_decode_t<KV, D, 1>(n_ctas, a, s);
    case 2: return launch_decode_t<KV, D, 2>(n_ctas, a, s);
    case 4: return launch_decode_t<KV, D, 4>(n_ctas, a, s);
    case 8: return launch_decode_t<KV, D, 8>(n_ctas, a, s);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

bool decode_supported(int kv_dtype, int d_head, int rows) {
    return (kv_dtype == EP_F32 || kv_dtype == EP_BF16) && (d_head == 64 || d_head == 128) &&
           (rows == 1 || rows == 2 || rows == 4 || rows == 8);
}

int decode_ctas_per_sm(int, int, int) { return 1; }

cudaError_t launch_spliced_decode(int kv_dtype, int d_head, int rows, int n_ctas,
                                  const DecodeArgs& a, cudaStream_t s) {
    if (kv_dtype == EP_BF16) {
        return d_head == 128 ? dispatch_rows<__nv_bfloat16, 128>(rows, n_ctas, a, s)
                             : dispatch_rows<__nv_bfloat16, 64>(rows, n_ctas, a, s);
    }
    return d_head == 128 ? dispatch_rows<float, 128>(rows, n_ctas, a, s)
                         : dispatch_rows<float, 64>(rows, n_ctas, a, s);
}

cudaError_t launch_split_merge(int d_head, int rows, const DecodeArgs& a, cudaStream_t s) {
    const int units = a.batch * a.n_kv_heads;
    if (units == 0) return cudaSuccess;
#define EP_MERGE_CASE(DD, RR) \
    if (d_head == DD && rows == RR) { split_merge_kernel<DD, RR><<<units, 128, 0, s>>>(a); return cudaGetLastError(); }
    EP_MERGE_CASE(64, 1) EP_MERGE_CASE(64, 2) EP_MERGE_CASE(64, 4) EP_MERGE_CASE(64, 8)
    EP_MERGE_CASE(128, 1) EP_MERGE_CASE(128, 2) EP_MERGE_CASE(128, 4) EP_MERGE_CASE(128, 8)
#undef EP_MERGE_CASE
    return cudaErrorInvalidValue;
}

}  // namespace ep
