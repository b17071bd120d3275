// kern_decode.cu — K1 spliced flash-decode with the K2 split merge fused in (sm_100a).
//
// Replaces, for a whole batch at once, the per-head loop of transformer_layer's
// attention block (/root/reference/proj/core/src/model.cpp:161-182): one
// partial_attention per visible segment (attention.cpp:80-114) recombined by
// fuse_partials/merge_partials (attention.cpp:116-156). Here the segments of a
// request are walked page by page straight out of the paged pool, with one
// online-softmax state per (request, kv-head) — the same log-sum-exp algebra —
// so no spliced copy of the cache is ever materialised.
//
// CTA anatomy (persistent, one CTA per SM; work = contiguous page ranges from
// capi.cpp's planner, so every SM streams the same number of bytes):
//   * warp NCW, one lane: producer. Streams each 64-token block of K and V of
//     the CTA's kv-head into an S-stage shared-memory ring with 1-D bulk-async
//     copies (TMA, SASS UBLKCP) completing on `full` mbarriers, and writes a
//     16-byte stage header {position, valid rows}. A block shorter than 64
//     rows (segment tail) gets its V tail filled from a zero page by one more
//     bulk copy, so the consumers' PV loop is branch-free.
//   * warps 0..NCW-1: consumers. Warp w owns keys [w*2J, w*2J+2J) of every
//     block; each half-warp J keys; lane l16 of a half owns E = D/16 contiguous
//     elements of d. Per block: QK^T as packed-fp32 FFMA2 partial dots (K
//     bf16 pairs unpacked with one shift/and each), a 16-lane butterfly
//     reduce-scatter (each lane ends with one (row, key) score), warp-shuffle
//     row max, exp2 online softmax, rescale + PV with FMUL2/FFMA2. The
//     R = group * n_q rows of one kv-head share every K/V element (GQA reuse).
//   * end of a work item: the consumer warps hand their (m, l, o) states to
//     the epilogue warp through shared memory (an mbarrier pair) and go on
//     with the next item at once, so the ring never stalls on an item end.
//     The epilogue warp combines the states by LSE; an item that covers its
//     whole (request, kv-head) writes the output directly; otherwise it
//     writes an fp32 partial, and the LAST CTA to finish a unit (per-unit
//     arrival counter) merges the unit's partials in page = segment order
//     (attention.cpp:116-145) — no second launch.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ep_common.cuh"
#include "ep_internal.h"
#include "merge.cuh"

namespace ep {
namespace {

constexpr int kLog2(int x) { return x <= 1 ? 0 : 1 + kLog2(x / 2); }

template <typename KV, int D, int R, int J, int S>
struct DecodeCfg {
    static constexpr int BT = 64;          // tokens per pipeline block
    static constexpr int E = D / 16;       // d-elements per lane
    static constexpr int KPW = 2 * J;      // keys per warp per block
    static constexpr int NCW = BT / KPW;   // consumer warps
    static constexpr int THREADS = (NCW + 2) * 32;  // + producer warp + epilogue warp
    static constexpr int NV = R * J;       // partial scores per half-warp
    static constexpr int LOGN = kLog2(NV);
    static constexpr int DUP = 4 - LOGN;   // low lane bits holding duplicate slots
    static constexpr int ROW_BYTES = D * int(sizeof(KV));
    static constexpr int BLK_BYTES = BT * ROW_BYTES;
    static constexpr int PW_FLOATS = 2 * J * R + R;  // per-warp p and corr slots
    static constexpr int OFF_V = S * BLK_BYTES;
    static constexpr int OFF_BAR = 2 * S * BLK_BYTES;
    static constexpr int OFF_HDR = OFF_BAR + 2 * S * 8;
    static constexpr int OFF_P = OFF_HDR + S * 16;
    static constexpr int OFF_CO = OFF_P + NCW * PW_FLOATS * 4;
    static constexpr int OFF_CM = OFF_CO + NCW * R * D * 4;
    static constexpr int OFF_CL = OFF_CM + NCW * R * 4;
    static constexpr int OFF_FLAG = OFF_CL + NCW * R * 4;
    static constexpr int Q_BYTES = R * D * 4;               // one item's q rows (fp32 worst case)
    static constexpr int OFF_Q = (OFF_FLAG + 16 + 127) / 128 * 128;  // [2] q slots (bulk-prefetched)
    static constexpr int OFF_QBAR = OFF_Q + 2 * Q_BYTES;      // q_full[2], q_empty[2], ep_full, ep_empty
    static constexpr int SMEM = OFF_QBAR + 6 * 8;
    static_assert((1 << LOGN) == NV && NV <= 16, "R*J must be a power of two <= 16");
    static_assert(E % 4 == 0, "vector width");
    static_assert(NCW * 32 <= 1024 - 32, "block size");
};

struct StageHdr {
    int64_t pos;  // absolute position of row 0
    int32_t nv;   // valid rows
    int32_t pad;
};

// Loads the E elements lane l16 owns of one K/V row; pair(i) is elements 2i, 2i+1.
template <typename KV, int E>
struct RowLoader;

template <int E>
struct RowLoader<__nv_bfloat16, E> {
    using Raw = uint32_t[E / 2];
    __device__ __forceinline__ static void load(const uint8_t* row, int l16, Raw& raw) {
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
    __device__ __forceinline__ static float2 pair(const Raw& raw, int i) {
        return bf16x2_to_float2(raw[i]);
    }
};

template <int E>
struct RowLoader<float, E> {
    using Raw = float4[E / 4];
    __device__ __forceinline__ static void load(const uint8_t* row, int l16, Raw& raw) {
        const float4* p = reinterpret_cast<const float4*>(row) + l16 * (E / 4);
#pragma unroll
        for (int i = 0; i < E / 4; ++i) raw[i] = p[i];
    }
    __device__ __forceinline__ static float2 pair(const Raw& raw, int i) {
        const float4 w = raw[i / 2];
        return (i % 2 == 0) ? make_float2(w.x, w.y) : make_float2(w.z, w.w);
    }
};

__device__ __forceinline__ float load_q(const void* q, int dtype, size_t idx) {
    return dtype == EP_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(q)[idx])
                            : static_cast<const float*>(q)[idx];
}

__device__ __forceinline__ void store_o(void* o, int dtype, size_t idx, float v) {
    if (dtype == EP_BF16)
        static_cast<__nv_bfloat16*>(o)[idx] = __float2bfloat16_rn(v);
    else
        static_cast<float*>(o)[idx] = v;
}

__device__ __forceinline__ int item_at(const DecodeArgs& a, int j) {
    return a.cta_item_idx ? a.cta_item_idx[j] : j;
}

// End of work item `it`: combines the NCW consumer warps' (m, l, o) states in
// c_m / c_l / c_o by LSE (row r: weights 2^(m_w - M)); an item covering its
// whole (request, kv-head) stores the output, otherwise an fp32 partial, and
// the last CTA to finish an item of the unit (arrival counter) merges the
// unit's partials in page = segment order (attention.cpp:116-145). Run by a
// group of n_grp warps (gw = this warp's index in it): the epilogue warp
// (kOneWarp) or the consumer warps. ep_empty (may be null) is arrived at once
// the states are read.
template <int D, int R, int NCW, bool kOneWarp>
__device__ __forceinline__ void item_end(const DecodeArgs& a, int it, int gw, int n_grp, const float* c_o,
                                         const float* c_m, const float* c_l, int* s_flag, uint64_t* ep_empty) {
    constexpr int EL = D / 32;  // columns per lane
    const int lane = threadIdx.x & 31;
    const int Hkv = a.n_kv_heads, G = a.n_q_heads / Hkv;
    const WorkItem w = a.items[it];
    const int unit = w.b * Hkv + w.g;
    EP_DCHECK(it >= 0 && it < a.n_items && unit >= 0 && unit < a.batch * Hkv);
    const int u0 = a.unit_item_ptr[unit], n_items = a.unit_item_ptr[unit + 1] - u0;
    EP_DCHECK(n_items >= 1 && u0 + n_items <= a.n_items && it >= u0 && it < u0 + n_items);
    const bool direct = n_items == 1;
#pragma unroll 1
    for (int r = gw; r < R; r += n_grp) {
        float M = -INFINITY;
#pragma unroll
        for (int ww = 0; ww < NCW; ++ww) M = fmaxf(M, c_m[ww * R + r]);
        float acc[EL];
#pragma unroll
        for (int e = 0; e < EL; ++e) acc[e] = 0.f;
        float Lsum = 0.f;
        if (M != -INFINITY) {
#pragma unroll
            for (int ww = 0; ww < NCW; ++ww) {
                const float wt = fast_exp2(c_m[ww * R + r] - M);
                Lsum += wt * c_l[ww * R + r];
                const float* src = c_o + (ww * R + r) * D + lane * EL;
                if constexpr (EL == 4) {
                    const float4 v = *reinterpret_cast<const float4*>(src);
                    acc[0] += wt * v.x; acc[1] += wt * v.y; acc[2] += wt * v.z; acc[3] += wt * v.w;
                } else {
                    const float2 v = *reinterpret_cast<const float2*>(src);
                    acc[0] += wt * v.x; acc[1] += wt * v.y;
                }
            }
        }
        const bool empty_row = !(Lsum > 0.f);
        const float inv = empty_row ? 0.f : 1.f / Lsum;
        const float lse2 = empty_row ? -INFINITY : M + fast_log2(Lsum);
        if (direct) {
            if (r < w.pad) {
                const int qi = r / G, h = w.g * G + r % G;
                const size_t orow = (q_row_base(a, w.b) + qi) * a.n_q_heads + h;
                EP_DCHECK(int64_t(orow) < a.n_q_rows * a.n_q_heads);
                if (a.peer.world) {  // fused split-KV: the row goes to every rank
                    float v[EL];
#pragma unroll
                    for (int e = 0; e < EL; ++e) v[e] = acc[e] * inv;
                    peer_push_row<D>(a, unit, orow, v, lse2);
                } else {
#pragma unroll
                    for (int e = 0; e < EL; ++e) store_o(a.o, a.o_dtype, orow * D + lane * EL + e, acc[e] * inv);
                    if (lane == 0 && a.lse) a.lse[orow] = lse2 * kLn2;
                }
            }
        } else {
            float* dst = a.o_part + (size_t(it) * R + r) * D + lane * EL;
            if constexpr (EL == 4)
                *reinterpret_cast<float4*>(dst) = make_float4(acc[0] * inv, acc[1] * inv, acc[2] * inv, acc[3] * inv);
            else
                *reinterpret_cast<float2*>(dst) = make_float2(acc[0] * inv, acc[1] * inv);
            if (lane == 0) a.lse_part[size_t(it) * R + r] = lse2;
        }
    }
    if (kOneWarp) {
        __syncwarp();
        if (lane == 0 && ep_empty) mbar_arrive(ep_empty);  // the consumers may overwrite c_o
    }
    if (direct) return;
    // Fused K2: the last CTA to finish one of this unit's items merges them
    // all, in page (= segment) order (attention.cpp:128-144).
    __threadfence();
    int last = 0;
    if (kOneWarp) {
        __syncwarp();
        if (lane == 0) last = atomicAdd(&a.unit_counter[unit], 1) == n_items - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
    } else {
        named_bar_sync(1, n_grp * 32);
        if (gw == 0 && lane == 0) *s_flag = atomicAdd(&a.unit_counter[unit], 1) == n_items - 1;
        named_bar_sync(1, n_grp * 32);
        last = *s_flag;
    }
    if (last) {
        __threadfence();
        merge_unit_rows<D>(a, u0, n_items, R, w.pad, gw, n_grp, [&](int r) {
            const int qi = r / G, h = w.g * G + r % G;
            return (q_row_base(a, w.b) + qi) * a.n_q_heads + h;
        }, unit);
        if (gw == 0 && lane == 0) a.unit_counter[unit] = 0;  // ready for the next launch
    }
}

template <typename KV, int D, int R, int J, int S>
__global__ void __launch_bounds__(DecodeCfg<KV, D, R, J, S>::THREADS, 1)
    spliced_decode_kernel(const DecodeArgs a) {
    using C = DecodeCfg<KV, D, R, J, S>;
    constexpr int BT = C::BT, E = C::E, KPW = C::KPW, NCW = C::NCW, NV = C::NV;
    constexpr int LOGN = C::LOGN, DUP = C::DUP;
    using L = RowLoader<KV, E>;

    extern __shared__ __align__(128) uint8_t smem[];
    // programmatic dependent launch: nothing global is read before the
    // predecessor (e.g. the Q/K/V projection writing q and the new K/V rows,
    // or the previous step) has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");
    uint8_t* sK = smem;
    uint8_t* sV = smem + C::OFF_V;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* empty = full + S;
    StageHdr* hdr = reinterpret_cast<StageHdr*>(smem + C::OFF_HDR);
    float* s_pw = reinterpret_cast<float*>(smem + C::OFF_P);
    float* c_o = reinterpret_cast<float*>(smem + C::OFF_CO);
    float* c_m = reinterpret_cast<float*>(smem + C::OFF_CM);
    float* c_l = reinterpret_cast<float*>(smem + C::OFF_CL);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it0 = a.cta_item_ptr[blockIdx.x], it1 = a.cta_item_ptr[blockIdx.x + 1];
    const int P = a.page_tokens, Hkv = a.n_kv_heads;
    if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // debug: per-CTA start (ns), work
        unsigned long long t, nb = 0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[18 * 1024 + 2 * blockIdx.x] = t;
        for (int it = it0; it < it1; ++it) nb += a.items[it].nblk;
        a.trace[20 * 1024 + 2 * blockIdx.x] = it1 - it0;
        a.trace[20 * 1024 + 2 * blockIdx.x + 1] = nb;
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        a.trace[30 * 1024 + blockIdx.x] = sm;
    }

    uint8_t* sq = smem + C::OFF_Q;
    uint64_t* q_full = reinterpret_cast<uint64_t*>(smem + C::OFF_QBAR);
    uint64_t* q_empty = q_full + 2;
    uint64_t* ep_full = q_full + 4;   // consumer warps -> epilogue warp: c_o / c_m / c_l written
    uint64_t* ep_empty = q_full + 5;  // epilogue warp -> consumers: c_o read
    int* s_flag = reinterpret_cast<int*>(smem + C::OFF_FLAG);
    const int qsz = a.q_dtype == EP_BF16 ? 2 : 4;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], NCW);
        }
        mbar_init(ep_full, NCW);
        mbar_init(ep_empty, 1);
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == NCW) {
        // ============================ producer ============================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint8_t* kp = static_cast<const uint8_t*>(a.k_pages);
            const uint8_t* vp = static_cast<const uint8_t*>(a.v_pages);
            const uint8_t* zp = static_cast<const uint8_t*>(a.zero_rows);
            const int G = a.n_q_heads / Hkv;
            for (int j = it0; j < it1; ++j) {
                const int it = item_at(a, j);
                EP_DCHECK(it >= 0 && it < a.n_items);
                const WorkItem w = a.items[it];
                const PageDesc* pd = a.pdesc + a.req_page_off[w.b];
                EP_DCHECK(w.lp0 < w.lp1 && w.g >= 0 && w.g < Hkv && w.pad >= 1 && w.pad <= R);
                {
                    // the item's R query rows: n_q runs of G consecutive heads
                    const int n = j - it0, slot = n & 1;
                    // (a prefill chunk's last item may hold fewer than n_q query tokens:
                    // w.pad = its valid rows; only those are loaded and stored)
                    const uint32_t run = uint32_t(G) * D * qsz;
                    const int nq = min(a.n_q, (w.pad + G - 1) / G);
                    EP_DCHECK(int64_t(q_row_base(a, w.b)) + nq <= a.n_q_rows);
                    mbar_wait(&q_empty[slot], ((n >> 1) & 1) ^ 1);
                    mbar_arrive_expect_tx(&q_full[slot], run * nq);
                    for (int qi = 0; qi < nq; ++qi)
                        bulk_g2s(sq + slot * C::Q_BYTES + qi * run,
                                 static_cast<const uint8_t*>(a.q) +
                                     ((q_row_base(a, w.b) + qi) * a.n_q_heads + size_t(w.g) * G) * D * qsz,
                                 run, &q_full[slot]);
                }
                for (int lp = w.lp0; lp < w.lp1; ++lp) {
                    const PageDesc d = pd[lp];
                    EP_DCHECK(d.page >= 0 && d.page < a.num_pages && d.n_tok >= 1 && d.n_tok <= P);
                    const size_t tile = (size_t(d.page) * Hkv + w.g) * size_t(P);
                    for (int t0 = 0; t0 < d.n_tok; t0 += BT) {
                        const int nv = min(BT, d.n_tok - t0);
                        const uint32_t bytes = uint32_t(nv) * C::ROW_BYTES;
                        const uint32_t tail = uint32_t(BT - nv) * C::ROW_BYTES;
                        mbar_wait(&empty[stage], phase ^ 1);
                        hdr[stage].pos = d.pos + t0;
                        hdr[stage].nv = nv;
                        mbar_arrive_expect_tx(&full[stage], 2 * bytes + tail);
                        const size_t off = (tile + t0) * C::ROW_BYTES;
                        uint8_t* dk = sK + stage * C::BLK_BYTES;
                        uint8_t* dv = sV + stage * C::BLK_BYTES;
                        bulk_g2s(dk, kp + off, bytes, &full[stage]);
                        bulk_g2s(dv, vp + off, bytes, &full[stage]);
                        if (tail) bulk_g2s(dv + bytes, zp, tail, &full[stage]);
                        if (++stage == S) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
            // every load is issued: the next kernel in the stream may be
            // scheduled (programmatic dependent launch; it still waits for
            // this grid's completion before reading anything it writes)
            asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        }
        return;
    }

    if (warp == NCW + 1) {
        // ============================ epilogue ============================
        // the item ends of every item but the CTA's last (that one the
        // consumer warps do together: nothing is left to stream behind it)
        for (int j = it0; j < it1 - 1; ++j) {
            const int n = j - it0, it = item_at(a, j);
            mbar_wait(ep_full, n & 1);
            item_end<D, R, NCW, true>(a, it, 0, 1, c_o, c_m, c_l, s_flag, ep_empty);
            if (a.trace && lane == 0 && blockIdx.x < 1024 && n < 4) {  // debug: item end done
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                a.trace[22 * 1024 + 8 * blockIdx.x + 2 * n + 1] = t;
            }
        }
        if (a.trace && lane == 0 && blockIdx.x < 1024) {  // debug: epilogue warp end (ns)
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[31 * 1024 + blockIdx.x] = t;
        }
        return;
    }

    // ============================== consumers ==============================
    const int hh = lane >> 4, l16 = lane & 15;
    const int my_idx = l16 >> DUP;           // (row, key) slot after the reduce-scatter
    const int my_r = my_idx / J, my_j = my_idx % J;
    const int G = a.n_q_heads / Hkv;
    float* pw = s_pw + warp * C::PW_FLOATS;  // [2][J][R] p, then [R] corr
    const int key0 = warp * KPW + hh * J;
    int stage = 0;
    uint32_t phase = 0;

    for (int j = it0; j < it1; ++j) {
        const int it = item_at(a, j);
        const WorkItem w = a.items[it];
        const int64_t q0 = a.q_pos[w.b];

        // q rows of this kv-head, pre-scaled by log2(e)/sqrt(d): logical row r
        // is (query row r / G, head g*G + r % G). Physical slot rp holds
        // logical row rp ^ my_r (see the reduce-scatter below).
        // (prefetched by the producer into q slot (j - it0) & 1; row r sits at r * D)
        float2 q2[R][E / 2];
        {
            const int n = j - it0, slot = n & 1;
            mbar_wait(&q_full[slot], (n >> 1) & 1);
            const uint8_t* qs = sq + slot * C::Q_BYTES;
#pragma unroll
            for (int rp = 0; rp < R; ++rp) {
                const int r = rp ^ my_r;
                const size_t base = size_t(r) * D + l16 * E;
                const bool live = r < w.pad;  // rows past a short prefill chunk: zero q
#pragma unroll
                for (int e = 0; e < E / 2; ++e)
                    q2[rp][e] = live ? make_float2(load_q(qs, a.q_dtype, base + 2 * e) * a.q_scale,
                                                   load_q(qs, a.q_dtype, base + 2 * e + 1) * a.q_scale)
                                     : make_float2(0.f, 0.f);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&q_empty[slot]);
        }
        const int64_t my_qpos = q0 + my_r / G;

        float m_run = -INFINITY, l_run = 0.f;
        float2 o2[R][E / 2];
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < E / 2; ++e) o2[r][e] = make_float2(0.f, 0.f);

        for (int blk = 0; blk < w.nblk; ++blk) {
            mbar_wait(&full[stage], phase);
            const StageHdr hd = hdr[stage];
            const bool fast = (hd.nv == BT) && (hd.pos + BT - 1 <= q0);
            const uint8_t* kb = sK + stage * C::BLK_BYTES;
            const uint8_t* vb = sV + stage * C::BLK_BYTES;

            // ---- S = Q K^T: partial dots over this lane's E elements ----
            // Physical score slot p = rp*J + jp holds logical (row, key) index
            // p ^ my_idx: rows via the q2 permutation, keys by loading key
            // jp ^ my_j into kr[jp]. Then at every reduce-scatter step the
            // values a lane keeps are its low half and the ones it sends its
            // high half, for every lane — no per-lane selects.
            float sc[NV];
            {
                typename L::Raw kr[J];
#pragma unroll
                for (int jp = 0; jp < J; ++jp)
                    L::load(kb + (key0 + (jp ^ my_j)) * C::ROW_BYTES, l16, kr[jp]);
#pragma unroll
                for (int rp = 0; rp < R; ++rp)
#pragma unroll
                    for (int jp = 0; jp < J; ++jp) {
                        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                        for (int e = 0; e < E / 2; ++e) acc = ffma2(q2[rp][e], L::pair(kr[jp], e), acc);
                        sc[rp * J + jp] = acc.x + acc.y;
                    }
            }
            // ---- butterfly reduce-scatter over the 16 lanes of a half ----
#pragma unroll
            for (int st = 0; st < LOGN; ++st) {
                const int half = NV >> (st + 1);
                const int mask = 8 >> st;
#pragma unroll
                for (int i = 0; i < half; ++i)
                    sc[i] += __shfl_xor_sync(0xffffffffu, sc[i + half], mask);
            }
            float s = sc[0];
#pragma unroll
            for (int st = LOGN; st < 4; ++st) s += __shfl_xor_sync(0xffffffffu, s, 8 >> st);
            if (!fast) {
                const int kk = key0 + my_j;
                const bool ok = kk < hd.nv && hd.pos + kk <= my_qpos;
                s = ok ? s : -INFINITY;
            }
            // ---- online softmax: a row's slots span the j bits, dup bits and the half ----
            float bm = s;
#pragma unroll
            for (int msk = 1; msk < (J << DUP); msk <<= 1)
                bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, msk));
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

            // ---- rescale, then O += P V (V tails are zero-filled: no branches) ----
            typename L::Raw vr[J];
#pragma unroll
            for (int j = 0; j < J; ++j) L::load(vb + (key0 + j) * C::ROW_BYTES, l16, vr[j]);
            if (!__all_sync(0xffffffffu, corr == 1.f)) {  // some row's max moved
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float cr = pw[2 * J * R + r];
                    const float2 c2 = make_float2(cr, cr);
#pragma unroll
                    for (int e = 0; e < E / 2; ++e) o2[r][e] = fmul2(o2[r][e], c2);
                }
            }
#pragma unroll
            for (int j = 0; j < J; ++j) {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float pj = pw[(hh * J + j) * R + r];
                    const float2 p2 = make_float2(pj, pj);
#pragma unroll
                    for (int e = 0; e < E / 2; ++e) o2[r][e] = ffma2(p2, L::pair(vr[j], e), o2[r][e]);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stage]);
            if (++stage == S) {
                stage = 0;
                phase ^= 1;
            }
        }

        if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024 && j - it0 < 4) {  // debug: item's last block done
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[22 * 1024 + 8 * blockIdx.x + 2 * (j - it0)] = t;
        }
        // ---- combine the two halves, then hand the warp's state to the epilogue warp ----
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int e = 0; e < E / 2; ++e) {
                o2[r][e].x += __shfl_xor_sync(0xffffffffu, o2[r][e].x, 16);
                o2[r][e].y += __shfl_xor_sync(0xffffffffu, o2[r][e].y, 16);
            }
        float l_row = l_run;  // sum over distinct slots of the row (skip duplicate lanes)
#pragma unroll
        for (int msk = 1 << DUP; msk < (J << DUP); msk <<= 1)
            l_row += __shfl_xor_sync(0xffffffffu, l_row, msk);
        l_row += __shfl_xor_sync(0xffffffffu, l_row, 16);
        mbar_wait(ep_empty, ((j - it0) & 1) ^ 1);  // the epilogue warp has read the previous item's states
        const bool last_item = j == it1 - 1;
        if (lane < 16) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int e = 0; e < E / 2; ++e)
                    *reinterpret_cast<float2*>(c_o + (warp * R + r) * D + l16 * E + 2 * e) = o2[r][e];
            if (my_j == 0 && (l16 & ((1 << DUP) - 1)) == 0) {
                c_m[warp * R + my_r] = m_run;
                c_l[warp * R + my_r] = l_row;
            }
        }
        if (last_item) {
            // nothing left to stream: all consumer warps do this item end
            named_bar_sync(1, NCW * 32);
            item_end<D, R, NCW, false>(a, it, warp, NCW, c_o, c_m, c_l, s_flag, nullptr);
            if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024 && j - it0 < 4) {  // debug: item end done
                unsigned long long t;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                a.trace[22 * 1024 + 8 * blockIdx.x + 2 * (j - it0) + 1] = t;
            }
        } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(ep_full);
        }
    }
    if (a.peer.world) {
        // fused split-KV: merge the rank partials of the units this CTA owns
        // (every push of this rank is issued without waiting, so these polls
        // cannot deadlock), then advance their epochs
        peer_merge_owned<D>(a, warp, NCW);
        named_bar_sync(1, NCW * 32);
        if (threadIdx.x == 0)
            for (int u = a.peer.cta_unit_ptr[blockIdx.x]; u < a.peer.cta_unit_ptr[blockIdx.x + 1]; ++u)
                a.peer.epoch[u] += 1u;
    }
    if (a.trace && threadIdx.x == 0 && blockIdx.x < 1024) {  // debug: per-CTA end (ns)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[18 * 1024 + 2 * blockIdx.x + 1] = t;
    }
}

// Units with no pages at all (empty requests) are identity rows: o = 0,
// lse = -inf (attention.cpp:37-43). Launched only when the plan has any.
__global__ void empty_units_kernel(const DecodeArgs a, int D, int R) {
    const int unit = blockIdx.x;
    if (a.unit_item_ptr[unit + 1] != a.unit_item_ptr[unit]) return;
    const int Hkv = a.n_kv_heads, G = a.n_q_heads / Hkv;
    const int b = unit / Hkv, g = unit % Hkv;
    if (!a.q_row0) R = min(R, valid_rows(a, b));  // K1 pads R to a power of two
    for (int idx = threadIdx.x; idx < R * D; idx += blockDim.x) {
        const int r = idx / D, c = idx % D;
        const int qi = r / G, h = g * G + r % G;
        const size_t orow = (q_row_base(a, b) + qi) * a.n_q_heads + h;
        store_o(a.o, a.o_dtype, orow * D + c, 0.f);
        if (c == 0 && a.lse) a.lse[orow] = -INFINITY;
    }
}

// Keys per half-warp. R*J = 16 partial scores per 16 lanes (one per lane
// after the reduce-scatter) with 2R consumer warps: measured on cfg2 (R = 4),
// 8 warps with J = 4 and ~150 registers beat 16 warps with J = 2 squeezed into
// 96 registers (5.71 vs 5.01 TB/s). R = 1 uses J = 8 (4 warps); R = 8 uses
// J = 2 (16 warps).
template <int R>
constexpr int keys_per_half() {
    return R == 1 ? 8 : 16 / R;
}

// Pipeline depth: 128-160 KB of K+V blocks per SM (5 stages of a 64-token
// bf16 d=128 block for up to 4 rows — measured on cfg2: 4 / 5 / 6 stages
// 104.5 / 103.2 / 104.2 us — 4 otherwise; 2 for fp32 d=128 whose blocks are
// twice as big).
template <typename KV, int D, int R>
constexpr int stages_for() {
    return (2 * 64 * D * int(sizeof(KV))) >= 65536 ? 2 : (sizeof(KV) == 2 && D == 128 && R <= 4 ? 5 : 4);
}

template <typename KV, int D, int R, int J = keys_per_half<R>(), int S = stages_for<KV, D, R>()>
cudaError_t launch_decode_t(int n_ctas, const DecodeArgs& a, cudaStream_t s) {
    using C = DecodeCfg<KV, D, R, J, S>;
    static_assert(C::SMEM <= 227 * 1024, "shared memory budget");
    auto kern = spliced_decode_kernel<KV, D, R, J, S>;
    if (cudaError_t e = ensure_smem<spliced_decode_kernel<KV, D, R, J, S>>(C::SMEM)) return e;
    if (n_ctas > 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(n_ctas);
        cfg.blockDim = dim3(C::THREADS);
        cfg.dynamicSmemBytes = C::SMEM;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, a);
    }
    return cudaGetLastError();
}

// rows: the plan's row stride (a power of two; the valid rows of a unit
// are its items' pad, the rest are zero-q rows that are never stored)
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

// ------------------------------------------------------------ generic ----
// Shapes outside K1 / K3 (d_head not 64 / 128, or more than 8 query heads per
// kv head outside K3): one CTA per (request, query token, query head) row,
// its four warps taking the request's pages round-robin with one online
// softmax each (lane = key for q.k, lane = columns for p.v), merged by LSE
// at the end — partial_attention + merge_partials (attention.cpp:80-145)
// with GQA as kv-head indexing. Correct for every shape; not tuned.
constexpr int kGenWarps = 4;
constexpr int kGenPerLane = 8;  // d_head <= 256

template <typename KV>
__device__ __forceinline__ float kvf(const KV* p, size_t i) {
    if constexpr (sizeof(KV) == 2)
        return __bfloat162float(p[i]);
    else
        return p[i];
}

template <typename KV>
__global__ void __launch_bounds__(kGenWarps * 32) generic_decode_kernel(const DecodeArgs a, int D) {
    const int b = blockIdx.x, qi = blockIdx.y, h = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int Hkv = a.n_kv_heads, G = a.n_q_heads / Hkv, g = h / G, P = a.page_tokens;
    extern __shared__ __align__(16) float gsm[];
    float* qs = gsm;            // [D], pre-scaled by log2(e) / sqrt(d)
    float* wo = qs + D;         // [warps][D]
    __shared__ float wm[kGenWarps], wl[kGenWarps];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const size_t row = (q_row_base(a, b) + qi) * a.n_q_heads + h;
    for (int c = tid; c < D; c += blockDim.x)
        qs[c] = (a.q_dtype == EP_BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(a.q)[row * D + c])
                                      : static_cast<const float*>(a.q)[row * D + c]) *
                a.q_scale;
    __syncthreads();
    const int64_t qpos = a.q_pos[b] + qi;
    const int64_t p0 = a.req_page_off[b], np = a.req_page_off[b + 1] - p0;
    const KV* kp = static_cast<const KV*>(a.k_pages);
    const KV* vp = static_cast<const KV*>(a.v_pages);
    float m = -INFINITY, l = 0.f, o[kGenPerLane];
#pragma unroll
    for (int i = 0; i < kGenPerLane; ++i) o[i] = 0.f;
    for (int64_t pi = warp; pi < np; pi += kGenWarps) {
        const PageDesc d = a.pdesc[p0 + pi];
        const int64_t vis = qpos - d.pos + 1;  // visible prefix of the page (attention.cpp:29-33)
        const int nk = vis <= 0 ? 0 : (vis < d.n_tok ? int(vis) : d.n_tok);
        const size_t tile = (size_t(d.page) * Hkv + g) * size_t(P);
        for (int j0 = 0; j0 < nk; j0 += 32) {
            const int j = j0 + lane;
            float sc = -INFINITY;
            if (j < nk) {
                const KV* kr = kp + (tile + j) * D;
                float dot = 0.f;
                for (int c = 0; c < D; ++c) dot = fmaf(qs[c], kvf(kr, c), dot);
                sc = dot;
            }
            float cm = sc;
#pragma unroll
            for (int msk = 16; msk > 0; msk >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, msk));
            const float nm = fmaxf(m, cm);
            const float corr = m == -INFINITY ? 0.f : exp2f(m - nm);
            const float pj_own = j < nk ? exp2f(sc - nm) : 0.f;
            l = l * corr + warp_sum(pj_own);
#pragma unroll
            for (int i = 0; i < kGenPerLane; ++i) o[i] *= corr;
            const int cnt = min(32, nk - j0);
            for (int jj = 0; jj < cnt; ++jj) {
                const float pj = __shfl_sync(0xffffffffu, pj_own, jj);
                const KV* vr = vp + (tile + j0 + jj) * D;
#pragma unroll
                for (int i = 0; i < kGenPerLane; ++i) {
                    const int c = lane + 32 * i;
                    if (c < D) o[i] = fmaf(pj, kvf(vr, c), o[i]);
                }
            }
            m = nm;
        }
    }
    if (lane == 0) {
        wm[warp] = m;
        wl[warp] = l;
    }
#pragma unroll
    for (int i = 0; i < kGenPerLane; ++i) {
        const int c = lane + 32 * i;
        if (c < D) wo[warp * D + c] = o[i];
    }
    __syncthreads();
    float M = -INFINITY;
    for (int w = 0; w < kGenWarps; ++w) M = fmaxf(M, wm[w]);
    float L = 0.f, wt[kGenWarps];
    for (int w = 0; w < kGenWarps; ++w) {
        wt[w] = wm[w] == -INFINITY ? 0.f : exp2f(wm[w] - M);
        L += wt[w] * wl[w];
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;  // no visible key: the identity (o = 0, lse = -inf)
    for (int c = tid; c < D; c += blockDim.x) {
        float acc = 0.f;
        for (int w = 0; w < kGenWarps; ++w) acc += wt[w] * wo[w * D + c];
        store_o(a.o, a.o_dtype, row * D + c, acc * inv);
    }
    if (tid == 0 && a.lse) a.lse[row] = L > 0.f ? (M + log2f(L)) * kLn2 : -INFINITY;
}

}  // namespace

bool decode_supported(int kv_dtype, int d_head, int rows) {
    return (kv_dtype == EP_F32 || kv_dtype == EP_BF16) && (d_head == 64 || d_head == 128) && rows >= 1 &&
           rows <= 8;
}

bool generic_supported(int kv_dtype, int d_head) {
    return (kv_dtype == EP_F32 || kv_dtype == EP_BF16) && d_head >= 1 && d_head <= 32 * kGenPerLane;
}

cudaError_t launch_generic_decode(int kv_dtype, int d_head, int batch, int n_q, const DecodeArgs& a,
                                  cudaStream_t s) {
    if (batch <= 0 || n_q <= 0) return cudaSuccess;
    const dim3 grid(batch, n_q, a.n_q_heads);
    const size_t smem = sizeof(float) * size_t(d_head) * (1 + kGenWarps);
    if (kv_dtype == EP_BF16)
        generic_decode_kernel<__nv_bfloat16><<<grid, kGenWarps * 32, smem, s>>>(a, d_head);
    else
        generic_decode_kernel<float><<<grid, kGenWarps * 32, smem, s>>>(a, d_head);
    return cudaGetLastError();
}

int decode_ctas_per_sm(int, int, int) { return 1; }

cudaError_t launch_spliced_decode(int kv_dtype, int d_head, int rows, int n_ctas,
                                  const DecodeArgs& a, cudaStream_t s) {
    rows = rows <= 1 ? 1 : rows <= 2 ? 2 : rows <= 4 ? 4 : rows <= 8 ? 8 : rows;
    if (kv_dtype == EP_BF16) {
        return d_head == 128 ? dispatch_rows<__nv_bfloat16, 128>(rows, n_ctas, a, s)
                             : dispatch_rows<__nv_bfloat16, 64>(rows, n_ctas, a, s);
    }
    return d_head == 128 ? dispatch_rows<float, 128>(rows, n_ctas, a, s)
                         : dispatch_rows<float, 64>(rows, n_ctas, a, s);
}

cudaError_t launch_empty_units(int d_head, int rows, const DecodeArgs& a, cudaStream_t s) {
    const int units = a.batch * a.n_kv_heads;
    if (units == 0) return cudaSuccess;
    // rows = G * n_q rows of one (request, kv-head) unit
    empty_units_kernel<<<units, 128, 0, s>>>(a, d_head, rows);
    return cudaGetLastError();
}

}  // namespace ep
