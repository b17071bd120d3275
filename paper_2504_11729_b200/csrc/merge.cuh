// merge.cuh — the fused K2 merge used by K1 and K3: the last CTA to finish an
// item of a split (request, kv-head) unit folds the unit's fp32 partials in
// item (= page = segment) order, as merge_partials does
// (/root/reference/proj/core/src/attention.cpp:116-145), but warp-per-row:
// lanes load the items' lse in parallel (warp max / sum), then stream the
// partial rows with vector loads (lane = D/32 contiguous columns).
#pragma once

#include <cstdint>

#include "ep_common.cuh"
#include "ep_internal.h"

namespace ep {

// ---- fused split-KV combine (config 4, K1 with a PeerLink) ----
// A unit's merged local row (this rank's KV shard) goes to slot [rank] of
// every rank's receive buffer (own included) as {value, flag} words of the
// step epoch; a lane holds columns [lane*E, lane*E + E). Never waits.
template <int D>
__device__ __forceinline__ void peer_push_row(const DecodeArgs& a, int unit, size_t orow, const float* v,
                                              float lse2) {
    constexpr int E = D / 32, H = D / 2;
    const int lane = threadIdx.x & 31;
    const uint32_t ep = __ldcg(a.peer.epoch + unit) + 1u;
    const size_t off = size_t(ep & 1u) * a.peer.world * a.peer.src_units +
                       size_t(a.peer.rank) * a.peer.src_units + orow * (H + 1);
    const float lse = lse2 == -INFINITY ? -INFINITY : lse2 * kLn2;  // natural log, as the combine
    for (int p = 0; p < a.peer.world; ++p) {
        uint4* dst = a.peer.recv[p] + off;
#pragma unroll
        for (int j = 0; j < E / 2; ++j) st_ll(dst + lane * (E / 2) + j, v[2 * j], v[2 * j + 1], ep);
        if (lane == 0) st_ll(dst + H, lse, 0.f, ep);
    }
}

// At the end of K1: the units this CTA owns (the CTA of each unit's last
// work item) — one warp per row polls the W ranks' words of the row and
// folds them in rank (= KV segment) order (attention.cpp:116-145): the same
// arithmetic on every rank, so every rank ends with identical rows. Called
// by n_grp warps (this one is gw); the caller advances the units' epochs
// once every warp is done.
template <int D>
__device__ __forceinline__ void peer_merge_owned(const DecodeArgs& a, int gw, int n_grp) {
    constexpr int E = D / 32, H = D / 2;
    const int lane = threadIdx.x & 31;
    const int Hkv = a.n_kv_heads, G = a.n_q_heads / Hkv, W = a.peer.world;
    const int u0 = a.peer.cta_unit_ptr[blockIdx.x], u1 = a.peer.cta_unit_ptr[blockIdx.x + 1];
    const uint4* mine = a.peer.recv[a.peer.rank];
    for (int u = u0; u < u1; ++u) {
        const uint32_t ep = __ldcg(a.peer.epoch + u) + 1u;
        const size_t par = size_t(ep & 1u) * W * a.peer.src_units;
        const int b = u / Hkv, g = u % Hkv, nrows = valid_rows(a, b);
        for (int r = gw; r < nrows; r += n_grp) {
            const size_t orow = (q_row_base(a, b) + r / G) * a.n_q_heads + size_t(g) * G + r % G;
            float lse_p[kPeerMaxWorld];
            float M = -INFINITY;
            for (int p = 0; p < W; ++p) {
                float2 x = make_float2(0.f, 0.f);
                if (lane == 0) x = ld_ll(mine + par + size_t(p) * a.peer.src_units + orow * (H + 1) + H, ep);
                lse_p[p] = __shfl_sync(0xffffffffu, x.x, 0);
                M = fmaxf(M, lse_p[p]);
            }
            float acc[E];
#pragma unroll
            for (int e = 0; e < E; ++e) acc[e] = 0.f;
            float L = 0.f;
            for (int p = 0; p < W; ++p) {
                const float wt = (M == -INFINITY || lse_p[p] == -INFINITY) ? 0.f : expf(lse_p[p] - M);
                L += wt;
                const uint4* src = mine + par + size_t(p) * a.peer.src_units + orow * (H + 1) + lane * (E / 2);
#pragma unroll
                for (int j = 0; j < E / 2; ++j) {  // every word is consumed (it carries the flag)
                    const float2 x = ld_ll(src + j, ep);
                    acc[2 * j] += wt * x.x;
                    acc[2 * j + 1] += wt * x.y;
                }
            }
            const float inv = L > 0.f ? 1.f / L : 0.f;
            if (a.o_dtype == EP_BF16) {
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(a.o) + orow * D + lane * E;
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e] = __float2bfloat16_rn(acc[e] * inv);
            } else {
                float* dst = static_cast<float*>(a.o) + orow * D + lane * E;
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e] = acc[e] * inv;
            }
            if (lane == 0 && a.lse) a.lse[orow] = L > 0.f ? M + logf(L) : -INFINITY;
        }
    }
}

// o_part[(item * stride + r) * D + c], lse_part[item * stride + r] (log2);
// rows r = r0, r0 + r_step, ... < nrows; orow(r) = output row index; with a
// PeerLink the merged rows of `unit` are pushed to every rank instead.
// Latency-bound by construction (a few rows x a few items of L2 reads), so a
// warp works on kRB rows at once: their lse loads, then their partial rows of
// two items at a time, all in flight together (a K3 shared-prefix tile merges
// 128 rows x 2-3 items; serial per-row loads made that the CTA's tail).
template <int D, typename RowMap>
__device__ __forceinline__ void merge_unit_rows(const DecodeArgs& a, int u0, int n, int stride,
                                                int nrows, int r0, int r_step, RowMap orow_of, int unit = -1) {
    constexpr int E = D / 32;
    constexpr int kRB = 4;
    static_assert(E == 2 || E == 4, "D must be 64 or 128");
    const int lane = threadIdx.x & 31;
    for (int rb = r0; rb < nrows; rb += kRB * r_step) {
        int rr[kRB];
        bool ok[kRB];
#pragma unroll
        for (int k = 0; k < kRB; ++k) {
            rr[k] = rb + k * r_step;
            ok[k] = rr[k] < nrows;
        }
        // row max / weights over the items' lse (lane = item within a chunk of 32)
        float M[kRB], L[kRB], inv[kRB], acc[kRB][E];
#pragma unroll
        for (int k = 0; k < kRB; ++k) {
            M[k] = -INFINITY;
            L[k] = 0.f;
#pragma unroll
            for (int e = 0; e < E; ++e) acc[k][e] = 0.f;
        }
        for (int base = 0; base < n; base += 32) {
            float ls[kRB];
#pragma unroll
            for (int k = 0; k < kRB; ++k)
                ls[k] = (ok[k] && base + lane < n) ? __ldcg(&a.lse_part[size_t(u0 + base + lane) * stride + rr[k]])
                                                   : -INFINITY;
#pragma unroll
            for (int k = 0; k < kRB; ++k) M[k] = fmaxf(M[k], warp_max(ls[k]));
        }
        for (int base = 0; base < n; base += 32) {
            float wt[kRB];
#pragma unroll
            for (int k = 0; k < kRB; ++k) {
                const float ls = (ok[k] && base + lane < n)
                                     ? __ldcg(&a.lse_part[size_t(u0 + base + lane) * stride + rr[k]])
                                     : -INFINITY;
                wt[k] = (ls == -INFINITY || M[k] == -INFINITY) ? 0.f : fast_exp2(ls - M[k]);
                L[k] += wt[k];
            }
            const int cnt = min(32, n - base);
            if (!ok[1]) {
                // one row in this warp's batch (a K1 unit has 4 rows for 8
                // warps): its items 8 at a time, all in flight (a long unit is
                // split into ~20 items at batch 1 — config 4)
                for (int j = 0; j < cnt; j += 8) {
                    float x[8][E];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const bool live = j + q < cnt;
                        const float* src = a.o_part + (size_t(u0 + base + (live ? j + q : j)) * stride + rr[0]) * D + lane * E;
                        if constexpr (E == 4) {
                            const float4 v = live ? __ldcg(reinterpret_cast<const float4*>(src)) : make_float4(0, 0, 0, 0);
                            x[q][0] = v.x; x[q][1] = v.y; x[q][2] = v.z; x[q][3] = v.w;
                        } else {
                            const float2 v = live ? __ldcg(reinterpret_cast<const float2*>(src)) : make_float2(0, 0);
                            x[q][0] = v.x; x[q][1] = v.y;
                        }
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float w = __shfl_sync(0xffffffffu, wt[0], min(j + q, cnt - 1));
                        if (j + q < cnt) {
#pragma unroll
                            for (int e = 0; e < E; ++e) acc[0][e] += w * x[q][e];
                        }
                    }
                }
                continue;
            }
            for (int j = 0; j < cnt; j += 2) {
                const bool two = j + 1 < cnt;
                float x0[kRB][E], x1[kRB][E];
#pragma unroll
                for (int k = 0; k < kRB; ++k) {
                    const float* s0 = a.o_part + (size_t(u0 + base + j) * stride + (ok[k] ? rr[k] : 0)) * D + lane * E;
                    const float* s1 = s0 + size_t(stride) * D;
                    if constexpr (E == 4) {
                        const float4 v0 = __ldcg(reinterpret_cast<const float4*>(s0));
                        const float4 v1 = two ? __ldcg(reinterpret_cast<const float4*>(s1)) : make_float4(0, 0, 0, 0);
                        x0[k][0] = v0.x; x0[k][1] = v0.y; x0[k][2] = v0.z; x0[k][3] = v0.w;
                        x1[k][0] = v1.x; x1[k][1] = v1.y; x1[k][2] = v1.z; x1[k][3] = v1.w;
                    } else {
                        const float2 v0 = __ldcg(reinterpret_cast<const float2*>(s0));
                        const float2 v1 = two ? __ldcg(reinterpret_cast<const float2*>(s1)) : make_float2(0, 0);
                        x0[k][0] = v0.x; x0[k][1] = v0.y;
                        x1[k][0] = v1.x; x1[k][1] = v1.y;
                    }
                }
#pragma unroll
                for (int k = 0; k < kRB; ++k) {
                    const float w0 = __shfl_sync(0xffffffffu, wt[k], j);
                    const float w1 = __shfl_sync(0xffffffffu, wt[k], two ? j + 1 : j);
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        acc[k][e] += w0 * x0[k][e];
                        if (two) acc[k][e] += w1 * x1[k][e];
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < kRB; ++k) {
            L[k] = warp_sum(L[k]);
            inv[k] = L[k] > 0.f ? 1.f / L[k] : 0.f;
        }
#pragma unroll
        for (int k = 0; k < kRB; ++k) {
            if (!ok[k]) continue;
            const bool er = !(L[k] > 0.f);
            const size_t orow = orow_of(rr[k]);
            EP_DCHECK(int64_t(orow) < a.n_q_rows * a.n_q_heads);
            if (a.peer.world) {  // fused split-KV: this rank's merged row goes to every rank
                float v[E];
#pragma unroll
                for (int e = 0; e < E; ++e) v[e] = acc[k][e] * inv[k];
                peer_push_row<D>(a, unit, orow, v, er ? -INFINITY : M[k] + fast_log2(L[k]));
                continue;
            }
            if (a.o_dtype == EP_BF16) {
                __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(a.o) + orow * D + lane * E;
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e] = __float2bfloat16_rn(acc[k][e] * inv[k]);
            } else {
                float* dst = static_cast<float*>(a.o) + orow * D + lane * E;
#pragma unroll
                for (int e = 0; e < E; ++e) dst[e] = acc[k][e] * inv[k];
            }
            if (lane == 0 && a.lse) a.lse[orow] = er ? -INFINITY : (M[k] + fast_log2(L[k])) * kLn2;
        }
    }
}

}  // namespace ep
