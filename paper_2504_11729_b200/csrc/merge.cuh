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

// o_part[(item * stride + r) * D + c], lse_part[item * stride + r] (log2);
// rows r = r0, r0 + r_step, ... < nrows; orow(r) = output row index.
template <int D, typename RowMap>
__device__ __forceinline__ void merge_unit_rows(const DecodeArgs& a, int u0, int n, int stride,
                                                int nrows, int r0, int r_step, RowMap orow_of) {
    constexpr int E = D / 32;
    static_assert(E == 2 || E == 4, "D must be 64 or 128");
    const int lane = threadIdx.x & 31;
    for (int r = r0; r < nrows; r += r_step) {
        float M = -INFINITY;
        for (int base = 0; base < n; base += 32) {
            const float ls = base + lane < n ? __ldcg(&a.lse_part[size_t(u0 + base + lane) * stride + r])
                                             : -INFINITY;
            M = fmaxf(M, ls);
        }
        M = warp_max(M);
        float L = 0.f;
        float acc[E];
#pragma unroll
        for (int e = 0; e < E; ++e) acc[e] = 0.f;
        if (M != -INFINITY) {
            for (int base = 0; base < n; base += 32) {
                const float ls = base + lane < n ? __ldcg(&a.lse_part[size_t(u0 + base + lane) * stride + r])
                                                 : -INFINITY;
                const float wt = ls == -INFINITY ? 0.f : fast_exp2(ls - M);
                L += wt;
                const int cnt = min(32, n - base);
#pragma unroll 4
                for (int j = 0; j < cnt; ++j) {
                    const float wj = __shfl_sync(0xffffffffu, wt, j);
                    const float* src = a.o_part + (size_t(u0 + base + j) * stride + r) * D + lane * E;
                    if constexpr (E == 4) {
                        const float4 x = __ldcg(reinterpret_cast<const float4*>(src));
                        acc[0] += wj * x.x;
                        acc[1] += wj * x.y;
                        acc[2] += wj * x.z;
                        acc[3] += wj * x.w;
                    } else {
                        const float2 x = __ldcg(reinterpret_cast<const float2*>(src));
                        acc[0] += wj * x.x;
                        acc[1] += wj * x.y;
                    }
                }
            }
            L = warp_sum(L);
        }
        const bool er = !(L > 0.f);
        const float inv = er ? 0.f : 1.f / L;
        const size_t orow = orow_of(r);
        if (a.o_dtype == EP_BF16) {
            __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(a.o) + orow * D + lane * E;
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e] = __float2bfloat16_rn(acc[e] * inv);
        } else {
            float* dst = static_cast<float*>(a.o) + orow * D + lane * E;
#pragma unroll
            for (int e = 0; e < E; ++e) dst[e] = acc[e] * inv;
        }
        if (lane == 0 && a.lse) a.lse[orow] = er ? -INFINITY : (M + fast_log2(L)) * kLn2;
    }
}

}  // namespace ep
