// kern_reference.cu — general-shape kernels behind the drop-in entry points:
// partial attention over one segment (attention.cpp:80-114), the K2 LSE merge
// (attention.cpp:116-145) and the SplitMix64 input generator (rng.hpp:10-29).
//
// These serve arbitrary (n_q, n_keys, d <= 256) shapes in fp64 or fp32 — the
// per-head calls the reference model makes (model.cpp:171-178). The
// bandwidth-critical batched path is kern_decode.cu.
#include <cmath>
#include <cstdint>

#include "ep_common.cuh"
#include "ep_internal.h"

namespace ep {
namespace {

constexpr int kGenWarps = 4;
constexpr int kMaxD = 256;

template <typename T>
__device__ __forceinline__ T dev_exp(T x);
template <>
__device__ __forceinline__ double dev_exp<double>(double x) {
    return exp(x);
}
template <>
__device__ __forceinline__ float dev_exp<float>(float x) {
    return expf(x);
}
template <typename T>
__device__ __forceinline__ T dev_log(T x);
template <>
__device__ __forceinline__ double dev_log<double>(double x) {
    return log(x);
}
template <>
__device__ __forceinline__ float dev_log<float>(float x) {
    return logf(x);
}

template <typename T>
__device__ __forceinline__ T neg_inf();
template <>
__device__ __forceinline__ double neg_inf<double>() {
    return -INFINITY;
}
template <>
__device__ __forceinline__ float neg_inf<float>() {
    return -INFINITY;
}

// One CTA per query row; warp w takes keys w, w+4, ... of the visible prefix
// (attention.cpp:29-33) with an online softmax, lanes stride over d; the four
// warp states are merged in shared memory. A row with no visible key is the
// identity: out = 0, lse = -inf (attention.cpp:91).
template <typename T>
__global__ void __launch_bounds__(kGenWarps * 32)
    partial_generic_kernel(const T* __restrict__ q, size_t ldq, const T* __restrict__ k,
                           size_t ldk, const T* __restrict__ v, size_t ldv, size_t n_keys,
                           int d, size_t q_off, size_t k_off, T* __restrict__ out, size_t ldo,
                           T* __restrict__ lse) {
    constexpr int kPer = kMaxD / 32;
    __shared__ T s_m[kGenWarps], s_l[kGenWarps];
    __shared__ T s_o[kGenWarps][kMaxD];

    const size_t row = blockIdx.x;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const size_t qpos = q_off + row;
    size_t vis = 0;
    if (qpos >= k_off) {
        vis = qpos - k_off + 1;
        if (vis > n_keys) vis = n_keys;
    }
    const T scale = T(1.0 / sqrt(double(d)));

    T qr[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = lane + 32 * i;
        qr[i] = c < d ? q[row * ldq + c] : T(0);
    }
    T m = neg_inf<T>(), l = T(0);
    T o[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) o[i] = T(0);

    for (size_t j = warp; j < vis; j += kGenWarps) {
        const T* kj = k + j * ldk;
        T dot = T(0);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = lane + 32 * i;
            if (c < d) dot += qr[i] * kj[c];
        }
        dot = warp_sum(dot);
        const T s = dot * scale;
        const T m_new = s > m ? s : m;
        const T corr = dev_exp(m - m_new);
        const T p = dev_exp(s - m_new);
        l = l * corr + p;
        const T* vj = v + j * ldv;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = lane + 32 * i;
            o[i] = o[i] * corr + (c < d ? p * vj[c] : T(0));
        }
        m = m_new;
    }
    if (lane == 0) {
        s_m[warp] = m;
        s_l[warp] = l;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = lane + 32 * i;
        if (c < d) s_o[warp][c] = o[i];
    }
    __syncthreads();
    T M = neg_inf<T>();
#pragma unroll
    for (int w = 0; w < kGenWarps; ++w) M = s_m[w] > M ? s_m[w] : M;
    if (vis == 0) {
        for (int c = threadIdx.x; c < d; c += blockDim.x) out[row * ldo + c] = T(0);
        if (threadIdx.x == 0) lse[row] = neg_inf<T>();
        return;
    }
    T L = T(0);
    T wgt[kGenWarps];
#pragma unroll
    for (int w = 0; w < kGenWarps; ++w) {
        wgt[w] = s_l[w] > T(0) ? dev_exp(s_m[w] - M) : T(0);
        L += wgt[w] * s_l[w];
    }
    const T inv = T(1) / L;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        T acc = T(0);
#pragma unroll
        for (int w = 0; w < kGenWarps; ++w) acc += wgt[w] * s_o[w][c];
        out[row * ldo + c] = acc * inv;
    }
    if (threadIdx.x == 0) lse[row] = M + dev_log(L);
}

// log(exp(a) + exp(b)) with -inf as identity (matrix.cpp:88-93).
template <typename T>
__device__ __forceinline__ T log_add_exp(T a, T b) {
    if (isinf(a) && a < T(0)) return b;
    if (isinf(b) && b < T(0)) return a;
    const T m = a > b ? a : b;
    return m + dev_log(dev_exp(a - m) + dev_exp(b - m));
}

// K2, general shape: one CTA per row; fold lse in part order, then
// out = sum_p exp(lse_p - total) * out_p skipping zero weights
// (attention.cpp:128-144). outs [P][rows][d], lses [P][rows].
template <typename T>
__global__ void merge_generic_kernel(size_t n_parts, const T* __restrict__ outs,
                                     const T* __restrict__ lses, size_t rows, int d,
                                     T* __restrict__ out, T* __restrict__ lse) {
    const size_t row = blockIdx.x;
    T total = neg_inf<T>();
    for (size_t p = 0; p < n_parts; ++p) total = log_add_exp(total, lses[p * rows + row]);
    if (threadIdx.x == 0) lse[row] = total;
    const bool empty = isinf(total) && total < T(0);
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        T acc = T(0);
        if (!empty) {
            for (size_t p = 0; p < n_parts; ++p) {
                const T alpha = dev_exp(lses[p * rows + row] - total);
                if (alpha == T(0)) continue;
                acc += alpha * outs[(p * rows + row) * d + c];
            }
        }
        out[row * d + c] = acc;
    }
}

// rng.hpp:15-27 at draw index i (state after i+1 increments).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void fill_uniform_kernel(int dt, void* dst, size_t n, uint64_t seed, double lo,
                                    double hi) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const double u = double(splitmix_at(seed, i) >> 11) * 0x1.0p-53;
        const double x = lo + (hi - lo) * u;
        if (dt == EP_BF16)
            static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(__double2float_rn(x));
        else if (dt == EP_F32)
            static_cast<float*>(dst)[i] = __double2float_rn(x);
        else
            static_cast<double*>(dst)[i] = x;
    }
}

}  // namespace

cudaError_t launch_partial_generic(int dt, const void* q, size_t ldq, size_t n_q, const void* k,
                                   size_t ldk, const void* v, size_t ldv, size_t n_keys, size_t d,
                                   size_t q_off, size_t k_off, void* out, size_t ldo, void* lse,
                                   cudaStream_t s) {
    if (n_q == 0) return cudaSuccess;
    if (dt == EP_F64)
        partial_generic_kernel<double><<<unsigned(n_q), kGenWarps * 32, 0, s>>>(
            static_cast<const double*>(q), ldq, static_cast<const double*>(k), ldk,
            static_cast<const double*>(v), ldv, n_keys, int(d), q_off, k_off,
            static_cast<double*>(out), ldo, static_cast<double*>(lse));
    else
        partial_generic_kernel<float><<<unsigned(n_q), kGenWarps * 32, 0, s>>>(
            static_cast<const float*>(q), ldq, static_cast<const float*>(k), ldk,
            static_cast<const float*>(v), ldv, n_keys, int(d), q_off, k_off,
            static_cast<float*>(out), ldo, static_cast<float*>(lse));
    return cudaGetLastError();
}

cudaError_t launch_merge_generic(int dt, size_t n_parts, const void* outs, const void* lses,
                                 size_t rows, size_t d, void* out, void* lse, cudaStream_t s) {
    if (rows == 0) return cudaSuccess;
    const unsigned threads = d >= 128 ? 128 : 32;
    if (dt == EP_F64)
        merge_generic_kernel<double><<<unsigned(rows), threads, 0, s>>>(
            n_parts, static_cast<const double*>(outs), static_cast<const double*>(lses), rows,
            int(d), static_cast<double*>(out), static_cast<double*>(lse));
    else
        merge_generic_kernel<float><<<unsigned(rows), threads, 0, s>>>(
            n_parts, static_cast<const float*>(outs), static_cast<const float*>(lses), rows,
            int(d), static_cast<float*>(out), static_cast<float*>(lse));
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform(int dt, void* dst, size_t n, uint64_t seed, double lo, double hi,
                                cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    size_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    fill_uniform_kernel<<<unsigned(blocks), 256, 0, s>>>(dt, dst, n, seed, lo, hi);
    return cudaGetLastError();
}

}  // namespace ep

namespace ep {
namespace {

// One CTA per appended token row: copies its n_kv_heads x d_head K and V rows
// into (page, slot) of the [page][head][slot][d] pool with 16-byte accesses.
__global__ void kv_append_kernel(int row_bytes, int n_kv_heads, int page_tokens,
                                 const int32_t* __restrict__ dst_page,
                                 const int32_t* __restrict__ dst_slot,
                                 const uint8_t* __restrict__ k_new, const uint8_t* __restrict__ v_new,
                                 uint8_t* __restrict__ k_pages, uint8_t* __restrict__ v_pages, int64_t num_pages) {
    const int i = blockIdx.x;
    // PDL: let the next kernel (the attention) start its prologue now; the
    // rows are written only after the predecessor (plan patch / previous
    // step) has completed
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    EP_DCHECK(num_pages < 0 || (dst_page[i] >= 0 && dst_page[i] < num_pages));
    EP_DCHECK(dst_slot[i] >= 0 && dst_slot[i] < page_tokens);
    const size_t page = size_t(dst_page[i]), slot = size_t(dst_slot[i]);
    const int chunks = row_bytes / 16;
    for (int c = threadIdx.x; c < n_kv_heads * chunks; c += blockDim.x) {
        const int g = c / chunks, x = c % chunks;
        const size_t src = (size_t(i) * n_kv_heads + g) * row_bytes + size_t(x) * 16;
        const size_t dst = ((page * n_kv_heads + g) * page_tokens + slot) * row_bytes + size_t(x) * 16;
        *reinterpret_cast<uint4*>(k_pages + dst) = *reinterpret_cast<const uint4*>(k_new + src);
        *reinterpret_cast<uint4*>(v_pages + dst) = *reinterpret_cast<const uint4*>(v_new + src);
    }
}

}  // namespace

__global__ void plan_patch_kernel(const PlanPatch pp) {
    // PDL: the descriptors change only after the previous attention (which
    // reads them) has completed; the next kernel may be scheduled meanwhile
    asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (int i = threadIdx.x; i < pp.n; i += blockDim.x) {
        pp.pdesc[pp.idx[i]].n_tok = pp.ntok[i];
        pp.q_pos[pp.req[i]] = pp.qpos[i];
    }
}

cudaError_t launch_plan_patch(const PlanPatch& pp, cudaStream_t s) {
    if (pp.n <= 0) return cudaSuccess;
    return launch_with_pdl(plan_patch_kernel, dim3(1), dim3(128), 0, s, pp);
}

cudaError_t launch_kv_append(int row_bytes, int n_kv_heads, int page_tokens, int n_rows,
                             const int32_t* dst_page, const int32_t* dst_slot, const void* k_new,
                             const void* v_new, void* k_pages, void* v_pages, cudaStream_t s,
                             int64_t num_pages) {
    if (n_rows <= 0) return cudaSuccess;
    return launch_with_pdl(kv_append_kernel, dim3(n_rows), dim3(128), 0, s, row_bytes, n_kv_heads, page_tokens,
                           dst_page, dst_slot, static_cast<const uint8_t*>(k_new),
                           static_cast<const uint8_t*>(v_new), static_cast<uint8_t*>(k_pages),
                           static_cast<uint8_t*>(v_pages), num_pages);
}

}  // namespace ep

namespace ep {
namespace {

// K5 merge: n_parts rank partials packed as [part][rows * d (o) | rows (lse,
// natural log)] — the layout one all-gather of each rank's (o, lse) produces.
// Folds in part (= rank = segment) order like merge_partials
// (attention.cpp:116-145): one warp per row, lanes over d.
__global__ void merge_packed_kernel(int n_parts, const float* __restrict__ packed, int rows, int d,
                                    void* out, int out_dtype, float* __restrict__ lse_out) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const size_t part_stride = size_t(rows) * (d + 1);
    float M = -INFINITY;
    for (int p = 0; p < n_parts; ++p)
        M = fmaxf(M, packed[p * part_stride + size_t(rows) * d + row]);
    float L = 0.f;
    float acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = 0.f;
    if (M != -INFINITY) {
        for (int p = 0; p < n_parts; ++p) {
            const float wt = expf(packed[p * part_stride + size_t(rows) * d + row] - M);
            if (wt == 0.f) continue;
            L += wt;
            const float* o = packed + p * part_stride + size_t(row) * d;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int c = lane + 32 * i;
                if (c < d) acc[i] += wt * o[c];
            }
        }
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int c = lane + 32 * i;
        if (c >= d) continue;
        if (out_dtype == EP_BF16)
            static_cast<__nv_bfloat16*>(out)[size_t(row) * d + c] = __float2bfloat16_rn(acc[i] * inv);
        else
            static_cast<float*>(out)[size_t(row) * d + c] = acc[i] * inv;
    }
    if (lane == 0 && lse_out) lse_out[row] = L > 0.f ? M + logf(L) : -INFINITY;
}

}  // namespace

cudaError_t launch_merge_packed(int n_parts, const float* packed, int rows, int d, void* out,
                                int out_dtype, float* lse, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    merge_packed_kernel<<<(rows + 3) / 4, 128, 0, s>>>(n_parts, packed, rows, d, out, out_dtype, lse);
    return cudaGetLastError();
}

}  // namespace ep

namespace ep {
namespace {

// Cascade merge (config 5): per output row, the shared-prefix partial (part 0,
// keys at the lowest positions — only for requests that have one) and the
// private-remainder partial (part 1), folded in that (segment) order by LSE as
// merge_partials does (attention.cpp:116-145). One warp per row.
__global__ void cascade_merge_kernel(int rows, int d, int row_per_req, const float* __restrict__ po,
                                     const float* __restrict__ pl, const uint8_t* __restrict__ has_shared,
                                     void* o, int o_dtype, float* __restrict__ lse) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= rows) return;
    const bool sh = has_shared[row / row_per_req] != 0;
    if (d == 128) {
        // one float4 of each part per lane, loaded with the lse values (one
        // round trip); an empty part's garbage is discarded by the select
        const float4 a = __ldcg(reinterpret_cast<const float4*>(po + size_t(row) * d) + lane);
        const float4 b = __ldcg(reinterpret_cast<const float4*>(po + (size_t(rows) + row) * d) + lane);
        const float l0 = sh ? pl[row] : -INFINITY, l1 = pl[rows + row];
        const float M = fmaxf(l0, l1);
        const float w0 = (M == -INFINITY || l0 == -INFINITY) ? 0.f : expf(l0 - M);
        const float w1 = (M == -INFINITY || l1 == -INFINITY) ? 0.f : expf(l1 - M);
        const float L = w0 + w1;
        const float inv = L > 0.f ? 1.f / L : 0.f;
        const float c0 = w0 * inv, c1 = w1 * inv;
        float v[4] = {a.x, a.y, a.z, a.w}, u[4] = {b.x, b.y, b.z, b.w}, r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = (w0 > 0.f ? v[k] * c0 : 0.f) + (w1 > 0.f ? u[k] * c1 : 0.f);
        if (o_dtype == EP_BF16) {
            const __nv_bfloat162 p0 = __floats2bfloat162_rn(r[0], r[1]), p1 = __floats2bfloat162_rn(r[2], r[3]);
            uint2 w;
            w.x = *reinterpret_cast<const uint32_t*>(&p0);
            w.y = *reinterpret_cast<const uint32_t*>(&p1);
            reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(o) + size_t(row) * d)[lane] = w;
        } else {
            reinterpret_cast<float4*>(static_cast<float*>(o) + size_t(row) * d)[lane] = make_float4(r[0], r[1], r[2], r[3]);
        }
        if (lane == 0 && lse) lse[row] = L > 0.f ? M + logf(L) : -INFINITY;
        return;
    }
    const float l0 = sh ? pl[row] : -INFINITY, l1 = pl[rows + row];
    const float M = fmaxf(l0, l1);
    const float w0 = (M == -INFINITY || l0 == -INFINITY) ? 0.f : expf(l0 - M);
    const float w1 = (M == -INFINITY || l1 == -INFINITY) ? 0.f : expf(l1 - M);
    const float L = w0 + w1;
    const float inv = L > 0.f ? 1.f / L : 0.f;
    for (int c = lane; c < d; c += 32) {
        const float x0 = w0 > 0.f ? po[size_t(row) * d + c] * w0 : 0.f;
        const float x1 = w1 > 0.f ? po[(size_t(rows) + row) * d + c] * w1 : 0.f;
        const float val = (x0 + x1) * inv;
        if (o_dtype == EP_BF16)
            static_cast<__nv_bfloat16*>(o)[size_t(row) * d + c] = __float2bfloat16_rn(val);
        else
            static_cast<float*>(o)[size_t(row) * d + c] = val;
    }
    if (lane == 0 && lse) lse[row] = L > 0.f ? M + logf(L) : -INFINITY;
}

}  // namespace

cudaError_t launch_cascade_merge(int rows, int d, int row_per_req, const float* o_parts,
                                 const float* lse_parts, const uint8_t* has_shared, void* o,
                                 int o_dtype, float* lse, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    cascade_merge_kernel<<<(rows + 7) / 8, 256, 0, s>>>(rows, d, row_per_req, o_parts, lse_parts,
                                                        has_shared, o, o_dtype, lse);
    return cudaGetLastError();
}

}  // namespace ep
