// kern_model.cu — the decoder layer around the spliced attention (SURVEY §8f
// rank 3): embedding, LayerNorm-fused projections with their epilogues
// (Q/K/V + page append, Wo + residual, W1 + bias + ReLU, W2 + bias +
// residual, unembedding), a generic paged causal attention for the shapes
// the specialised kernels do not cover (fp64, any d_head), and argmax.
//
// Reference: /root/reference/proj/core/src/model.cpp — embed :104-129,
// layer_norm :131-150, transformer_layer :152-209, unembed_logits :238-246,
// argmax_token :248-255; matmul matrix.cpp:41-61; partial_attention
// attention.cpp:80-114.
//
// The tiny reference models (d_model 8..256) are launch- and L2-latency
// bound, not HBM or tensor bound: weights of config 1 are 6.6 MB (fp32) and
// stay in L2 across steps. Two dense kernels, both with the LayerNorm of the
// input rows in the prologue (the reference's two-pass mean / variance) and
// the layer's elementwise work in the epilogue:
//   * widths % 4 == 0 (every reference shape of interest): a split-K GEMV on
//     a thread-block cluster per 8-row block — CS CTAs of one cluster take
//     K/CS rows each, every thread keeps 8+ independent 16-byte weight loads
//     in flight, and the cluster's partial tiles are summed in rank order
//     through distributed shared memory by rank 0 (deterministic, no
//     atomics, no second launch); weights are re-read from L2 per row block;
//   * other shapes: a CTA owns 64 output columns of MR rows, its 256 threads
//     split K four ways, every weight element read once per CTA is used for
//     MR FMAs.
#include <algorithm>
#include <cmath>
#include <cstdint>

#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "ep_common.cuh"
#include "model_internal.h"

namespace ep {

namespace {

constexpr int kDenseThreads = 256;
constexpr int kBN = 64;                      // output columns per CTA
constexpr int kKS = kDenseThreads / kBN;     // K slices
constexpr int kKC = 128;                     // K chunk staged in smem
constexpr double kLayerNormEps = 1e-5;       // model.cpp:14
constexpr int kGvCols = 64;                  // output columns per CTA (16 threads x 4)
constexpr int kGvKS = kDenseThreads / 16;    // k-slices per CTA
constexpr int kGvRows = 8;                   // rows (decode batch) per CTA
constexpr int kGvPre = 8;        // weight rows per thread held in registers before the wait
constexpr int kGvMaxK = 32 * 32; // LN rows kept in registers (K <= 1024 with LN)

template <typename T>
__device__ __forceinline__ T ld(const void* p, size_t i) {
    return static_cast<const T*>(p)[i];
}

template <typename T>
__device__ __forceinline__ void store_kv(void* pages, int kv_dtype, size_t idx, T v) {
    if (kv_dtype == EP_F64)
        static_cast<double*>(pages)[idx] = double(v);
    else if (kv_dtype == EP_F32)
        static_cast<float*>(pages)[idx] = float(v);
    else
        static_cast<__nv_bfloat16*>(pages)[idx] = __float2bfloat16_rn(float(v));
}

// Rollout rows: step 0 embeds tokens[r], step s > 0 the previous step's
// greedy token prev[(s - 1) * n + r]; positions are pos[s * n + r].
__device__ __forceinline__ int embed_token(const int32_t* tokens, const int32_t* prev, const int32_t* step, int n,
                                           int r) {
    const int st = step ? *step : 0;
    return st == 0 ? tokens[r] : prev[size_t(st - 1) * n + r];
}

__device__ __forceinline__ int embed_pos(const int32_t* pos, const int32_t* step, int n, int r) {
    return pos[size_t(step ? *step : 0) * n + r];
}

template <typename T, int EPI>
__device__ __forceinline__ void dense_epilogue(const DenseArgs& a, int row, int col, T v) {
    if constexpr (EPI == kEpiStore) {
        static_cast<T*>(a.out)[size_t(row) * a.N + col] = v;
    } else if constexpr (EPI == kEpiResid) {
        // x = hidden + proj (model.cpp:184-185); out = x + h2 + b2 (:199-204)
        v = ld<T>(a.resid, size_t(row) * a.N + col) + v;
        if (a.bias) v = v + ld<T>(a.bias, col);
        static_cast<T*>(a.out)[size_t(row) * a.N + col] = v;
    } else if constexpr (EPI == kEpiRelu) {
        v = v + ld<T>(a.bias, col);  // model.cpp:188-194
        if (v < T(0)) v = T(0);
        static_cast<T*>(a.out)[size_t(row) * a.N + col] = v;
    } else {  // kEpiQKV
        const int D = a.N / 3, which = col / D, cc = col - which * D;
        if (which == 0) {
            static_cast<T*>(a.q_out)[size_t(row) * D + cc] = v;
        } else {
            const int h = cc / a.dh, e = cc - h * a.dh;
            const size_t r = (a.step ? size_t(*a.step) * a.n : 0) + row;  // rollout step rows
            const size_t idx = ((size_t(a.dst_page[r]) * a.H + h) * a.P + a.dst_slot[r]) * a.dh + e;
            store_kv<T>(which == 1 ? a.k_pages : a.v_pages, a.kv_dtype, idx, v);
        }
    }
}

// Dynamic smem: A chunk [MR][kKC] + k-slice partials [kKS-1][MR][kBN].
template <typename T, int MR>
constexpr size_t dense_smem() {
    return sizeof(T) * (size_t(MR) * kKC + size_t(kKS - 1) * MR * kBN);
}

template <typename T, int MR, int EPI, bool LN>
__global__ void __launch_bounds__(kDenseThreads) dense_kernel(const DenseArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = reinterpret_cast<T*>(smem_raw);
    T* red = As + MR * kKC;
    __shared__ T s_mean[MR], s_inv[MR];
    __shared__ int s_row[MR];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int col_l = tid % kBN, ks = tid / kBN;
    const int row0 = blockIdx.y * MR;
    const int nr = min(MR, a.n - row0);
    const int col = blockIdx.x * kBN + col_l;
    const bool cvalid = col < a.N;

    if (tid < MR) s_row[tid] = tid < nr ? (a.row_map ? a.row_map[row0 + tid] : row0 + tid) : 0;
    __syncthreads();
    const T* X = static_cast<const T*>(a.x);

    if constexpr (LN) {
        // layer_norm (model.cpp:131-150): mean, then mean squared deviation,
        // inv = 1 / sqrt(var + eps); one warp per row.
        for (int r = warp; r < nr; r += kDenseThreads / 32) {
            const T* xr = X + size_t(s_row[r]) * a.K;
            T s = 0;
            for (int c = lane; c < a.K; c += 32) s += xr[c];
            s = warp_sum(s);
            const T mean = s / T(a.K);
            T q = 0;
            for (int c = lane; c < a.K; c += 32) {
                const T dx = xr[c] - mean;
                q += dx * dx;
            }
            q = warp_sum(q);
            const T var = q / T(a.K);
            if (lane == 0) {
                s_mean[r] = mean;
                s_inv[r] = T(1) / sqrt(var + T(kLayerNormEps));
            }
        }
        __syncthreads();
    }

    // this thread's weight column (column blocks wq | wk | wv for kEpiQKV)
    const int nb = a.N / a.n_wblk;
    const T* wp = nullptr;
    if (cvalid) {
        const int blk = col / nb;
        wp = static_cast<const T*>(a.w[blk]) + (col - blk * nb);
    }

    T acc[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) acc[r] = T(0);

    for (int k0 = 0; k0 < a.K; k0 += kKC) {
        const int kc = min(kKC, a.K - k0);
        for (int i = tid; i < MR * kKC; i += kDenseThreads) {
            const int r = i / kKC, kk = i - r * kKC;
            T v = T(0);
            if (r < nr && kk < kc) {
                v = X[size_t(s_row[r]) * a.K + k0 + kk];
                if constexpr (LN) v = (v - s_mean[r]) * s_inv[r];
            }
            As[i] = v;
        }
        __syncthreads();
        if (cvalid) {
            const int per = (kc + kKS - 1) / kKS;
            const int kb = ks * per, ke = min(kc, kb + per);
            const T* wk = wp + size_t(k0) * nb;
#pragma unroll 4
            for (int kk = kb; kk < ke; ++kk) {
                const T wv = wk[size_t(kk) * nb];
#pragma unroll
                for (int r = 0; r < MR; ++r) acc[r] += As[r * kKC + kk] * wv;
            }
        }
        __syncthreads();
    }

    // K slices -> slice 0, summed in slice order (deterministic)
    if (ks > 0) {
#pragma unroll
        for (int r = 0; r < MR; ++r) red[((ks - 1) * MR + r) * kBN + col_l] = acc[r];
    }
    __syncthreads();
    if (ks == 0 && cvalid) {
#pragma unroll
        for (int r = 0; r < MR; ++r) {
            if (r >= nr) break;
            T v = acc[r];
#pragma unroll
            for (int s = 0; s < kKS - 1; ++s) v += red[(s * MR + r) * kBN + col_l];
            dense_epilogue<T, EPI>(a, row0 + r, col, v);
        }
    }
}

template <typename T, int MR, int EPI, bool LN>
cudaError_t launch_dense_t(const DenseArgs& a, cudaStream_t s) {
    const size_t smem = dense_smem<T, MR>();
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem<dense_kernel<T, MR, EPI, LN>>(int(smem))) return e;
    dim3 grid((a.N + kBN - 1) / kBN, (a.n + MR - 1) / MR);
    dense_kernel<T, MR, EPI, LN><<<grid, kDenseThreads, smem, s>>>(a);
    return cudaGetLastError();
}

template <typename T, int EPI, bool LN>
cudaError_t launch_gemv_t(const DenseArgs& a, cudaStream_t s);

bool gemv_ok(const DenseArgs& a, bool ln) {
    const int nb = a.N / a.n_wblk;
    bool aligned = nb % 4 == 0 && (!ln || a.K <= kGvMaxK);
    for (int i = 0; i < a.n_wblk; ++i) aligned = aligned && reinterpret_cast<uintptr_t>(a.w[i]) % 16 == 0;
    return aligned;
}

template <typename T, int EPI, bool LN>
cudaError_t dispatch_rows(const DenseArgs& a, cudaStream_t s) {
    // the cluster split-K GEMV (8-row blocks) wherever 16-byte weight loads
    // are aligned (every column block a multiple of 4 wide, 16-byte bases);
    // else the scalar kernel: every CTA streams its weight columns once for up
    // to 8 rows (decode) or 32 rows (prefill).
    if (gemv_ok(a, LN)) return launch_gemv_t<T, EPI, LN>(a, s);
    if (a.emb || a.next) return cudaErrorInvalidValue;  // fused work exists only in the GEMV
    if (a.n <= 8) return launch_dense_t<T, 8, EPI, LN>(a, s);
    return launch_dense_t<T, 32, EPI, LN>(a, s);
}

template <typename T>
cudaError_t dispatch_epi(int epi, bool ln, const DenseArgs& a, cudaStream_t s) {
    switch (epi) {
    case kEpiStore: return ln ? dispatch_rows<T, kEpiStore, true>(a, s) : dispatch_rows<T, kEpiStore, false>(a, s);
    case kEpiQKV: return ln ? dispatch_rows<T, kEpiQKV, true>(a, s) : dispatch_rows<T, kEpiQKV, false>(a, s);
    case kEpiResid: return ln ? dispatch_rows<T, kEpiResid, true>(a, s) : dispatch_rows<T, kEpiResid, false>(a, s);
    case kEpiRelu: return ln ? dispatch_rows<T, kEpiRelu, true>(a, s) : dispatch_rows<T, kEpiRelu, false>(a, s);
    default: return cudaErrorInvalidValue;
    }
}

// ------------------------------------------------------ cluster split-K GEMV --


template <typename T>
struct Vec4 {
    T x, y, z, w;
};

template <typename T>
__device__ __forceinline__ Vec4<T> ld4(const T* p) {
    if constexpr (sizeof(T) == 4) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p));
        return {v.x, v.y, v.z, v.w};
    } else {
        const double2 a = __ldg(reinterpret_cast<const double2*>(p));
        const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
        return {a.x, a.y, b.x, b.y};
    }
}

// Programmatic dependent launch: the weights do not depend on the previous
// kernel, so their loads are issued before griddepcontrol.wait and overlap
// the predecessor's tail; inputs are read only after it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }


// smem: A slice [kGvRows][KR] | k-slice partials [kGvKS][kGvRows][kGvCols]
//       | cluster partial [kGvRows][kGvCols]
template <typename T, int EPI, bool LN>
__global__ void __launch_bounds__(kDenseThreads) gemv_cluster_kernel(const DenseArgs a, int KR) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int crank = int(cluster.block_rank()), csize = int(cluster.num_blocks());
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* As = reinterpret_cast<T*>(smem_raw);
    T* red = As + kGvRows * KR;
    T* part = red + kGvKS * kGvRows * kGvCols;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int row0 = blockIdx.z * kGvRows;
    const int nr = min(kGvRows, a.n - row0);
    const int k0 = crank * KR, kr = max(0, min(KR, a.K - k0));
    const T* X = static_cast<const T*>(a.x);

    // ---- 1. this thread's weight rows (independent of the predecessor) ----
    const int cg4 = tid % 16, ks = tid / 16;
    const int col0 = blockIdx.x * kGvCols + cg4 * 4;
    const bool cvalid = col0 < a.N;  // N % 4 == 0 and block width % 4 == 0
    const int per = (kr + kGvKS - 1) / kGvKS;
    const int kb = ks * per, ke = min(kr, kb + per);
    const T* wp = nullptr;
    int nb = 1;
    Vec4<T> wpre[kGvPre];
    if (cvalid) {
        nb = a.N / a.n_wblk;
        const int blk = col0 / nb;
        wp = static_cast<const T*>(a.w[blk]) + (col0 - blk * nb) + size_t(k0) * nb;
#pragma unroll
        for (int i = 0; i < kGvPre; ++i)
            if (kb + i < ke) wpre[i] = ld4(wp + size_t(kb + i) * nb);
    }

    // ---- 2. inputs: wait for the producer of x, LayerNorm from registers ----
    pdl_wait();
    for (int r = warp; r < kGvRows; r += kDenseThreads / 32) {
        T* dst = As + r * KR;
        if (r >= nr) {
            for (int kk = lane; kk < KR; kk += 32) dst[kk] = T(0);
            continue;
        }
        const int grow = a.row_map ? a.row_map[row0 + r] : row0 + r;
        const T* xr = X + size_t(grow) * a.K;
        if constexpr (LN) {
            // layer_norm (model.cpp:131-150): mean, mean squared deviation,
            // inv = 1 / sqrt(var + eps) — the row is read once into registers
            constexpr int NV = kGvMaxK / 32;
            T v[NV];
            T sm = 0;
            if (a.emb) {
                // fused embedding of the first layer: embedding[token] + pe[pos]
                const int n_rows = a.n;
                const T* e = static_cast<const T*>(a.emb) +
                             size_t(embed_token(a.tok, a.tok_prev, a.step, n_rows, grow)) * a.K;
                const double* pr = a.pe + size_t(embed_pos(a.pos, a.step, n_rows, grow)) * a.K;
                T* xs = (blockIdx.x == 0 && crank == 0) ? static_cast<T*>(a.x_store) + size_t(grow) * a.K : nullptr;
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int c = lane + 32 * i;
                    v[i] = c < a.K ? T(double(e[c]) + pr[c]) : T(0);
                    if (xs && c < a.K) xs[c] = v[i];
                    sm += v[i];
                }
            } else {
#pragma unroll
                for (int i = 0; i < NV; ++i) {
                    const int c = lane + 32 * i;
                    v[i] = c < a.K ? xr[c] : T(0);
                    sm += v[i];
                }
            }
            const T mean = warp_sum(sm) / T(a.K);
            T q = 0;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int c = lane + 32 * i;
                const T dx = v[i] - mean;
                q += c < a.K ? dx * dx : T(0);
            }
            const T inv = T(1) / sqrt(warp_sum(q) / T(a.K) + T(kLayerNormEps));
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int c = lane + 32 * i;
                if (c >= k0 && c < k0 + KR) dst[c - k0] = c < a.K ? (v[i] - mean) * inv : T(0);
            }
        } else {
            for (int kk = lane; kk < KR; kk += 32) dst[kk] = kk < kr ? xr[k0 + kk] : T(0);
        }
    }
    __syncthreads();

    T acc[kGvRows][4];
#pragma unroll
    for (int r = 0; r < kGvRows; ++r) acc[r][0] = acc[r][1] = acc[r][2] = acc[r][3] = T(0);
    if (cvalid) {
#pragma unroll
        for (int i = 0; i < kGvPre; ++i) {
            if (kb + i >= ke) break;
            const Vec4<T> w = wpre[i];
            const int kk = kb + i;
#pragma unroll
            for (int r = 0; r < kGvRows; ++r) {
                const T x = As[r * KR + kk];
                acc[r][0] += x * w.x;
                acc[r][1] += x * w.y;
                acc[r][2] += x * w.z;
                acc[r][3] += x * w.w;
            }
        }
#pragma unroll 4
        for (int kk = kb + kGvPre; kk < ke; ++kk) {
            const Vec4<T> w = ld4(wp + size_t(kk) * nb);
#pragma unroll
            for (int r = 0; r < kGvRows; ++r) {
                const T x = As[r * KR + kk];
                acc[r][0] += x * w.x;
                acc[r][1] += x * w.y;
                acc[r][2] += x * w.z;
                acc[r][3] += x * w.w;
            }
        }
    }
    pdl_trigger();  // the successor may start prefetching its weights
#pragma unroll
    for (int r = 0; r < kGvRows; ++r)
#pragma unroll
        for (int e = 0; e < 4; ++e) red[(ks * kGvRows + r) * kGvCols + cg4 * 4 + e] = acc[r][e];
    __syncthreads();
    // k-slices summed in order -> this CTA's partial tile
    for (int i = tid; i < kGvRows * kGvCols; i += kDenseThreads) {
        T v = T(0);
#pragma unroll 4
        for (int k = 0; k < kGvKS; ++k) v += red[k * kGvRows * kGvCols + i];
        part[i] = v;
    }
    cluster.sync();
    if (crank == 0) {
        for (int i = tid; i < nr * kGvCols; i += kDenseThreads) {
            const int r = i / kGvCols, c = blockIdx.x * kGvCols + (i % kGvCols);
            if (c >= a.N) continue;
            T v = part[i];
            for (int q = 1; q < csize; ++q) v += cluster.map_shared_rank(part, q)[i];
            dense_epilogue<T, EPI>(a, row0 + r, c, v);
        }
    }
    cluster.sync();  // peers' partials stay mapped until rank 0 has read them
    if constexpr (EPI == kEpiStore) {
        if (a.next && crank == 0) {
            // fused argmax_token (model.cpp:248-255): the last CTA to store its
            // logits takes the first maximum of every row, then advances the
            // rollout step
            __shared__ int s_last;
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = atomicAdd(a.arrive, 1) == int(gridDim.x * gridDim.z) - 1;
            __syncthreads();
            if (s_last) {
                __threadfence();
                const T* lg = static_cast<const T*>(a.out);
                const size_t so = a.step ? size_t(*a.step) * a.n : 0;
                for (int r = warp; r < a.n; r += kDenseThreads / 32) {
                    T bv = T(0);
                    int bi = a.N;
                    for (int c = lane; c < a.N; c += 32) {
                        const T v = __ldcg(lg + size_t(r) * a.N + c);
                        if (v == v && (bi == a.N || v > bv)) {  // NaN: see argmax_rows_kernel
                            bv = v;
                            bi = c;
                        }
                    }
#pragma unroll
                    for (int m = 16; m > 0; m >>= 1) {
                        const T ov = __shfl_xor_sync(0xffffffffu, bv, m);
                        const int oi = __shfl_xor_sync(0xffffffffu, bi, m);
                        if (oi < a.N && (bi == a.N || ov > bv || (ov == bv && oi < bi))) {
                            bv = ov;
                            bi = oi;
                        }
                    }
                    if (lane == 0) {
                        const T x0 = __ldcg(lg + size_t(r) * a.N);
                        a.next[so + r] = (bi == a.N || x0 != x0) ? 0 : bi;
                    }
                }
                __syncthreads();
                if (tid == 0) {
                    *a.arrive = 0;  // ready for the next launch
                    if (a.adv_step) *a.adv_step += 1;
                }
                if (a.adv_qpos)
                    for (int b = tid; b < a.n; b += kDenseThreads) a.adv_qpos[b] += 1;
            }
        }
    }
}

template <typename T, int EPI, bool LN>
cudaError_t launch_gemv_t(const DenseArgs& a, cudaStream_t s) {
    // ~128 K-rows per CTA, at most 8 CTAs (the portable cluster size)
    int cs = std::min(8, std::max(1, (a.K + 127) / 128));
    const int KR = (((a.K + cs - 1) / cs) + 15) / 16 * 16;
    cs = (a.K + KR - 1) / KR;
    const size_t smem = sizeof(T) * (size_t(kGvRows) * KR + size_t(kGvKS + 1) * kGvRows * kGvCols);
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem<gemv_cluster_kernel<T, EPI, LN>>(int(smem))) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((a.N + kGvCols - 1) / kGvCols, cs, (a.n + kGvRows - 1) / kGvRows);
    cfg.blockDim = dim3(kDenseThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = cs;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, gemv_cluster_kernel<T, EPI, LN>, a, KR);
}

// ------------------------------------------------------------------ embed --

// With a rollout step counter, step 0 embeds tokens[r] and step s > 0 the
// previous step's greedy token prev[(s - 1) * n + r]; positions are pos[s * n + r].
// out = T(embedding (as fp64) + pe): model.cpp:121-126 adds in double.
template <typename T>
__global__ void embed_kernel(const T* emb, const double* pe, const int32_t* tokens, const int32_t* prev,
                             const int32_t* step, const int32_t* pos, int D, T* out) {
    const int r = blockIdx.x, n = gridDim.x;
    const T* e = emb + size_t(embed_token(tokens, prev, step, n, r)) * D;
    const double* pr = pe + size_t(embed_pos(pos, step, n, r)) * D;
    for (int c = threadIdx.x; c < D; c += blockDim.x) out[size_t(r) * D + c] = T(double(e[c]) + pr[c]);
}

__global__ void posenc_kernel(double* pe, int D) {
    const int p = blockIdx.x;
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
        // model.cpp:121-126: pair = c - c % 2, freq = 10000^(-pair / d)
        const int pair = c - (c % 2);
        const double freq = pow(10000.0, -double(pair) / double(D));
        const double angle = double(p) * freq;
        pe[size_t(p) * D + c] = (c % 2 == 0) ? sin(angle) : cos(angle);
    }
}

// ------------------------------------------------------ generic attention --

constexpr int kAttnWarps = 4;
constexpr int kMaxDhPerLane = 8;  // d_head <= 256

template <typename T, typename KV>
__device__ __forceinline__ T kv_at(const KV* p, size_t i) {
    if constexpr (sizeof(KV) == 2)
        return T(__bfloat162float(p[i]));
    else
        return T(p[i]);
}

template <typename T>
__device__ __forceinline__ T exp_t(T x) {
    if constexpr (sizeof(T) == 8)
        return exp(x);
    else
        return expf(x);
}

// partial_attention's math (attention.cpp:80-114: s = (q . k) * 1/sqrt(d),
// w = exp(s - max), out = sum w v / sum w) over every visible key of the
// request's pages as one online-softmax pass; warps take pages round-robin
// and are merged by LSE at the end (merge_partials, attention.cpp:116-145).
template <typename T, typename KV>
__global__ void __launch_bounds__(kAttnWarps * 32)
    attention_generic_kernel(const T* q, int H, int dh, const PageDesc* pdesc,
                             const int64_t* req_page_off, const int32_t* row_req,
                             const int32_t* row_pos, const int32_t* step, const KV* kp,
                             const KV* vp, int P, T* out) {
    const int r = blockIdx.x, h = blockIdx.y;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* qs = reinterpret_cast<T*>(smem_raw);        // [dh]
    T* wo = qs + dh;                                // [warps][dh]
    __shared__ T wm[kAttnWarps], wl[kAttnWarps];

    const T* qr = q + (size_t(r) * H + h) * dh;
    for (int c = tid; c < dh; c += blockDim.x) qs[c] = qr[c];
    __syncthreads();

    const T scale = T(1) / sqrt(T(dh));
    const int64_t qpos = row_pos[(step ? size_t(*step) * gridDim.x : 0) + r];
    const int b = row_req[r];
    const int64_t p0 = req_page_off[b], np = req_page_off[b + 1] - p0;

    T m = T(-INFINITY), l = T(0);
    T o[kMaxDhPerLane];
#pragma unroll
    for (int i = 0; i < kMaxDhPerLane; ++i) o[i] = T(0);

    for (int64_t pi = warp; pi < np; pi += kAttnWarps) {
        const PageDesc d = pdesc[p0 + pi];
        // visible keys of this page: positions d.pos .. min(d.pos + n_tok, qpos + 1) - 1
        const int64_t vis = qpos - d.pos + 1;
        const int nk = vis <= 0 ? 0 : (vis < d.n_tok ? int(vis) : d.n_tok);
        const size_t tile = (size_t(d.page) * H + h) * size_t(P);
        for (int j0 = 0; j0 < nk; j0 += 32) {
            const int j = j0 + lane;
            T sc = T(-INFINITY);
            if (j < nk) {
                const KV* kr = kp + (tile + j) * dh;
                T dot = T(0);
                for (int c = 0; c < dh; ++c) dot += qs[c] * kv_at<T>(kr, c);
                sc = dot * scale;
            }
            T cm = sc;
#pragma unroll
            for (int msk = 16; msk > 0; msk >>= 1) cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, msk));
            const T nm = max(m, cm);
            const T corr = (m == T(-INFINITY)) ? T(0) : exp_t(m - nm);
            const T p = (j < nk) ? exp_t(sc - nm) : T(0);
            l = l * corr + warp_sum(p);
#pragma unroll
            for (int i = 0; i < kMaxDhPerLane; ++i) o[i] *= corr;
            const int cnt = min(32, nk - j0);
            for (int jj = 0; jj < cnt; ++jj) {
                const T pj = __shfl_sync(0xffffffffu, p, jj);
                const KV* vr = vp + (tile + j0 + jj) * dh;
#pragma unroll
                for (int i = 0; i < kMaxDhPerLane; ++i) {
                    const int c = lane + 32 * i;
                    if (c < dh) o[i] += pj * kv_at<T>(vr, c);
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
    for (int i = 0; i < kMaxDhPerLane; ++i) {
        const int c = lane + 32 * i;
        if (c < dh) wo[warp * dh + c] = o[i];
    }
    __syncthreads();
    T M = T(-INFINITY);
    for (int w = 0; w < kAttnWarps; ++w) M = max(M, wm[w]);
    T L = T(0);
    T wt[kAttnWarps];
    for (int w = 0; w < kAttnWarps; ++w) {
        wt[w] = wm[w] == T(-INFINITY) ? T(0) : exp_t(wm[w] - M);
        L += wt[w] * wl[w];
    }
    const T inv = L > T(0) ? T(1) / L : T(0);
    for (int c = tid; c < dh; c += blockDim.x) {
        T acc = T(0);
        for (int w = 0; w < kAttnWarps; ++w) acc += wt[w] * wo[w * dh + c];
        out[(size_t(r) * H + h) * dh + c] = acc * inv;
    }
}

template <typename T, typename KV>
cudaError_t launch_attn_t(const void* q, int n, int H, int dh, const PageDesc* pdesc,
                          const int64_t* req_page_off, const int32_t* row_req,
                          const int32_t* row_pos, const int32_t* step, const void* kp,
                          const void* vp, int P, void* out, cudaStream_t s) {
    const size_t smem = sizeof(T) * size_t(dh) * (1 + kAttnWarps);
    attention_generic_kernel<T, KV><<<dim3(n, H), kAttnWarps * 32, smem, s>>>(
        static_cast<const T*>(q), H, dh, pdesc, req_page_off, row_req, row_pos, step,
        static_cast<const KV*>(kp), static_cast<const KV*>(vp), P, static_cast<T*>(out));
    return cudaGetLastError();
}

// ----------------------------------------------------------------- argmax --

// argmax_token (model.cpp:248-255): first index of the maximum (strict >).
template <typename T>
__global__ void argmax_rows_kernel(const T* logits, int V, const int32_t* step, int32_t* next) {
    const int r = blockIdx.x, tid = threadIdx.x;
    if (step) next += size_t(*step) * gridDim.x;  // rollout: row block of this step
    const T* x = logits + size_t(r) * V;
    T bv = T(-INFINITY);
    int bi = V;
    for (int i = tid; i < V; i += blockDim.x) {
        const T v = x[i];
        if (v == v && (bi == V || v > bv)) {  // a NaN is never taken (x[0] below)
            bv = v;
            bi = i;
        }
    }
    __shared__ T sv[256];
    __shared__ int si[256];
    sv[tid] = bv;
    si[tid] = bi;
    __syncthreads();
    for (int st = blockDim.x / 2; st > 0; st >>= 1) {
        if (tid < st) {
            const T ov = sv[tid + st];
            const int oi = si[tid + st];
            if (oi < V && (si[tid] == V || ov > sv[tid] || (ov == sv[tid] && oi < si[tid]))) {
                sv[tid] = ov;
                si[tid] = oi;
            }
        }
        __syncthreads();
    }
    // argmax_token starts at id 0: a NaN there is never replaced
    if (tid == 0) next[r] = (si[0] == V || x[0] != x[0]) ? 0 : si[0];
}

// ------------------------------------------------------------- init draws --

__device__ __forceinline__ uint64_t splitmix_draw(uint64_t seed, uint64_t i) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;  // rng.hpp:15-20
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void fill_at_kernel(int dt, void* dst, size_t n, uint64_t seed, uint64_t first,
                               double lo, double hi) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const double u = double(splitmix_draw(seed, first + i) >> 11) * 0x1.0p-53;
        // lo + (hi - lo) * u exactly as rng.hpp:25 (no FMA contraction)
        const double x = __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u));
        if (dt == EP_F64)
            static_cast<double*>(dst)[i] = x;
        else if (dt == EP_F32)
            static_cast<float*>(dst)[i] = __double2float_rn(x);
        else
            static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(__double2float_rn(x));
    }
}

}  // namespace

bool dense_uses_gemv(const DenseArgs& a, bool ln) { return a.n > 0 && a.N > 0 && gemv_ok(a, ln); }

cudaError_t launch_dense(int dt, int epi, bool ln, const DenseArgs& a, cudaStream_t s) {
    if (a.n <= 0 || a.N <= 0) return cudaSuccess;
    return dt == EP_F64 ? dispatch_epi<double>(epi, ln, a, s) : dispatch_epi<float>(epi, ln, a, s);
}

cudaError_t launch_embed(int dt, const void* emb, const double* pe, const int32_t* tokens, const int32_t* prev,
                         const int32_t* step, const int32_t* pos, int n, int D, void* out,
                         cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    const int threads = D >= 256 ? 256 : ((D + 31) / 32) * 32;
    if (dt == EP_F64)
        embed_kernel<double><<<n, threads, 0, s>>>(static_cast<const double*>(emb), pe, tokens, prev, step, pos,
                                                   D, static_cast<double*>(out));
    else
        embed_kernel<float><<<n, threads, 0, s>>>(static_cast<const float*>(emb), pe, tokens, prev, step, pos, D,
                                                  static_cast<float*>(out));
    return cudaGetLastError();
}

cudaError_t launch_posenc(double* pe, int max_positions, int D, cudaStream_t s) {
    if (max_positions <= 0) return cudaSuccess;
    posenc_kernel<<<max_positions, D >= 256 ? 256 : ((D + 31) / 32) * 32, 0, s>>>(pe, D);
    return cudaGetLastError();
}

cudaError_t launch_attention_generic(int dt, int kv_dtype, const void* q, int n, int H, int dh,
                                     const PageDesc* pdesc, const int64_t* req_page_off,
                                     const int32_t* row_req, const int32_t* row_pos,
                                     const int32_t* step, const void* k_pages,
                                     const void* v_pages, int P, void* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (dh > 32 * kMaxDhPerLane) return cudaErrorInvalidValue;
    if (dt == EP_F64) {
        if (kv_dtype != EP_F64) return cudaErrorInvalidValue;
        return launch_attn_t<double, double>(q, n, H, dh, pdesc, req_page_off, row_req, row_pos,
                                             step, k_pages, v_pages, P, out, s);
    }
    if (kv_dtype == EP_F32)
        return launch_attn_t<float, float>(q, n, H, dh, pdesc, req_page_off, row_req, row_pos,
                                           step, k_pages, v_pages, P, out, s);
    if (kv_dtype == EP_BF16)
        return launch_attn_t<float, __nv_bfloat16>(q, n, H, dh, pdesc, req_page_off, row_req,
                                                   row_pos, step, k_pages, v_pages, P, out, s);
    return cudaErrorInvalidValue;
}

__global__ void accept_rows_kernel(const int32_t* tokens, const int32_t* targets, const int32_t* last_row,
                                   int batch, int32_t* n_accepted) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const int r0 = b == 0 ? 0 : last_row[b - 1] + 1, r1 = last_row[b];
    int n = 0;
    while (r0 + n + 1 <= r1 && tokens[r0 + n + 1] == targets[r0 + n]) ++n;
    n_accepted[b] = n;
}

cudaError_t launch_accept_rows(const int32_t* tokens, const int32_t* targets, const int32_t* last_row, int batch,
                               int32_t* n_accepted, cudaStream_t s) {
    if (batch <= 0) return cudaSuccess;
    accept_rows_kernel<<<(batch + 127) / 128, 128, 0, s>>>(tokens, targets, last_row, batch, n_accepted);
    return cudaGetLastError();
}

cudaError_t launch_argmax_rows(int dt, const void* logits, int rows, int V, const int32_t* step,
                               int32_t* next, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    if (dt == EP_F64)
        argmax_rows_kernel<double><<<rows, 256, 0, s>>>(static_cast<const double*>(logits), V, step,
                                                        next);
    else
        argmax_rows_kernel<float><<<rows, 256, 0, s>>>(static_cast<const float*>(logits), V, step,
                                                       next);
    return cudaGetLastError();
}

namespace {
// End of one rollout step: step += 1 and every request's query position
// (the decode plan's q_pos, read by K1/K3) moves to the next token.
__global__ void advance_kernel(int32_t* step, int64_t* q_pos, int batch) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) *step += 1;
    if (q_pos && i < batch) q_pos[i] += 1;
}
}  // namespace

cudaError_t launch_advance(int32_t* step, int64_t* q_pos, int batch, cudaStream_t s) {
    advance_kernel<<<(batch + 255) / 256, 256, 0, s>>>(step, q_pos, batch);
    return cudaGetLastError();
}

cudaError_t launch_fill_uniform_at(int dt, void* dst, size_t n, uint64_t seed, uint64_t first,
                                   double lo, double hi, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    size_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_at_kernel<<<unsigned(blocks), 256, 0, s>>>(dt, dst, n, seed, first, lo, hi);
    return cudaGetLastError();
}

}  // namespace ep
