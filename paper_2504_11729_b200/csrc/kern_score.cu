// kern_score.cu — K4: fused score + greedy accept of speculative verify.
//
// Reference construction: for each verify row j of a request
// (last accepted token, then drafts d1..dk) the target token is
//     g_j = argmax( unembed_logits(row_j) ) = argmax( LN(row_j) @ W )
// (model.cpp:238-255: parameterless LayerNorm, eps 1e-5, then the D x V
// product; argmax with strict '>' so ties keep the lowest id). Accepted
// n = largest n <= k with d_i == g_{i-1} for all i <= n; emitted d1..dn + g_n.
//
// B200 mapping:
//   * row_stats: mean and 1/std of each attention-output row (4096 wide).
//   * score GEMM on tcgen05: Z[128 rows x 256 vocab] (TMEM fp32) over K = 4096
//     in 64-wide TMA-fed stages (A = attention rows, B = W^T, both bf16,
//     128B-swizzled K-major). LayerNorm is folded into the epilogue:
//     LN(x).w = rstd * (x.w - mean * colsum(w)); rstd > 0 does not move the
//     argmax, so the epilogue ranks z = x.w - mean * colsum(w) and reduces
//     (z, lowest index) across the vocab tiles with one 64-bit atomicMax per
//     row per CTA on an order-preserving key.
//   * accept: per request, decode g_j and apply the acceptance rule.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ep_common.cuh"
#include "ep_internal.h"
#include "umma.cuh"

namespace ep {
namespace {

constexpr int kTM = 128, kTN = 256, kTK = 64;
constexpr int kStagesS = 4;
constexpr int kABytes = kTM * kTK * 2;  // 16 KB
constexpr int kBBytes = kTN * kTK * 2;  // 32 KB
constexpr int kStage = kABytes + kBBytes;
constexpr int kScoreThreads = 192;  // warps 0-3 epilogue, 4 TMA, 5 MMA
constexpr int kScoreSmem = kStagesS * kStage + 1024 + 256 + kTN * 4;  // stages, barriers, colsum slice
constexpr uint32_t kIdescScore = umma::idesc_bf16_f32(kTM, kTN, false, false);

__device__ __forceinline__ uint64_t order_key(float z, uint32_t idx) {
    uint32_t b = __float_as_uint(z);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (uint64_t(b) << 32) | uint64_t(0xFFFFFFFFu - idx);
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
template <>
__device__ __forceinline__ float ldf<float>(const float* p) {
    return *p;
}
template <>
__device__ __forceinline__ float ldf<__nv_bfloat16>(const __nv_bfloat16* p) {
    return __bfloat162float(*p);
}

// mean and 1/sqrt(var + 1e-5) per row (model.cpp:131-150), fp32 two-pass.
// For fp32 rows also writes the bf16 hi/lo split [hi(x) | lo(x)] used as a
// 2*width-long A operand: x = hi + lo to ~2^-17, so the bf16 tensor-core
// product keeps fp32-level accuracy.
template <typename T>
__global__ void row_stats_kernel(const T* __restrict__ x, int width, float* __restrict__ mean,
                                 float* __restrict__ rstd, __nv_bfloat16* __restrict__ split) {
    const int row = blockIdx.x;
    const T* xr = x + size_t(row) * width;
    __shared__ float red[32];
    float s = 0.f;
    for (int c = threadIdx.x; c < width; c += blockDim.x) {
        const float v = ldf(xr + c);
        s += v;
        if (split) {
            const __nv_bfloat16 hi = __float2bfloat16_rn(v);
            split[size_t(row) * 2 * width + c] = hi;
            split[size_t(row) * 2 * width + width + c] = __float2bfloat16_rn(v - __bfloat162float(hi));
        }
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    float tot = 0.f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += red[w];
    const float mu = tot / float(width);
    __syncthreads();
    float v = 0.f;
    for (int c = threadIdx.x; c < width; c += blockDim.x) {
        const float dx = ldf(xr + c) - mu;
        v += dx * dx;
    }
    v = warp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        float var = 0.f;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) var += red[w];
        mean[row] = mu;
        rstd[row] = rsqrtf(var / float(width) + 1e-5f);
    }
}

// colsum[n] = sum_k W^T[n][k] (once per W).
__global__ void colsum_kernel(const __nv_bfloat16* __restrict__ wt, int width, int vocab,
                              float* __restrict__ colsum) {
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n >= vocab) return;
    float s = 0.f;
    for (int c = threadIdx.x & 31; c < width; c += 32) s += __bfloat162float(wt[size_t(n) * width + c]);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) colsum[n] = s;
}

struct ScoreArgs {
    int rows, width, vocab, a_passes;
    const float* mean;
    const float* rstd;
    const float* colsum;
    unsigned long long* best;  // [rows] packed (z, ~idx), zero-initialised
    float* logits;             // optional [rows][vocab]: rstd * z (= LN(x) @ W)
    unsigned long long* trace; // debug (EP_TRACE=1): per CTA [start, first stage, mma done, end] ns
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kScoreThreads, 1)
    score_argmax_kernel(const ScoreArgs sa, const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_w) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStagesS * kStage);
    uint64_t* empty = full + kStagesS;
    uint64_t* acc_full = empty + kStagesS;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kTM, n0 = blockIdx.y * kTN;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    if (sa.trace && threadIdx.x == 0) sa.trace[4 * cta] = gtimer();
    const int nkw = sa.width / kTK;         // k-blocks of W per pass
    const int nk = nkw * sa.a_passes;        // A is [hi | lo] when a_passes == 2

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStagesS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        fence_mbar_init();
    }
    if (warp == 5) umma::tmem_alloc(tmem_slot, 256);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == 4) {
        if (lane == 0) {
            umma::tma_prefetch_desc(&tmap_a);
            umma::tma_prefetch_desc(&tmap_w);
            const uint64_t pol = l2_policy_evict_last();  // W tiles are shared by the M tiles
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kStagesS;
                mbar_wait(&empty[s], ((kb / kStagesS) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kStage);
                uint8_t* dst = smem + s * kStage;
                umma::tma_load_2d(dst, &tmap_a, kb * kTK, m0, &full[s], pol);
                umma::tma_load_2d(dst + kABytes, &tmap_w, (kb % nkw) * kTK, n0, &full[s], pol);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t base = smem_u32(smem);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % kStagesS;
                mbar_wait(&full[s], (kb / kStagesS) & 1);
                if (kb == 0 && sa.trace) sa.trace[4 * cta + 1] = gtimer();
                umma::fence_after_sync();
                const uint32_t a_addr = base + s * kStage, b_addr = a_addr + kABytes;
#pragma unroll
                for (int kk = 0; kk < kTK / 16; ++kk) {
                    const uint64_t ad = umma::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
                    const uint64_t bd = umma::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                    umma::mma_bf16_ss(tmem, ad, bd, kIdescScore, (kb | kk) ? 1u : 0u);
                }
                umma::mma_commit(&empty[s]);
            }
            umma::mma_commit(acc_full);
        }
    } else {
        // epilogue: thread = row (TMEM lane), 256 vocab columns. The tile's
        // colsum slice and the row's mean are fetched while the MMAs run; TMEM
        // is read 64 columns per wait.
        const int row = warp * 32 + lane;
        const int grow = m0 + row;
        float* s_cs = reinterpret_cast<float*>(tmem_slot + 4);  // [kTN] colsum of this tile
        for (int i = threadIdx.x; i < kTN; i += 128) s_cs[i] = sa.colsum[n0 + i];
        const bool valid = grow < sa.rows;
        const float mu = valid ? sa.mean[grow] : 0.f;
        const float rs = valid ? sa.rstd[grow] : 0.f;
        named_bar_sync(1, 128);
        mbar_wait(acc_full, 0);
        if (sa.trace && threadIdx.x == 0) sa.trace[4 * cta + 2] = gtimer();
        umma::fence_after_sync();
        float best = -INFINITY;
        uint32_t best_i = 0;
#pragma unroll 1
        for (int c = 0; c < kTN / 32; c += 2) {
            uint32_t r[64];
            umma::tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c * 32, *reinterpret_cast<uint32_t(*)[32]>(r));
            umma::tmem_ld32(tmem + (uint32_t(warp * 32) << 16) + c * 32 + 32,
                            *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            umma::tmem_wait_ld();
            if (valid) {
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    const int nl = c * 32 + j;
                    const float z = fmaf(-mu, s_cs[nl], __uint_as_float(r[j]));
                    const bool up = z > best;  // strict: ties keep the lowest id
                    best = up ? z : best;
                    best_i = up ? uint32_t(n0 + nl) : best_i;
                    if (sa.logits) sa.logits[size_t(grow) * sa.vocab + n0 + nl] = z * rs;
                }
            }
        }
        if (valid) atomicMax(&sa.best[grow], order_key(best, best_i));
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 5) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, 256);
    }
    if (sa.trace && threadIdx.x == 0) sa.trace[4 * cta + 3] = gtimer();
}

// g_j from the packed keys; n = longest draft prefix reproduced by the target.
__global__ void accept_kernel(const unsigned long long* __restrict__ best, int batch, int n_q,
                              const int32_t* __restrict__ drafts, int32_t* __restrict__ target,
                              int32_t* __restrict__ n_accepted) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const int k = n_q - 1;
    int n = 0;
    bool run = true;
    for (int j = 0; j < n_q; ++j) {
        const int32_t g = int32_t(0xFFFFFFFFu - uint32_t(best[size_t(b) * n_q + j] & 0xFFFFFFFFull));
        target[size_t(b) * n_q + j] = g;
        if (j < k && run) {
            if (drafts[size_t(b) * k + j] == g)
                ++n;
            else
                run = false;
        }
    }
    n_accepted[b] = n;
}

}  // namespace

cudaError_t launch_colsum(const void* wt, int width, int vocab, float* colsum, cudaStream_t s) {
    colsum_kernel<<<(vocab + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(wt), width,
                                                  vocab, colsum);
    return cudaGetLastError();
}

cudaError_t launch_score_accept(int rows, int width, int vocab, const void* attn_out, void* split,
                                const CUtensorMap& tmap_a, const CUtensorMap& tmap_w,
                                const float* colsum, float* mean, float* rstd,
                                unsigned long long* best, float* logits, int batch, int n_q,
                                const int32_t* drafts, int32_t* target, int32_t* n_accepted,
                                cudaStream_t s) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(score_argmax_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, kScoreSmem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    if (split)
        row_stats_kernel<float><<<rows, 256, 0, s>>>(static_cast<const float*>(attn_out), width,
                                                     mean, rstd, static_cast<__nv_bfloat16*>(split));
    else
        row_stats_kernel<__nv_bfloat16><<<rows, 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(attn_out), width, mean, rstd, nullptr);
    cudaError_t e = cudaMemsetAsync(best, 0, sizeof(unsigned long long) * rows, s);
    if (e != cudaSuccess) return e;
    static unsigned long long* trace = [] {
        unsigned long long* b = nullptr;
        const char* e = std::getenv("EP_TRACE");
        if (e && e[0] == '1' && cudaMalloc(&b, 4096 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(b, 0, 4096 * sizeof(unsigned long long));
        return b;
    }();
    ScoreArgs sa{rows, width, vocab, split ? 2 : 1, mean, rstd, colsum, best, logits, trace};
    dim3 grid((rows + kTM - 1) / kTM, vocab / kTN);
    score_argmax_kernel<<<grid, kScoreThreads, kScoreSmem, s>>>(sa, tmap_a, tmap_w);
    if (trace) {  // debug: dump the per-CTA timeline of this launch
        std::vector<unsigned long long> host(4096);
        cudaStreamSynchronize(s);
        cudaMemcpy(host.data(), trace, host.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        const char* f = std::getenv("EP_TRACE_SCORE_FILE");
        if (FILE* fp = std::fopen(f ? f : "ep_trace_score.bin", "wb")) {
            std::fwrite(host.data(), sizeof(unsigned long long), host.size(), fp);
            std::fclose(fp);
        }
    }
    accept_kernel<<<(batch + 127) / 128, 128, 0, s>>>(best, batch, n_q, drafts, target, n_accepted);
    return cudaGetLastError();
}

}  // namespace ep
