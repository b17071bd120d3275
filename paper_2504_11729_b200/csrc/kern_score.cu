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
//   * score GEMM on tcgen05: Z[128 rows x 128 vocab] (TMEM fp32) over K = 4096
//     in 64-wide TMA-fed stages (A = attention rows, B = W^T, both bf16,
//     128B-swizzled K-major). LayerNorm is folded into the epilogue:
//     LN(x).w = rstd * (x.w - mean * colsum(w)); rstd > 0 does not move the
//     argmax, so the epilogue ranks z = x.w - mean * colsum(w) and reduces
//     (z, lowest index) across the vocab tiles with one 64-bit atomicMax per
//     row per CTA on an order-preserving key.
//   * fp32 attention rows (the verify default) are scored in two steps
//     rather than one bf16 hi+lo GEMM of twice the K: the GEMM runs on the
//     bf16 hi part of the centred row xc = x - mean (LN(x).w = rstd * xc.w
//     ranks like xc.w); since xc = hi + lo exactly, every logit satisfies
//     |z - z_hi| <= E_row = max_n ||w_n||_2 * (||lo||_2 + 2^-12 ||xc||_2)
//     (Cauchy-Schwarz on the lo term + the fp32 accumulation bound), so only
//     vocab entries within 2 E_row of the row's best z_hi can be its argmax.
//     The GEMM epilogue emits those candidates per tile; refine_kernel
//     computes their logits exactly (fp32 dot of the centred fp32 row with
//     the bf16 W row) and picks the first maximum — the ids of the
//     full-precision product at half the tensor work.
//   * accept: per request, decode g_j and apply the acceptance rule.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <vector>

#include "ep_common.cuh"
#include "ep_internal.h"
#include "umma.cuh"

namespace ep {
namespace {

// Tiles are kTM = 128 rows x tn vocabulary columns, tn chosen per launch so
// that one wave of CTAs (one per SM) covers the product: tn = 32-multiple
// of ceil(vocab / floor(SMs / M tiles)), <= 256 (config 3: 160 at k = 8, 96
// at k = 4). One CTA per SM with as deep a ring as shared memory allows.
constexpr int kTM = 128, kTNMax = kScoreTileNMax, kTK = 64;
constexpr int kStagesMax = 8;
constexpr int kABytes = kTM * kTK * 2;  // 16 KB
constexpr int kScoreThreads = 192;      // warps 0-3 epilogue, 4 TMA, 5 MMA
constexpr int kStash = 24;              // per-thread candidate stash of the epilogue (smem)
constexpr int kScoreSmemFixed = 1024 + 256 + kTNMax * 4 + kStash * 128 * 5;  // align, barriers, colsum slice, stash
constexpr int kScoreSmemBudget = 227 * 1024 - kScoreSmemFixed;
// stream-K kernel: 8 epilogue warps (two per TMEM lane quarter, each taking
// half of a tile's chunks), then the TMA and MMA warps
constexpr int kSkEpiThreads = 256;
constexpr int kSkThreads = kSkEpiThreads + 64;
constexpr int kSkWarpTma = kSkEpiThreads / 32, kSkWarpMma = kSkWarpTma + 1;
constexpr int kSkSmemFixed = 1024 + 256 + kTNMax * 4 + kStash * kSkEpiThreads * 5;

__host__ __device__ inline int score_stage_bytes(int tn) { return kABytes + tn * kTK * 2; }
__host__ __device__ inline int score_stages(int tn) {
    const int s = kScoreSmemBudget / score_stage_bytes(tn);
    return s < kStagesMax ? s : kStagesMax;
}

__device__ __forceinline__ uint64_t order_key(float z, uint32_t idx) {
    // argmax_token compares with '>': -0 == +0 (canonicalised so the lower
    // id wins the tie), and a NaN is never taken over a number — except at
    // id 0, where the scan starts and nothing compares greater than it
    if (z != z) return idx == 0 ? ~0ull : 0ull;
    uint32_t b = __float_as_uint(z == 0.f ? 0.f : z);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (uint64_t(b) << 32) | uint64_t(0xFFFFFFFFu - idx);
}

template <typename T>
__device__ __forceinline__ float ldf(const T* p);
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
                                 float* __restrict__ rstd, __nv_bfloat16* __restrict__ split,
                                 unsigned long long* __restrict__ best_key) {
    const int row = blockIdx.x;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the attention output is complete
    if (threadIdx.x == 0) best_key[row] = 0ull;
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

// fp32 rows: mean, 1/sqrt(var + 1e-5) (two-pass, from registers), the bf16 hi
// part (the GEMM's A operand) and the refinement bound E_row. 128 threads per
// row, 8 float4 per thread (width <= 4096).
constexpr int kStatThreads = 128;
constexpr int kStatVec = 8;
__global__ void __launch_bounds__(kStatThreads)
    row_stats_split_kernel(const float* __restrict__ x, int width, float* __restrict__ mean,
                           float* __restrict__ rstd, __nv_bfloat16* __restrict__ hi_out,
                           const float* __restrict__ wmax2, float* __restrict__ ebound,
                           const uint8_t* __restrict__ w_bytes, size_t w_size,
                           unsigned long long* __restrict__ best_key) {
    const int row = blockIdx.x, tid = threadIdx.x;
    const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * width);
    const int nv = width / 4;
    // W_score is constant: bring this CTA's slice of it into L2 before
    // waiting for the attention (programmatic dependent launch lets this
    // overlap the attention's tail), so the GEMM's W tiles are L2 hits
    // instead of first-touch DRAM reads on the critical path
    if (w_bytes && tid < 4) {
        const size_t per = ((w_size + gridDim.x - 1) / gridDim.x + 63) & ~size_t(63);
        const size_t b0 = size_t(row) * per;
        for (size_t off = b0 + size_t(tid) * 16384; off < b0 + per && off < w_size; off += 4 * 16384) {
            const size_t n = min(min(size_t(16384), b0 + per - off), w_size - off);
            bulk_prefetch_l2(w_bytes + off, uint32_t(n) & ~15u);
        }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the attention output is complete
    __shared__ float red[3][kStatThreads / 32];
    float4 v[kStatVec];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < kStatVec; ++i) {
        const int c = tid + i * kStatThreads;
        v[i] = c < nv ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
        s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) red[0][tid >> 5] = s;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < kStatThreads / 32; ++w) tot += red[0][w];
    const float mu = tot / float(width);
    // the centred row xc = x - mean is what gets scored: LN(x).w = rstd *
    // xc.w ranks like xc.w, and the hi / lo split of xc (not of x) keeps the
    // refinement bound proportional to the logit spread
    float q = 0.f, lo2 = 0.f;
    uint2* ho = reinterpret_cast<uint2*>(hi_out + size_t(row) * width);
#pragma unroll
    for (int i = 0; i < kStatVec; ++i) {
        const int c = tid + i * kStatThreads;
        if (c < nv) {
            const float e[4] = {v[i].x - mu, v[i].y - mu, v[i].z - mu, v[i].w - mu};
            uint32_t hp[2];
#pragma unroll
            for (int k = 0; k < 4; k += 2) {
                const __nv_bfloat162 h = __floats2bfloat162_rn(e[k], e[k + 1]);
                hp[k / 2] = *reinterpret_cast<const uint32_t*>(&h);
                const float2 hf = __bfloat1622float2(h);
                const float l0 = e[k] - hf.x, l1 = e[k + 1] - hf.y;  // exact
                lo2 += l0 * l0 + l1 * l1;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) q += e[k] * e[k];
            ho[c] = make_uint2(hp[0], hp[1]);
        }
    }
    float x2 = q;
    q = warp_sum(q);
    lo2 = warp_sum(lo2);
    x2 = warp_sum(x2);
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = q;
        red[1][tid >> 5] = lo2;
        red[2][tid >> 5] = x2;
    }
    __syncthreads();
    if (tid == 0) {
        best_key[row] = 0ull;  // the GEMM's argmax key of this row starts empty
        float tq = 0.f, tl = 0.f, tx = 0.f;
#pragma unroll
        for (int w = 0; w < kStatThreads / 32; ++w) {
            tq += red[0][w];
            tl += red[1][w];
            tx += red[2][w];
        }
        mean[row] = mu;
        rstd[row] = rsqrtf(tq / float(width) + 1e-5f);
        // |xc.w - hi.w| <= ||lo|| ||w||; fp32 accumulation of hi.w <= 2^-12 ||xc|| ||w||
        // (<= 4096 terms); 1 % slack for the rounding of the bound itself
        ebound[row] = 1.01f * (*wmax2) * (sqrtf(tl) + 0x1.0p-12f * sqrtf(tx));
    }
}

// max_n ||W^T[n]||_2 (once per W), as float bits (non-negative: integer order).
__global__ void colnorm_max_kernel(const __nv_bfloat16* __restrict__ wt, int width, int vocab,
                                   float* __restrict__ wmax2) {
    const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (n >= vocab) return;
    float s = 0.f;
    for (int c = threadIdx.x & 31; c < width; c += 32) {
        const float w = __bfloat162float(wt[size_t(n) * width + c]);
        s += w * w;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0)
        atomicMax(reinterpret_cast<unsigned int*>(wmax2), __float_as_uint(sqrtf(s) * 1.0001f));
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

constexpr int kPerTile = kScoreCandPerTile;  // candidates kept per (row, vocab tile) (overflow -> every n exactly)

struct ScoreArgs {
    int rows, width, vocab, a_passes;
    const float* mean;
    const float* rstd;
    const float* colsum;
    unsigned long long* best;  // [rows] packed (z, ~idx), zero-initialised
    float* logits;             // optional [rows][vocab]: rstd * z (= LN(x) @ W)
    unsigned long long* trace; // debug (EP_TRACE=1): per CTA [start, first stage, mma done, end] ns
    // hi-only pass (fp32 rows): per-(row, vocab tile) candidates for refine_kernel
    const float* ebound;       // [rows] |z - z_hi| bound
    int32_t* cand_cnt;         // [rows][n_tiles]
    int32_t* cand_n;           // [rows][n_tiles][kPerTile]
    float* cand_z;             // [rows][n_tiles][kPerTile]
    int n_tiles;
    int tn, stages;            // tile width (vocab columns, multiple of 32) and ring depth
    uint32_t idesc;            // M = 128, N = tn
    // stream-K (score_argmax_streamk_kernel): tiles_m x n_tiles tiles of nkt
    // k-blocks, flattened M-fastest and cut into gridDim.x equal ranges
    int tiles_m = 0, nkt = 0, n_vt = 0;  // (n_tiles counts the 128-column candidate tiles)
    float* sk_ws = nullptr;          // [ctas][kTNMax / 32][8][128] float4 partial tiles
    unsigned int* sk_flags = nullptr;  // [ctas] partial published (1) / consumed (0)
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Scan of one finished score tile by the 4 epilogue warps, thread =
// accumulator row (TMEM lane) of the 128 rows [m0, m0 + 128), TN vocab
// columns from n0 (vocab tile `ntile`): LN fold, tile argmax (64-bit key
// atomicMax per row) and, on the hi-only pass, the refinement candidates of
// the tile. The tile's colsum slice is in s_cs. Stream-K owners add the
// fp32 partial tiles of CTAs [cp0, cp0 + n_part) (ws: [cta][chunk][4-float group][row])
// to each accumulator chunk before scoring it.
//
// Chunks [c_lo, c_hi) of the tile are scanned by this warp (the stream-K
// kernel splits a tile's 8 chunks over two warps per TMEM lane quarter);
// their candidates go to candidate tile `ntile` (columns [n0 + 32 c_lo,
// n0 + 32 c_hi)); nthr = epilogue threads (the stash stride).
__device__ __forceinline__ void score_scan(const ScoreArgs& sa, uint32_t tmem, const float* s_cs, int m0, int n0,
                                           int ntile, int TN, int c_lo, int c_hi, int nthr,
                                           const float* __restrict__ ws, int cp0, int n_part,
                                           const float4* spart, uint64_t* pbar, unsigned long long* tr) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int row = (warp & 3) * 32 + lane;
    const int grow = m0 + row;
    const int ncols = min(TN, sa.vocab - n0);
    const bool valid = grow < sa.rows;
    // (rows already centred for the hi-only pass: no mean * colsum term)
    const float mu = valid && !sa.cand_n ? sa.mean[grow] : 0.f;
    const float rs = valid ? sa.rstd[grow] : 0.f;
    float best = -INFINITY;
    uint32_t best_i = 0;
    // hi-only pass: every n of the tile that can still be the row's
    // argmax has z_hi >= tile max - 2 E_row (the row max is >= the tile
    // max). One TMEM pass: after each 32-column chunk, the chunk's values
    // within 2 E_row of the running max go to a per-thread smem stash (a
    // superset: the max only grows), filtered by the final max at the end.
    const bool emit = sa.cand_n != nullptr;
    const float eb2 = emit && valid ? 2.f * sa.ebound[grow] : 0.f;
    float* st_z = const_cast<float*>(s_cs) + kTNMax;                    // [kStash][nthr]
    uint8_t* st_n = reinterpret_cast<uint8_t*>(st_z + kStash * nthr);   // [kStash][nthr]
    const int me = threadIdx.x;
    int n_st = 0;
    const uint32_t trow = tmem + (uint32_t((warp & 3) * 32) << 16);
    // bf16 rows: LN(x).w = rstd (x.w - mean colsum(w)); warp-uniform, so the
    // hi-only pass (rows centred already) carries no colsum loads
    const bool fold = !emit;
    float* logits_row = sa.logits ? sa.logits + size_t(grow) * sa.vocab + n0 : nullptr;
    // one 32-column TMEM load per chunk, the chunk loop kept rolled: the
    // scan is straight-line code executed once per warp, and an unrolled
    // 8-chunk body (~40 KB of SASS) ran at instruction-fetch speed
    // stream-K partials: chunk c + 1 of the first partial is loaded while
    // chunk c is scored (the loads are L2 round trips; 4 warps alone cannot
    // hide them one chunk at a time)
    // (ws layout [cta][chunk][j4][row] float4: one load instruction of a
    // warp reads 512 contiguous bytes)
    auto part_ptr = [&](int q, int c) {
        return reinterpret_cast<const float4*>(ws) + (size_t(cp0 + q) * (kTNMax / 32) + c) * 8 * 128 + row;
    };
    // (spart: the first partial already on its way into shared memory, one
    // bulk copy per chunk completing on pbar[chunk])
    float4 pre[8];
    if (n_part > 0 && !spart) {
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) pre[j4] = __ldcg(part_ptr(0, c_lo) + j4 * 128);
    }
#pragma unroll 1
    for (int c = c_lo; c < c_hi; ++c) {
        uint32_t buf[32];
        umma::tmem_ld32(trow + c * 32, buf);
        umma::tmem_wait_ld();
        if (c == c_lo && tr) tr[6] = gtimer();
        if (spart) {
            const unsigned long long w0 = tr ? gtimer() : 0ull;
            mbar_wait(&pbar[c], 0);
            if (tr) tr[7] += gtimer() - w0;
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
                const float4 v = spart[(c * 8 + j4) * 128 + row];
                buf[4 * j4 + 0] = __float_as_uint(__uint_as_float(buf[4 * j4 + 0]) + v.x);
                buf[4 * j4 + 1] = __float_as_uint(__uint_as_float(buf[4 * j4 + 1]) + v.y);
                buf[4 * j4 + 2] = __float_as_uint(__uint_as_float(buf[4 * j4 + 2]) + v.z);
                buf[4 * j4 + 3] = __float_as_uint(__uint_as_float(buf[4 * j4 + 3]) + v.w);
            }
        } else if (n_part > 0) {
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
                const float4 v = pre[j4];
                buf[4 * j4 + 0] = __float_as_uint(__uint_as_float(buf[4 * j4 + 0]) + v.x);
                buf[4 * j4 + 1] = __float_as_uint(__uint_as_float(buf[4 * j4 + 1]) + v.y);
                buf[4 * j4 + 2] = __float_as_uint(__uint_as_float(buf[4 * j4 + 2]) + v.z);
                buf[4 * j4 + 3] = __float_as_uint(__uint_as_float(buf[4 * j4 + 3]) + v.w);
            }
            if (c + 1 < c_hi) {
#pragma unroll
                for (int j4 = 0; j4 < 8; ++j4) pre[j4] = __ldcg(part_ptr(0, c + 1) + j4 * 128);
            }
        }
#pragma unroll 1
        for (int q = 1; q < n_part; ++q) {
            const float4* pp = part_ptr(q, c);
#pragma unroll
            for (int j4 = 0; j4 < 8; ++j4) {
                const float4 v = __ldcg(pp + j4 * 128);
                buf[4 * j4 + 0] = __float_as_uint(__uint_as_float(buf[4 * j4 + 0]) + v.x);
                buf[4 * j4 + 1] = __float_as_uint(__uint_as_float(buf[4 * j4 + 1]) + v.y);
                buf[4 * j4 + 2] = __float_as_uint(__uint_as_float(buf[4 * j4 + 2]) + v.z);
                buf[4 * j4 + 3] = __float_as_uint(__uint_as_float(buf[4 * j4 + 3]) + v.w);
            }
        }
        // warp-uniform (rows past the last valid one score -inf)
        const int nlim = valid ? ncols - c * 32 : 0;  // valid columns of this chunk
        float z[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            float v = __uint_as_float(buf[j]);
            if (fold) v = fmaf(-mu, s_cs[c * 32 + j], v);
            z[j] = j < nlim ? v : -INFINITY;
        }
        // chunk maximum by a tree (fmaxf drops NaN, as '>' never takes
        // one), then the first column reaching it: the same result as the
        // sequential strict '>' scan, without its 32-long dependency chain
        float m[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) m[j] = fmaxf(z[j], z[j + 16]);
#pragma unroll
        for (int w = 8; w > 0; w >>= 1)
#pragma unroll
            for (int j = 0; j < w; ++j) m[j] = fmaxf(m[j], m[j + w]);
        if (m[0] > best) {  // strict: ties keep the lowest id
            uint32_t eq = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) eq |= (z[j] == m[0] ? 1u : 0u) << j;
            best = m[0];
            best_i = uint32_t(n0 + c * 32 + __ffs(eq) - 1);
        }
        if (logits_row && valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if (j < nlim) logits_row[c * 32 + j] = z[j] * rs;
        }
        if (emit) {
            // candidates (rare after the first chunks): a bit mask of the
            // columns within 2 E_row of the running max, built only when
            // the chunk maximum itself is within it for some lane of the warp
            const float thr = best - eb2;
            if (__any_sync(0xffffffffu, valid && m[0] >= thr)) {
                uint32_t pass = 0;
#pragma unroll
                for (int j = 0; j < 32; ++j) pass |= (valid && z[j] >= thr ? 1u : 0u) << j;
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    if (pass & (1u << j)) {
                        if (n_st < kStash) {
                            st_z[n_st * nthr + me] = z[j];
                            st_n[n_st * nthr + me] = uint8_t(c * 32 + j);
                        }
                        ++n_st;
                    }
                }
            }
        }
    }
    if (tr) tr[3] = gtimer();
    if (valid) atomicMax(&sa.best[grow], order_key(best, best_i));
    if (emit && valid) {
        const float thr = best - eb2;
        const size_t slot0 = (size_t(grow) * sa.n_tiles + ntile) * kPerTile;
        int cnt = 0;
        if (n_st > kStash) {
            cnt = kPerTile + 1;  // stash overflow: refine scores the whole row
        } else {
            for (int i = 0; i < n_st; ++i) {
                const float z = st_z[i * nthr + me];
                if (z >= thr) {
                    if (cnt < kPerTile) {
                        sa.cand_n[slot0 + cnt] = n0 + st_n[i * nthr + me];
                        sa.cand_z[slot0 + cnt] = z;
                    }
                    ++cnt;
                }
            }
        }
        sa.cand_cnt[size_t(grow) * sa.n_tiles + ntile] = cnt;
    }
    if (tr) tr[4] = gtimer();
}

// Epilogue of the one-tile-per-CTA kernels: colsum slice fetched while the
// MMAs run (columns past the vocabulary — a partial last tile, TMA
// zero-filled — are skipped by the scan), then the scan of the accumulator.
__device__ __forceinline__ void score_epilogue(const ScoreArgs& sa, uint32_t tmem, uint64_t* acc_full,
                                               uint32_t* tmem_slot, int m0, int n0, int TN,
                                               unsigned long long* tr) {
    float* s_cs = reinterpret_cast<float*>(tmem_slot + 4);  // [kTNMax] colsum of this tile
    const int ncols = min(TN, sa.vocab - n0);
    for (int i = threadIdx.x; i < ncols; i += 128) s_cs[i] = sa.colsum[n0 + i];
    named_bar_sync(1, 128);
    mbar_wait(acc_full, 0);
    if (tr) tr[2] = gtimer();
    umma::fence_after_sync();
    score_scan(sa, tmem, s_cs, m0, n0, blockIdx.y, TN, 0, TN / 32, 128, nullptr, 0, 0, nullptr, nullptr, tr);
}

__global__ void __launch_bounds__(kScoreThreads, 1)
    score_argmax_kernel(const ScoreArgs sa, const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_w) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    // 1 KB aligned base (SW128 atoms) derived from the __shared__ array by an
    // offset, so every pointer below stays in the shared window (LDS / STS,
    // not generic loads: the generic form made the epilogue scan 8.6 us)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int TN = sa.tn, NS = sa.stages, kStage = score_stage_bytes(TN);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kStage);
    uint64_t* empty = full + kStagesMax;
    uint64_t* acc_full = empty + kStagesMax;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kTM, n0 = blockIdx.y * TN;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    // debug (EP_TRACE=1): per CTA [start, first stage, MMAs done, scan done, candidates done, end, first TMEM load] ns
    unsigned long long* trc = sa.trace && cta < 512 ? sa.trace + 8 * cta : nullptr;
    unsigned long long* tr = threadIdx.x == 0 ? trc : nullptr;
    if (tr) tr[0] = gtimer();
    const int nkw = sa.width / kTK;         // k-blocks of W per pass
    const int nk = nkw * sa.a_passes;        // A is [hi | lo] when a_passes == 2

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        fence_mbar_init();
    }
    if (warp == 5) umma::tmem_alloc(tmem_slot, kTNMax);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // A (row stats output) is complete

    if (warp == 4) {
        if (lane == 0) {
            umma::tma_prefetch_desc(&tmap_a);
            umma::tma_prefetch_desc(&tmap_w);
            const uint64_t pol = l2_policy_evict_last();  // W tiles are shared by the M tiles
            const uint32_t wbytes = uint32_t(TN) * kTK * 2;
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % NS;
                mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kABytes + wbytes);
                uint8_t* dst = smem + s * kStage;
                umma::tma_load_2d(dst, &tmap_a, kb * kTK, m0, &full[s], pol);
                umma::tma_load_2d(dst + kABytes, &tmap_w, (kb % nkw) * kTK, n0, &full[s], pol);
            }
        }
    } else if (warp == 5) {
        if (lane == 0) {
            const uint32_t base = smem_u32(smem);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % NS;
                mbar_wait(&full[s], (kb / NS) & 1);
                if (kb == 0 && trc) trc[1] = gtimer();
                umma::fence_after_sync();
                const uint32_t a_addr = base + s * kStage, b_addr = a_addr + kABytes;
#pragma unroll
                for (int kk = 0; kk < kTK / 16; ++kk) {
                    const uint64_t ad = umma::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
                    const uint64_t bd = umma::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                    umma::mma_bf16_ss(tmem, ad, bd, sa.idesc, (kb | kk) ? 1u : 0u);
                }
                umma::mma_commit(&empty[s]);
            }
            umma::mma_commit(acc_full);
        }
    } else {
        score_epilogue(sa, tmem, acc_full, tmem_slot, m0, n0, TN, tr);
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 5) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, kTNMax);
    }
    if (tr) tr[5] = gtimer();
}

// The same GEMM on CTA pairs (cta_group::2): a cluster of two CTAs on one TPC
// computes a 256-row x tn tile with M = 256 MMAs issued by the even CTA. Each
// CTA streams its 128 rows of A and half of the tile's W rows (tn / 2) into
// the same shared-memory offsets; the tensor cores read A from each CTA and B
// from both, so the shared-memory bytes per FLOP halve against the 1-SM form
// (whose mainloop is shared-memory-bandwidth bound: operand reads + TMA writes
// of ~230 B/clk per SM against the 128 B/clk port). Stage fills complete on
// the even CTA's mbarriers; each MMA commit frees the stage in both CTAs.
__global__ void __launch_bounds__(kScoreThreads, 1)
    score_argmax_pair_kernel(const ScoreArgs sa, const __grid_constant__ CUtensorMap tmap_a,
                             const __grid_constant__ CUtensorMap tmap_w) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int TN = sa.tn, NS = sa.stages, kStage = kABytes + (TN / 2) * kTK * 2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kStage);
    uint64_t* empty = full + kStagesMax;
    uint64_t* acc_full = empty + kStagesMax;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = umma::cluster_ctarank();
    const int m0 = (blockIdx.x >> 1) * (2 * kTM) + int(rank) * kTM, n0 = blockIdx.y * TN;
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    unsigned long long* trc = sa.trace && cta < 512 ? sa.trace + 8 * cta : nullptr;
    unsigned long long* tr = threadIdx.x == 0 ? trc : nullptr;
    if (tr) tr[0] = gtimer();
    const int nkw = sa.width / kTK;
    const int nk = nkw * sa.a_passes;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc_full, 1);
        fence_mbar_init();
    }
    if (warp == 5) umma::tmem_alloc_pair(tmem_slot, kTNMax);
    umma::fence_before_sync();
    umma::cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
    umma::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // A (row stats output) is complete

    if (warp == 4) {
        if (lane == 0) {
            umma::tma_prefetch_desc(&tmap_a);
            umma::tma_prefetch_desc(&tmap_w);
            const uint64_t pol = l2_policy_evict_last();
            const int nb = n0 + int(rank) * (TN / 2);  // this CTA's half of the tile's W rows
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % NS;
                mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
                if (rank == 0) mbar_arrive_expect_tx(&full[s], 2u * uint32_t(kStage));
                const uint32_t bar0 = umma::mapa_shared(&full[s], 0);
                uint8_t* dst = smem + s * kStage;
                umma::tma_load_2d_pair(dst, &tmap_a, kb * kTK, m0, bar0, pol);
                umma::tma_load_2d_pair(dst + kABytes, &tmap_w, (kb % nkw) * kTK, nb, bar0, pol);
            }
        }
    } else if (warp == 5) {
        if (lane == 0 && rank == 0) {
            const uint32_t base = smem_u32(smem);
            for (int kb = 0; kb < nk; ++kb) {
                const int s = kb % NS;
                mbar_wait(&full[s], (kb / NS) & 1);
                if (kb == 0 && trc) trc[1] = gtimer();
                umma::fence_after_sync();
                const uint32_t a_addr = base + s * kStage, b_addr = a_addr + kABytes;
#pragma unroll
                for (int kk = 0; kk < kTK / 16; ++kk) {
                    const uint64_t ad = umma::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
                    const uint64_t bd = umma::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                    umma::mma_bf16_ss_pair(tmem, ad, bd, sa.idesc, (kb | kk) ? 1u : 0u);
                }
                umma::mma_commit_pair(&empty[s], 0x3);
            }
            umma::mma_commit_pair(acc_full, 0x3);
        }
    } else {
        score_epilogue(sa, tmem, acc_full, tmem_slot, m0, n0, TN, tr);
    }
    umma::fence_before_sync();
    umma::cluster_sync();  // no CTA leaves while its peer may still signal or read it
    if (warp == 5) {
        umma::fence_after_sync();
        umma::tmem_dealloc_pair(tmem, kTNMax);
    }
    if (tr) tr[5] = gtimer();
}

// Stream-K form of the score GEMM. A tcgen05 MMA costs ~176 SM cycles
// whatever its N (32 ... 256) or M (64 / 128) when it accumulates into the
// same TMEM tile as the previous one (tools/gemm_probe.cu, measured), so a
// tile's K loop is a chain of K / 16 such steps and only the number of
// chained steps per SM sets the GEMM time: tiles are 128 x 256 (the most
// work per step) and the flattened (tile, k-block) space is cut into
// gridDim.x (= SMs) equal ranges, ~35 k-blocks per CTA at config 3 k = 8
// instead of 64 per one-tile CTA. A range covers the tail of one tile and /
// or the head of the next: the CTA holding a tile's last k-block owns it
// (scores it); a CTA whose range ends inside a tile publishes that fp32
// partial tile to its own workspace slot and raises its flag, and it does
// that segment first so the owner rarely waits. TMEM holds two 256-column
// accumulators so a segment's epilogue overlaps the next segment's MMAs.
// The epilogue is 8 warps (two per TMEM lane quarter, 4 chunks each: the
// scan is latency-bound per warp) and its candidates are kept per 128-column
// half tile.
__device__ __forceinline__ long long sk_begin(int c, int G, long long total) { return total * c / G; }
__device__ __forceinline__ int sk_cta_of(long long x, int G, long long total) {
    int c = int(x * G / total);
    while (c + 1 < G && sk_begin(c + 1, G, total) <= x) ++c;
    while (c > 0 && sk_begin(c, G, total) > x) --c;
    return c;
}
struct SkSeg {
    int tile, k0, k1;
    bool owner;
};
// Segment p (processing order) of CTA c: the trailing partial segment, if
// any, first, then the rest in k order.
__device__ __forceinline__ SkSeg sk_segment(int p, long long b, long long e, int nkt) {
    const long long t0 = b / nkt;
    const int nseg = int((e - 1) / nkt - t0 + 1);
    const bool tail_first = nseg > 1 && (e - ((e - 1) / nkt) * nkt) < nkt;
    const int j = tail_first ? (p == 0 ? nseg - 1 : p - 1) : p;
    SkSeg sg;
    sg.tile = int(t0) + j;
    const long long ts = (long long)sg.tile * nkt;
    sg.k0 = j == 0 ? int(b - ts) : 0;
    sg.k1 = int(min((long long)nkt, e - ts));
    sg.owner = sg.k1 == nkt;
    return sg;
}
__device__ __forceinline__ int sk_num_segments(long long b, long long e, int nkt) {
    return b >= e ? 0 : int((e - 1) / nkt - b / nkt + 1);
}

__global__ void __launch_bounds__(kSkThreads, 1)
    score_argmax_streamk_kernel(const ScoreArgs sa, const __grid_constant__ CUtensorMap tmap_a,
                                const __grid_constant__ CUtensorMap tmap_w) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int TN = kTNMax;
    const int NS = sa.stages, kStage = score_stage_bytes(TN);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kStage);
    uint64_t* empty = full + kStagesMax;
    uint64_t* acc_full = empty + kStagesMax;  // [2]
    uint64_t* acc_empty = acc_full + 2;       // [2]
    uint64_t* pbar = acc_empty + 2;           // [kTNMax / 32] staged partial chunks
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pbar + kTNMax / 32);
    float* s_cs = reinterpret_cast<float*>(tmem_slot + 4);  // [kTNMax] colsum of the tile being scored

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int G = gridDim.x, c = blockIdx.x;
    const long long total = (long long)sa.tiles_m * sa.n_vt * sa.nkt;
    const long long b = sk_begin(c, G, total), e = sk_begin(c + 1, G, total);
    const int nseg = sk_num_segments(b, e, sa.nkt);
    unsigned long long* trc = sa.trace && c < 512 ? sa.trace + 8 * c : nullptr;
    unsigned long long* tr = threadIdx.x == 0 ? trc : nullptr;
    if (tr) {
        tr[0] = gtimer();
        tr[7] = 0ull;
    }
    const int nkw = sa.width / kTK;  // k-blocks of W per pass

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], kSkEpiThreads);
        }
        for (int i = 0; i < kTNMax / 32; ++i) mbar_init(&pbar[i], 1);
        fence_mbar_init();
    }
    if (warp == kSkWarpMma) umma::tmem_alloc(tmem_slot, 2 * TN);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *tmem_slot;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // A (row stats output) is complete

    if (warp == kSkWarpTma) {
        if (lane == 0) {
            umma::tma_prefetch_desc(&tmap_a);
            umma::tma_prefetch_desc(&tmap_w);
            const uint64_t pol = l2_policy_evict_last();
            const uint32_t bytes = uint32_t(kStage);
            int kc = 0;
            for (int p = 0; p < nseg; ++p) {
                const SkSeg sg = sk_segment(p, b, e, sa.nkt);
                const int m0 = (sg.tile % sa.tiles_m) * kTM, n0 = (sg.tile / sa.tiles_m) * TN;
                for (int k = sg.k0; k < sg.k1; ++k, ++kc) {
                    const int s = kc % NS;
                    mbar_wait(&empty[s], ((kc / NS) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], bytes);
                    uint8_t* dst = smem + s * kStage;
                    umma::tma_load_2d(dst, &tmap_a, k * kTK, m0, &full[s], pol);
                    umma::tma_load_2d(dst + kABytes, &tmap_w, (k % nkw) * kTK, n0, &full[s], pol);
                }
            }
        }
    } else if (warp == kSkWarpMma) {
        if (lane == 0) {
            const uint32_t base = smem_u32(smem);
            int kc = 0;
            for (int p = 0; p < nseg; ++p) {
                const SkSeg sg = sk_segment(p, b, e, sa.nkt);
                const int slot = p & 1;
                if (p >= 2) mbar_wait(&acc_empty[slot], ((p >> 1) - 1) & 1);  // scanned / published
                umma::fence_after_sync();
                const uint32_t d = tmem + uint32_t(slot * TN);
                for (int k = sg.k0; k < sg.k1; ++k, ++kc) {
                    const int s = kc % NS;
                    mbar_wait(&full[s], (kc / NS) & 1);
                    if (kc == 0 && trc) trc[1] = gtimer();
                    umma::fence_after_sync();
                    const uint32_t a_addr = base + s * kStage, b_addr = a_addr + kABytes;
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk) {
                        const uint64_t ad = umma::smem_desc_sw128(a_addr + kk * 32, 16, 1024);
                        const uint64_t bd = umma::smem_desc_sw128(b_addr + kk * 32, 16, 1024);
                        umma::mma_bf16_ss(d, ad, bd, sa.idesc, (k > sg.k0 || kk) ? 1u : 0u);
                    }
                    umma::mma_commit(&empty[s]);
                }
                umma::mma_commit(&acc_full[slot]);
            }
        }
    } else {
        const int row = (warp & 3) * 32 + lane;
        const uint32_t trow = uint32_t((warp & 3) * 32) << 16;
        const int half = warp >> 2;  // this warp's chunks: [4 half, 4 half + 4)
        constexpr int kHalfCh = TN / 64;
        for (int p = 0; p < nseg; ++p) {
            const SkSeg sg = sk_segment(p, b, e, sa.nkt);
            const int slot = p & 1;
            const int m0 = (sg.tile % sa.tiles_m) * kTM, n0 = (sg.tile / sa.tiles_m) * TN;
            const uint32_t acc = tmem + uint32_t(slot * TN);
            if (sg.owner) {
                // the other CTAs covering this tile: [cp0, c), each with its
                // trailing partial segment on this tile. An owner only waits
                // for lower-indexed CTAs, which the hardware dispatches first,
                // so the spin cannot wait on a CTA that is not resident (the
                // grid is at most one CTA per SM).
                const int cp0 = sg.k0 > 0 ? sk_cta_of((long long)sg.tile * sa.nkt, G, total) : c;
                named_bar_sync(1, kSkEpiThreads);  // the previous scan is done with s_cs
                const int ncols = min(TN, sa.vocab - n0);
                for (int i = threadIdx.x; i < ncols; i += kSkEpiThreads) s_cs[i] = sa.colsum[n0 + i];
                if (threadIdx.x == 0)
                    for (int q = cp0; q < c; ++q)
                        while (ld_acquire_gpu(&sa.sk_flags[q]) == 0u) {
                        }
                named_bar_sync(1, kSkEpiThreads);
                mbar_wait(&acc_full[slot], (p >> 1) & 1);
                if (tr && p == nseg - 1) tr[2] = gtimer();
                umma::fence_after_sync();
                // the CTA's last segment: the MMAs are done with the operand
                // ring, so the first partial tile streams into it by bulk
                // copies (one per 32-column chunk) while the scan starts
                const bool staged = c > cp0 && p == nseg - 1;
                if (staged && threadIdx.x == 0) {
                    asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired partial -> async proxy
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(sa.sk_ws) +
                                         size_t(cp0) * (TN / 32) * 8 * 128 * sizeof(float4);
                    for (int ch = 0; ch < TN / 32; ++ch) {
                        mbar_arrive_expect_tx(&pbar[ch], 8 * 128 * sizeof(float4));
                        bulk_g2s(smem + ch * 8 * 128 * sizeof(float4), src + ch * 8 * 128 * sizeof(float4),
                                 8 * 128 * sizeof(float4), &pbar[ch]);
                    }
                }
                score_scan(sa, acc, s_cs, m0, n0, (sg.tile / sa.tiles_m) * 2 + half, TN, half * kHalfCh,
                           half * kHalfCh + kHalfCh, kSkEpiThreads, sa.sk_ws, cp0, c - cp0,
                           staged ? reinterpret_cast<const float4*>(smem) : nullptr, pbar,
                           p == nseg - 1 ? tr : nullptr);
                named_bar_sync(1, kSkEpiThreads);
                if (threadIdx.x == 0)
                    for (int q = cp0; q < c; ++q) sa.sk_flags[q] = 0u;  // consumed: clear for the next launch
            } else {
                // publish the partial tile: [chunk][j4][row] float4, so each
                // store instruction of a warp writes 512 contiguous bytes
                mbar_wait(&acc_full[slot], (p >> 1) & 1);
                umma::fence_after_sync();
                float4* dst = reinterpret_cast<float4*>(sa.sk_ws) + size_t(c) * (TN / 32) * 8 * 128 + row;
#pragma unroll 1
                for (int ch = half * kHalfCh; ch < half * kHalfCh + kHalfCh; ++ch) {
                    uint32_t r[32];
                    umma::tmem_ld32(acc + trow + ch * 32, r);
                    umma::tmem_wait_ld();
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4)
                        __stcg(dst + (size_t(ch) * 8 + j4) * 128,
                               make_float4(__uint_as_float(r[4 * j4]), __uint_as_float(r[4 * j4 + 1]),
                                           __uint_as_float(r[4 * j4 + 2]), __uint_as_float(r[4 * j4 + 3])));
                }
                __threadfence();
                named_bar_sync(1, kSkEpiThreads);
                if (threadIdx.x == 0) st_release_gpu(&sa.sk_flags[c], 1u);
            }
            umma::fence_before_sync();
            mbar_arrive(&acc_empty[slot]);
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == kSkWarpMma) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, 2 * TN);
    }
    if (tr) tr[5] = gtimer();
}

__device__ __forceinline__ float key_value(unsigned long long k) {
    uint32_t b = uint32_t(k >> 32);
    b = (b & 0x80000000u) ? (b & 0x7FFFFFFFu) : ~b;
    return __uint_as_float(b);
}

constexpr int kRefineThreads = 256;
constexpr int kMaxList = 1024;  // candidate list of one row (n_tiles * kPerTile)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// The acceptance rule of request b from the packed argmax keys of its rows.
__device__ __forceinline__ void accept_request(const unsigned long long* best, int b, int n_q,
                                               const int32_t* drafts, int32_t* target, int32_t* n_accepted) {
    const int k = n_q - 1;
    int n = 0;
    bool run = true;
    for (int j = 0; j < n_q; ++j) {
        const int32_t g = int32_t(0xFFFFFFFFu - uint32_t(__ldcg(&best[size_t(b) * n_q + j]) & 0xFFFFFFFFull));
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

// Per row: of the candidates the GEMM epilogue kept, those with z_hi >= row
// max z_hi - 2 E_row get their exact logit z = (x - mean) . w_n (the centred
// fp32 row staged in smem; one warp per candidate, all in flight); the first
// maximum -> best[row]. With `logits` every logit is computed exactly and
// written scaled by rstd (diagnostics); a candidate overflow does the same.
// The last row of a request to finish applies the acceptance rule (fused
// accept: a per-request arrival counter, reset by that row).
__global__ void __launch_bounds__(kRefineThreads)
    refine_kernel(const float* __restrict__ x, const __nv_bfloat16* __restrict__ wt, int width, int vocab,
                  int n_tiles, const int32_t* __restrict__ cand_cnt, const int32_t* __restrict__ cand_n,
                  const float* __restrict__ cand_z, const float* __restrict__ mean, const float* __restrict__ rstd,
                  const float* __restrict__ ebound, unsigned long long* __restrict__ best,
                  float* __restrict__ logits, int n_q, int32_t* __restrict__ req_count,
                  const int32_t* __restrict__ drafts, int32_t* __restrict__ target, int32_t* __restrict__ n_accepted) {
    const int row = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    extern __shared__ float4 s_x4[];  // [width / 4]
    __shared__ int s_list[kMaxList];
    __shared__ int s_n;
    __shared__ bool s_all;
    __shared__ unsigned long long s_top;
    pdl_wait();
    const float4* xr = reinterpret_cast<const float4*>(x + size_t(row) * width);
    const float mu = mean[row];
    for (int i = tid; i < width / 4; i += kRefineThreads) {  // the centred row
        const float4 v = xr[i];
        s_x4[i] = make_float4(v.x - mu, v.y - mu, v.z - mu, v.w - mu);
    }
    // gather (all threads): thread t reads the counts of tiles t, t + 256, ...
    // and appends their candidates within the bound to the row's list (value
    // and index in one round trip); a tile whose slots overflowed, or a list
    // longer than kMaxList, falls back to scoring every vocab entry
    if (tid == 0) {
        s_all = logits != nullptr;
        s_n = 0;
        s_top = 0ull;
    }
    __syncthreads();
    const float thresh = key_value(best[row]) - 2.f * ebound[row];
    if (!s_all) {
        for (int t = tid; t < n_tiles; t += kRefineThreads) {
            const int c = cand_cnt[size_t(row) * n_tiles + t];
            if (c > kPerTile) {
                s_all = true;
                continue;
            }
            const size_t b0 = (size_t(row) * n_tiles + t) * kPerTile;
            for (int i = 0; i < c; ++i) {
                const float z = cand_z[b0 + i];
                const int n = cand_n[b0 + i];
                if (z >= thresh) {
                    const int k = atomicAdd(&s_n, 1);
                    if (k < kMaxList) s_list[k] = n;
                    else s_all = true;
                }
            }
        }
    }
    __syncthreads();
    const bool all = s_all;
    const int count = all ? vocab : s_n;
    unsigned long long top = 0ull;
    for (int i = warp; i < count; i += kRefineThreads / 32) {
        const int n = all ? i : s_list[i];
        EP_DCHECK(n >= 0 && n < vocab);
        const uint2* wr = reinterpret_cast<const uint2*>(wt + size_t(n) * width);
        float acc = 0.f;
#pragma unroll 16
        for (int c = lane; c < width / 4; c += 32) {
            const float4 xv = s_x4[c];
            const uint2 w = wr[c];
            const float2 w01 = bf16x2_to_float2(w.x), w23 = bf16x2_to_float2(w.y);
            acc = fmaf(xv.x, w01.x, acc);
            acc = fmaf(xv.y, w01.y, acc);
            acc = fmaf(xv.z, w23.x, acc);
            acc = fmaf(xv.w, w23.y, acc);
        }
        const float z = warp_sum(acc);
        const unsigned long long k = order_key(z, uint32_t(n));
        top = k > top ? k : top;
        if (logits && lane == 0) logits[size_t(row) * vocab + n] = z * rstd[row];
    }
    if (lane == 0 && top) atomicMax(&s_top, top);
    __syncthreads();
    if (tid == 0) {
        best[row] = s_top;
        if (req_count) {
            const int b = row / n_q;
            __threadfence();
            if (atomicAdd(&req_count[b], 1) == n_q - 1) {
                __threadfence();
                accept_request(best, b, n_q, drafts, target, n_accepted);
                req_count[b] = 0;  // ready for the next launch
            }
        }
    }
}

// g_j from the packed keys; n = longest draft prefix reproduced by the target.
__global__ void accept_kernel(const unsigned long long* __restrict__ best, int batch, int n_q,
                              const int32_t* __restrict__ drafts, int32_t* __restrict__ target,
                              int32_t* __restrict__ n_accepted) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < batch) accept_request(best, b, n_q, drafts, target, n_accepted);
}

// Launch with programmatic dependent launch: the kernel may start while its
// predecessor drains; it calls griddepcontrol.wait before reading its inputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace

cudaError_t launch_colsum(const void* wt, int width, int vocab, float* colsum, float* wmax2, cudaStream_t s) {
    colsum_kernel<<<(vocab + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(wt), width,
                                                  vocab, colsum);
    cudaError_t e = cudaMemsetAsync(wmax2, 0, sizeof(float), s);
    if (e != cudaSuccess) return e;
    colnorm_max_kernel<<<(vocab + 7) / 8, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(wt), width,
                                                       vocab, wmax2);
    return cudaGetLastError();
}

// GEMM form: stream-K 128 x 256 tiles over one CTA per SM (default),
// EP_K4_PAIR=1 CTA-pair tiles (cta_group::2, 256 rows), EP_K4_1SM=1 one
// 128 x tn tile per CTA.
int score_mode() {
    static const int mode = [] {
        const char* p = std::getenv("EP_K4_PAIR");
        const char* o = std::getenv("EP_K4_1SM");
        if (o && o[0] == '1') return kScoreOneSm;
        if (p && p[0] == '1') return kScorePair;
        return kScoreStreamK;
    }();
    return mode;
}

// Tile width: 256 for stream-K; for the one-tile-per-CTA forms the width
// giving one wave (1-SM tiles of 128 rows over n_sms CTAs or CTA-pair tiles
// of 256 rows over n_sms / 2 pairs), a multiple of 32 (epilogue chunks; for
// pairs also the per-CTA half of 16-row TMA boxes).
int score_tile_n(int rows, int vocab, int n_sms) {
    const int mode = score_mode();
    if (mode == kScoreStreamK) return kTNMax;
    const bool pairs = mode == kScorePair;
    const int m_tiles = pairs ? (rows + 2 * kTM - 1) / (2 * kTM) : (rows + kTM - 1) / kTM;
    const int slots = pairs ? n_sms / 2 : n_sms;
    const int n_max = slots / m_tiles > 0 ? slots / m_tiles : 1;
    int tn = (vocab + n_max - 1) / n_max;
    tn = (tn + 31) / 32 * 32;
    return tn < 32 ? 32 : tn > kTNMax ? kTNMax : tn;
}

int score_w_box_rows(int tn) { return score_mode() == kScorePair ? tn / 2 : tn; }

// Candidate tiles of the refinement (per row): one per vocab tile, or per
// 128-column half tile for stream-K (two epilogue warps per tile).
int score_cand_tiles(int vocab, int tn) {
    return score_mode() == kScoreStreamK ? (vocab + 127) / 128 : (vocab + tn - 1) / tn;
}

size_t score_streamk_ws_bytes(int n_sms) { return size_t(n_sms) * kTNMax * kTM * sizeof(float); }

cudaError_t launch_score_accept(int rows, int width, int vocab, int tn, const void* attn_out, void* split,
                                const CUtensorMap& tmap_a, const CUtensorMap& tmap_w,
                                const float* colsum, float* mean, float* rstd,
                                unsigned long long* best, float* logits, int batch, int n_q,
                                const int32_t* drafts, int32_t* target, int32_t* n_accepted,
                                const RefineArgs& rf, cudaStream_t s) {
    // (the argmax keys are cleared by the row-stats kernel, so attention ->
    // row stats -> GEMM -> refine are adjacent kernels for programmatic
    // dependent launch)
    cudaError_t e = cudaSuccess;
    if (split)
        e = launch_pdl(row_stats_split_kernel, dim3(rows), dim3(kStatThreads), 0, s,
                       static_cast<const float*>(attn_out), width, mean, rstd,
                       static_cast<__nv_bfloat16*>(split), static_cast<const float*>(rf.wmax2), rf.ebound,
                       static_cast<const uint8_t*>(rf.wt), size_t(width) * size_t(vocab) * 2, best);
    else
        e = launch_pdl(row_stats_kernel<__nv_bfloat16>, dim3(rows), dim3(256), 0, s,
                       static_cast<const __nv_bfloat16*>(attn_out), width, mean, rstd,
                       static_cast<__nv_bfloat16*>(nullptr), best);
    if (e != cudaSuccess) return e;

    static unsigned long long* trace = [] {
        unsigned long long* b = nullptr;
        const char* e = std::getenv("EP_TRACE");
        if (e && e[0] == '1' && cudaMalloc(&b, 4096 * sizeof(unsigned long long)) == cudaSuccess)
            cudaMemset(b, 0, 4096 * sizeof(unsigned long long));
        return b;
    }();
    // fp32 rows: the GEMM on the bf16 hi part only, then the exact refinement
    const int n_tiles = score_cand_tiles(vocab, tn);
    ScoreArgs sa{rows, width, vocab, 1, mean, rstd, colsum, best, split ? nullptr : logits, trace,
                 split ? rf.ebound : nullptr, split ? rf.cand_cnt : nullptr, split ? rf.cand_n : nullptr,
                 split ? rf.cand_z : nullptr, n_tiles, tn, score_stages(tn),
                 umma::idesc_bf16_f32(kTM, tn, false, false)};
    const int mode = score_mode();
    if (mode == kScoreStreamK) {
        sa.tiles_m = (rows + kTM - 1) / kTM;
        sa.nkt = width / kTK;
        sa.n_vt = (vocab + kTNMax - 1) / kTNMax;
        sa.sk_ws = rf.sk_ws;
        sa.sk_flags = rf.sk_flags;
        sa.stages = std::min(kStagesMax, (227 * 1024 - kSkSmemFixed) / score_stage_bytes(kTNMax));
        const long long total = (long long)sa.tiles_m * sa.n_vt * sa.nkt;
        const int grid = int(std::min<long long>(total, rf.sk_ctas));
        const int smem = sa.stages * score_stage_bytes(kTNMax) + kSkSmemFixed;
        if (cudaError_t e2 = ensure_smem<score_argmax_streamk_kernel>(227 * 1024)) return e2;
        e = launch_pdl(score_argmax_streamk_kernel, dim3(grid), dim3(kSkThreads), smem, s, sa, tmap_a, tmap_w);
    } else if (mode == kScorePair) {
        // CTA pairs: stage = A 16 KB + half of the W rows
        const int stage = kABytes + (tn / 2) * kTK * 2;
        sa.stages = std::min(kStagesMax, kScoreSmemBudget / stage);
        sa.idesc = umma::idesc_bf16_f32(2 * kTM, tn, false, false);
        const int smem = sa.stages * stage + kScoreSmemFixed;
        if (cudaError_t e2 = ensure_smem<score_argmax_pair_kernel>(227 * 1024)) return e2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * ((rows + 2 * kTM - 1) / (2 * kTM)), n_tiles);
        cfg.blockDim = dim3(kScoreThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = 2;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        e = cudaLaunchKernelEx(&cfg, score_argmax_pair_kernel, sa, tmap_a, tmap_w);
    } else {
        const int smem = score_stages(tn) * score_stage_bytes(tn) + kScoreSmemFixed;
        if (cudaError_t e2 = ensure_smem<score_argmax_kernel>(227 * 1024)) return e2;
        dim3 grid((rows + kTM - 1) / kTM, n_tiles);
        e = launch_pdl(score_argmax_kernel, grid, dim3(kScoreThreads), smem, s, sa, tmap_a, tmap_w);
    }
    if (e != cudaSuccess) return e;
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
    if (split)
        e = launch_pdl(refine_kernel, dim3(rows), dim3(kRefineThreads), size_t(width) * 4, s,
                       static_cast<const float*>(attn_out), static_cast<const __nv_bfloat16*>(rf.wt), width, vocab,
                       n_tiles, static_cast<const int32_t*>(rf.cand_cnt), static_cast<const int32_t*>(rf.cand_n),
                       static_cast<const float*>(rf.cand_z), static_cast<const float*>(mean),
                       static_cast<const float*>(rstd), static_cast<const float*>(rf.ebound), best, logits, n_q,
                       rf.req_count, drafts, target, n_accepted);
    else
        accept_kernel<<<(batch + 127) / 128, 128, 0, s>>>(best, batch, n_q, drafts, target, n_accepted);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace ep
