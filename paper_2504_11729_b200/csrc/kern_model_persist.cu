// kern_model_persist.cu — K9: a whole greedy rollout of a small decoder in ONE
// persistent cooperative kernel (decode_greedy, model.cpp:285-297, for the
// BASELINE config-1 class of models: fp32, a few rows).
//
// The CUDA-graph rollout of ep_model_generate replays ~11 kernels per token;
// for config 1 (d_model 256, 2 layers) every kernel is a few microseconds of
// launch, fill and drain around well under a microsecond of work. Here one CTA
// per SM stays resident for all n_steps tokens and the layer's stages are
// separated by grid-wide barriers instead of kernel boundaries:
//
//   per step:  [LN + Q|K|V, K/V rows -> pages]  (layer 0: embedding fused)
//              [attention partials: one (row, head, page) task per CTA]
//              [LSE merge of the partials + Wo + residual]
//              [LN + W1 + b1 + ReLU]
//              [W2 + b2 + residual]                         x n_layers
//              [LN + unembedding; the last CTA: argmax -> next token]
//
// Weights stay in SHARED memory for the whole rollout: every GEMV stage gives
// CTA i the contiguous output columns [i N / G, (i + 1) N / G) and the CTA
// copies those columns of every layer's matrices into shared memory once
// (config 1: ~26 KB per CTA). A stage is then one L2 read of its B input rows
// (LayerNorm recomputed per CTA, model.cpp:131-150), shared-memory FMAs split
// over k-slices and reduced in a fixed order (deterministic), and the
// epilogue stores — no split-K partials through global memory. Attention is
// partial_attention per 64-key page with the causal rule (keys at positions
// <= the query, attention.cpp:29-33, :80-114), merged by LSE
// (attention.cpp:116-145).
#include <algorithm>
#include <cmath>
#include <cstdint>

#include "ep_common.cuh"
#include "model_internal.h"

namespace ep {
namespace {

constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr int kMaxB = 8;
constexpr int kMaxNcp = 32;    // output columns of one stage per CTA (power of two)
constexpr float kEps = 1e-5f;  // model.cpp:14

// Order-preserving 64-bit key of (logit, id): larger logit first, then the
// lower id (argmax_token's strict '>' keeps the first maximum).
__device__ __forceinline__ unsigned long long order_key(float z, uint32_t idx) {
    // argmax_token compares with '>': -0 == +0 (canonicalised so the lower
    // id wins the tie), and a NaN is never taken over a number — except at
    // id 0, where the scan starts and nothing compares greater than it
    if (z != z) return idx == 0 ? ~0ull : 0ull;
    uint32_t b = __float_as_uint(z == 0.f ? 0.f : z);
    b = (b & 0x80000000u) ? ~b : (b | 0x80000000u);
    return (uint64_t(b) << 32) | uint64_t(0xFFFFFFFFu - idx);
}

__host__ __device__ inline int pow2ceil(int v) {
    int p = 1;
    while (p < v) p <<= 1;
    return p;
}
// Columns per CTA of an N-column stage, rounded up to a power of two.
__host__ __device__ inline int stage_ncp(int N, int G) { return pow2ceil((N + G - 1) / G); }

__host__ __device__ inline size_t pad4(size_t v) { return (v + 3) & ~size_t(3); }

// Shared-memory floats of the resident weights (layers x {QKV, Wo, W1 + b1,
// W2 + b2} + unembedding), each block padded to 16 bytes.
__host__ __device__ inline size_t resident_floats(int L, int D, int F, int V, int G) {
    const size_t layer = pad4(size_t(D) * stage_ncp(3 * D, G)) + pad4(size_t(D) * stage_ncp(D, G)) +
                         pad4(size_t(D + 1) * stage_ncp(F, G)) + pad4(size_t(F + 1) * stage_ncp(D, G));
    return L * layer + pad4(size_t(D) * stage_ncp(V, G));
}

// GEMV reduction / attention q scratch floats ([8 warps][kMaxB][kMaxNcp] >= [8 warps][128]).
__host__ __device__ inline size_t scratch_floats() { return size_t(kPThreads / 32) * kMaxB * kMaxNcp; }

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier k (1, 2, ...): a monotonic arrival counter, zero at launch;
// release on arrival, acquire on the poll (cooperative launch: all CTAs are
// resident).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned k) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned target = k * gridDim.x;
        while (ld_acquire(bar) < target) {
        }
    }
    __syncthreads();
}

// LayerNorm in place of B rows of width D in shared memory.
__device__ void ln_smem(float* xs, int B, int D) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < B; b += kPWarps) {
        float* xr = xs + size_t(b) * D;
        float s = 0.f;
        for (int c = lane; c < D; c += 32) s += xr[c];
        const float mean = warp_sum(s) / float(D);
        float q = 0.f;
        for (int c = lane; c < D; c += 32) {
            const float d = xr[c] - mean;
            q += d * d;
        }
        const float inv = 1.f / sqrtf(warp_sum(q) / float(D) + kEps);
        for (int c = lane; c < D; c += 32) xr[c] = (xr[c] - mean) * inv;
    }
}

// xs[B][n] = src[B][n] from global (L2), float4 when aligned.
__device__ void load_rows(const float* src, int count, float* xs) {
    if ((count & 3) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        float4* d4 = reinterpret_cast<float4*>(xs);
        for (int i = threadIdx.x; i < count / 4; i += kPThreads) d4[i] = __ldcg(s4 + i);
    } else {
        for (int i = threadIdx.x; i < count; i += kPThreads) xs[i] = __ldcg(src + i);
    }
}

// One GEMV stage over this CTA's columns [c0, c0 + nc): y[b][c] = xs[b][:] . W[:, c]
// with W resident as ws[K][ncp]. Thread (column j, k-slice s) sums k = s, s + S,
// ...; the S slices are added in a fixed order. epi(b, c, value).
template <typename Epi>
__device__ void gemv_cols(const float* xs, const float* ws, int B, int K, int ncp, int c0, int nc, float* red,
                          Epi epi) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int j = tid & (ncp - 1), s = tid / ncp, S = kPThreads / ncp;
    float acc[kMaxB];
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) acc[b] = 0.f;
    if (j < nc) {
#pragma unroll 4
        for (int k = s; k < K; k += S) {
            const float w = ws[size_t(k) * ncp + j];
#pragma unroll
            for (int b = 0; b < kMaxB; ++b)
                if (b < B) acc[b] = fmaf(xs[size_t(b) * K + k], w, acc[b]);
        }
    }
    // slices inside the warp (lanes differing in the bits above j)
#pragma unroll
    for (int b = 0; b < kMaxB; ++b) {
        if (b < B)
            for (int m = ncp; m < 32; m <<= 1) acc[b] += __shfl_xor_sync(0xffffffffu, acc[b], m);
    }
    // then across warps, in warp order
    if (lane < ncp) {  // lane == j here
#pragma unroll
        for (int b = 0; b < kMaxB; ++b)
            if (b < B) red[(warp * kMaxB + b) * kMaxNcp + j] = acc[b];
    }
    __syncthreads();
    for (int i = tid; i < nc * B; i += kPThreads) {
        const int b = i / nc, jj = i - b * nc;
        float v = 0.f;
        for (int w = 0; w < kPWarps; ++w) v += red[(w * kMaxB + b) * kMaxNcp + jj];
        epi(b, c0 + jj, v);
    }
    __syncthreads();
}

struct Stage {
    int K, N, ncp, c0, nc;
    float* ws;    // [K][ncp]
    float* bias;  // [ncp] (stages with a bias)
};

__device__ Stage make_stage(int K, int N, bool has_bias, float*& wcur) {
    Stage st;
    st.K = K;
    st.N = N;
    st.ncp = stage_ncp(N, gridDim.x);
    st.c0 = int((int64_t(blockIdx.x) * N) / gridDim.x);
    st.nc = int((int64_t(blockIdx.x + 1) * N) / gridDim.x) - st.c0;
    st.ws = wcur;
    st.bias = has_bias ? wcur + size_t(K) * st.ncp : nullptr;
    wcur += pad4(size_t(K + (has_bias ? 1 : 0)) * st.ncp);
    return st;
}

__device__ void load_bias(const Stage& st, const float* b) {
    for (int j = threadIdx.x; j < st.ncp; j += kPThreads) st.bias[j] = j < st.nc ? __ldg(b + st.c0 + j) : 0.f;
}

// Copy this CTA's columns of W (column pointer col_ptr(c, k)) into ws: eight
// loads per thread in flight (a launch for one decode step spends most of its
// time here otherwise).
template <typename ColPtr>
__device__ void load_stage(const Stage& st, ColPtr col_ptr) {
    const int total = st.K * st.ncp;
    for (int i0 = threadIdx.x; i0 < total; i0 += 8 * kPThreads) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * kPThreads, k = i / st.ncp, j = i - k * st.ncp;
            v[u] = (i < total && j < st.nc) ? __ldg(col_ptr(st.c0 + j, k)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (i0 + u * kPThreads < total) st.ws[i0 + u * kPThreads] = v[u];
    }
}

// One warp: partial attention (attention.cpp:80-114) of q over nk <= 32
// consecutive keys (rows of kt / vt, DH floats each) -> part = {max, sum,
// o[DH]}.
template <int DH>
__device__ __forceinline__ void attn_task(const float* kt, const float* vt, const float* q, int nk, float scale,
                                          float* part) {
    constexpr int KV4 = DH / 4, VPL = DH / 32;
    const int lane = threadIdx.x & 31;
    float4 kv[KV4];
    float vv[32][VPL];
    const float4* kr = reinterpret_cast<const float4*>(kt + size_t(lane) * DH);
#pragma unroll
    for (int i = 0; i < KV4; ++i) kv[i] = lane < nk ? __ldcg(kr + i) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < 32; ++j)
#pragma unroll
        for (int v = 0; v < VPL; ++v) vv[j][v] = j < nk ? __ldcg(vt + size_t(j) * DH + lane * VPL + v) : 0.f;
    // the dot product of this lane's key; q is a shared-memory broadcast
    const float4* q4 = reinterpret_cast<const float4*>(q);
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int i = 0; i < KV4; i += 2) {
        const float4 a0 = q4[i], b0 = kv[i];
        s0 = fmaf(a0.x, b0.x, fmaf(a0.y, b0.y, fmaf(a0.z, b0.z, fmaf(a0.w, b0.w, s0))));
        const float4 a1 = q4[i + 1], b1 = kv[i + 1];
        s1 = fmaf(a1.x, b1.x, fmaf(a1.y, b1.y, fmaf(a1.z, b1.z, fmaf(a1.w, b1.w, s1))));
    }
    const float sc = lane < nk ? (s0 + s1) * scale : -INFINITY;
    const float m = warp_max(sc);
    const float p = lane < nk ? __expf(sc - m) : 0.f;
    const float l = warp_sum(p);
    float o[VPL];
#pragma unroll
    for (int v = 0; v < VPL; ++v) o[v] = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const float pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
        for (int v = 0; v < VPL; ++v) o[v] = fmaf(pj, vv[j][v], o[v]);
    }
    if (lane == 0) {
        part[0] = m;
        part[1] = l;
    }
#pragma unroll
    for (int v = 0; v < VPL; ++v) part[2 + lane * VPL + v] = o[v];
}

// One warp: merge the n2 partials {max, sum, o[dh]} at part (row stride dh + 2)
// into out[dh], online in chunks of 32 (attention.cpp:116-145); empty
// partials (max = -inf) have weight 0 and are never multiplied.
__device__ void merge_head(const float* part, int n2, int dh, float* out) {
    const int lane = threadIdx.x & 31;
    const int S = dh + 2, vpl = dh / 32;
    float M = -INFINITY, Ls = 0.f, o[4] = {0.f, 0.f, 0.f, 0.f};
    for (int c0 = 0; c0 < n2; c0 += 32) {
        const int c = c0 + lane;
        const float mv = c < n2 ? __ldcg(part + size_t(c) * S) : -INFINITY;
        const float lv = c < n2 ? __ldcg(part + size_t(c) * S + 1) : 0.f;
        const float Mb = fmaxf(M, warp_max(mv));
        const float sc = M == -INFINITY ? 0.f : __expf(M - Mb);
        Ls *= sc;
#pragma unroll
        for (int r = 0; r < 4; ++r) o[r] *= sc;
        const float w = mv == -INFINITY ? 0.f : __expf(mv - Mb);
        Ls += warp_sum(w * lv);
        const int cnt = min(32, n2 - c0);
        for (int j0 = 0; j0 < cnt; j0 += 8) {
            float v[8][4];
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    v[j][r] = (j0 + j < cnt && r < vpl) ? __ldcg(part + size_t(c0 + j0 + j) * S + 2 + lane + 32 * r) : 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float wj = __shfl_sync(0xffffffffu, w, (j0 + j) & 31);
                if (j0 + j < cnt && wj != 0.f)
#pragma unroll
                    for (int r = 0; r < 4; ++r) o[r] = fmaf(wj, v[j][r], o[r]);
            }
        }
        M = Mb;
    }
    for (int r = 0; r < vpl; ++r) out[lane + 32 * r] = o[r] / Ls;
}

// The shared-memory layout of one CTA's resident weights from `base`: per
// layer the Q|K|V, Wo, W1 (+ b1) and W2 (+ b2) column slices, then the
// unembedding's; base is advanced past them.
__device__ void resident_layout(int L, int D, int F, int V, float*& base, Stage* sq, Stage* so, Stage* s1,
                                Stage* s2, Stage& su) {
    for (int l = 0; l < L; ++l) {
        sq[l] = make_stage(D, 3 * D, false, base);
        so[l] = make_stage(D, D, false, base);
        s1[l] = make_stage(D, F, true, base);
        s2[l] = make_stage(F, D, true, base);
    }
    su = make_stage(D, V, false, base);
}

// CTA i of a G-CTA grid writes CTA i's resident image (the same bytes the
// rollout kernel keeps in shared memory) to image + i * resident_floats.
__global__ void __launch_bounds__(kPThreads) persist_image_kernel(const PersistArgs a) {
    const int L = a.L, D = a.D, F = a.F, V = a.V;
    float* base = a.image_out + size_t(blockIdx.x) * resident_floats(L, D, F, V, gridDim.x);
    constexpr int kMaxL = 8;
    Stage sq[kMaxL], so[kMaxL], s1[kMaxL], s2[kMaxL];
    Stage su;
    resident_layout(L, D, F, V, base, sq, so, s1, s2, su);
    for (int l = 0; l < L; ++l) {
        const PersistLayer& Lw = a.layers[l];
        load_bias(s1[l], Lw.b1);
        load_bias(s2[l], Lw.b2);
        load_stage(sq[l], [&](int c, int k) {
            const int which = c / D;
            const float* W = which == 0 ? Lw.wq : which == 1 ? Lw.wk : Lw.wv;
            return W + size_t(k) * D + (c - which * D);
        });
        load_stage(so[l], [&](int c, int k) { return Lw.wo + size_t(k) * D + c; });
        load_stage(s1[l], [&](int c, int k) { return Lw.w1 + size_t(k) * F + c; });
        load_stage(s2[l], [&](int c, int k) { return Lw.w2 + size_t(k) * D + c; });
    }
    load_stage(su, [&](int c, int k) { return a.unembed + size_t(k) * V + c; });
}

__global__ void __launch_bounds__(kPThreads, 1) decode_persist_kernel(const PersistArgs a) {
    extern __shared__ __align__(16) float smem_f[];
    const int B = a.B, D = a.D, H = a.H, dh = a.dh, F = a.F, V = a.V, P = a.P, L = a.L;
    const int Kmax = F > D ? F : D;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.f / sqrtf(float(dh));
    unsigned* bar = reinterpret_cast<unsigned*>(a.counters);
    int* bh_arrive = a.counters + 2;  // [B][H] attention tasks finished per (row, head)

    // ---- resident weights: this CTA's columns of every stage ----
    // a.image (built once per model by persist_image_kernel) holds every
    // CTA's shared-memory image contiguously: one bulk async copy
    float* wcur = smem_f;
    constexpr int kMaxL = 8;
    Stage sq[kMaxL], so[kMaxL], s1[kMaxL], s2[kMaxL];
    Stage su;
    resident_layout(L, D, F, V, wcur, sq, so, s1, s2, su);
    {
        __shared__ __align__(8) uint64_t img_bar;
        if (tid == 0) {
            mbar_init(&img_bar, 1);
            fence_mbar_init();
            const uint32_t bytes = uint32_t((wcur - smem_f) * sizeof(float));
            mbar_arrive_expect_tx(&img_bar, bytes);
            bulk_g2s(smem_f, a.image + size_t(blockIdx.x) * (wcur - smem_f), bytes, &img_bar);
        }
        __syncthreads();
        mbar_wait(&img_bar, 0);
    }
    float* xs = wcur;                          // [B][Kmax] stage input rows
    const int ncp_d = so[0].ncp;               // Wo and W2 share the column split (N = D)
    float* res = xs + size_t(B) * Kmax;        // [B][ncp_d] residual stream of this CTA's columns
    float* s_att = res + pad4(size_t(B) * ncp_d);  // attention / reduction scratch
    float* red = s_att;                        // [8 warps][kMaxB][kMaxNcp]
    const int MC = 2 * a.max_chunks;            // partials per (row, head): 32-key halves
    // batch > 1: the last task of each (row, head) merges it once (fewer L2
    // reads than every CTA merging every row); batch 1: every CTA merges
    const bool fuse_merge = B > 1;
    __shared__ unsigned long long s_key[kMaxB];
    __shared__ int tok_s[kMaxB];
    // argmax_token (model.cpp:248-255) of step s: the maximum over every
    // CTA's candidate key (first maximum: ties go to the lowest id) -> tok_s;
    // CTA 0 also writes it to out[s]
    auto next_tokens = [&](int s) {
        for (int b = warp; b < B; b += kPWarps) {
            unsigned long long k = 0ull;
            for (int g = lane; g < int(gridDim.x); g += 32) {
                const unsigned long long o = __ldcg(a.keys + size_t(g) * B + b);
                k = o > k ? o : k;
            }
#pragma unroll
            for (int m = 16; m > 0; m >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xffffffffu, k, m);
                k = o > k ? o : k;
            }
            if (lane == 0) {
                const int tok = k ? int(0xFFFFFFFFu - uint32_t(k & 0xFFFFFFFFull)) : 0;
                tok_s[b] = tok;
                if (blockIdx.x == 0) a.out[size_t(s) * B + b] = tok;
            }
        }
    };
    __syncthreads();

    unsigned n_bar = 0;
    int n_step_bar = 0;
    // debug (a.trace): CTA 0 stamps the globaltimer after every grid barrier
    auto sync = [&](int t) {
        grid_barrier(bar, ++n_bar);
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 8 && n_step_bar < 31) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            a.trace[t * 32 + n_step_bar] = ts;
        }
        ++n_step_bar;
    };

    for (int t = 0; t < a.n_steps; ++t) {
        n_step_bar = 0;
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 8) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            a.trace[t * 32 + 31] = ts;
        }
        for (int l = 0; l < L; ++l) {
            const PersistLayer& Lw = a.layers[l];
            // ---- LN(x) -> Q | K | V; layer 0 embeds the step's tokens first ----
            if (l == 0) {
                // model.cpp:104-129 with the fp64 sinusoid table; CTA 0 stores
                // the embedded rows (the residual input)
                if (t == 0) {
                    if (tid < B) tok_s[tid] = a.first[tid];
                } else {
                    next_tokens(t - 1);
                }
                __syncthreads();
                for (int i = tid; i < B * D; i += kPThreads) {
                    const int b = i / D, c = i - b * D;
                    const int tok = tok_s[b];
                    const int pos = a.pos[size_t(t) * B + b];
                    const float v = float(double(a.emb[size_t(tok) * D + c]) + a.pe[size_t(pos) * D + c]);
                    xs[i] = v;
                }
                __syncthreads();
                for (int i = tid; i < B * so[0].nc; i += kPThreads) {
                    const int b = i / so[0].nc, j = i - b * so[0].nc;
                    res[b * ncp_d + j] = xs[size_t(b) * D + so[0].c0 + j];
                }
            } else {
                load_rows(a.x, B * D, xs);
            }
            __syncthreads();
            ln_smem(xs, B, D);
            __syncthreads();
            gemv_cols(xs, sq[l].ws, B, D, sq[l].ncp, sq[l].c0, sq[l].nc, red, [&](int b, int c, float v) {
                const int which = c / D, cc = c - which * D;
                if (which == 0) {
                    a.q[size_t(b) * D + cc] = v;
                } else {
                    const int h = cc / dh, e = cc - h * dh;
                    const size_t idx = ((size_t(a.dst_page[size_t(t) * B + b]) * H + h) * P +
                                        a.dst_slot[size_t(t) * B + b]) * dh + e;
                    (which == 1 ? Lw.kp : Lw.vp)[idx] = v;
                }
            });
            sync(t);

            // ---- attention partials: (row, head, page, 32-key half) warp tasks ----
            // spread one per CTA first (task u: CTA u % G, warp u / G); a task's
            // K and V rows are loaded in one L2 round trip (attn_task)
            {
                int total = 0;
                for (int b = 0; b < B; ++b) total += H * 2 * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                for (int u = warp * gridDim.x + blockIdx.x; u < total; u += gridDim.x * kPWarps) {
                    int b = 0, rem = u;
                    while (rem >= H * 2 * int(a.req_page_off[b + 1] - a.req_page_off[b])) {
                        rem -= H * 2 * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                        ++b;
                    }
                    const int n2 = 2 * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const int h = rem / n2, c2 = rem - h * n2;
                    const PageDesc d = a.pdesc[a.req_page_off[b] + c2 / 2];
                    const int64_t vis = int64_t(a.pos[size_t(t) * B + b]) - d.pos + 1;
                    const int nk_page = vis <= 0 ? 0 : (vis < d.n_tok ? int(vis) : d.n_tok);
                    const int k0 = (c2 & 1) * 32;
                    const int nk = nk_page - k0 < 0 ? 0 : (nk_page - k0 > 32 ? 32 : nk_page - k0);
                    float* part = a.part + (size_t(b * H + h) * MC + c2) * (dh + 2);
                    if (nk == 0) {  // no visible key: an empty partial (weight 0, zero output)
                        if (lane == 0) {
                            part[0] = -INFINITY;
                            part[1] = 0.f;
                        }
                        for (int e = lane; e < dh; e += 32) part[2 + e] = 0.f;
                    } else {
                        // q of (b, h) straight from L2 (written before the barrier)
                        float* qs = s_att + warp * 128;
                        for (int e = lane; e < dh; e += 32) qs[e] = __ldcg(a.q + size_t(b) * D + h * dh + e);
                        __syncwarp();
                        const size_t off = ((size_t(d.page) * H + h) * P + k0) * dh;
                        if (dh == 64)
                            attn_task<64>(Lw.kp + off, Lw.vp + off, qs, nk, scale, part);
                        else
                            attn_task<32>(Lw.kp + off, Lw.vp + off, qs, nk, scale, part);
                    }
                    if (!fuse_merge) {
                        __syncwarp();
                        continue;
                    }
                    // the last of the (row, head)'s n2 tasks to finish merges them
                    // (attention.cpp:116-145) into att[b][h dh, (h + 1) dh)
                    __threadfence();
                    __syncwarp();
                    int last = 0;
                    if (lane == 0) last = atomicAdd(&bh_arrive[b * H + h], 1) == n2 - 1;
                    last = __shfl_sync(0xffffffffu, last, 0);
                    if (last) {
                        __threadfence();
                        merge_head(a.part + size_t(b * H + h) * MC * (dh + 2), n2, dh, a.att + size_t(b) * D + h * dh);
                        if (lane == 0) bh_arrive[b * H + h] = 0;
                    }
                    __syncwarp();
                }
            }
            sync(t);

            // ---- merged attention rows + Wo + residual ----
            if (fuse_merge) {
                load_rows(a.att, B * D, xs);
                __syncthreads();
            } else {
                // batch 1: every CTA merges the row itself — a thread's (row,
                // dimension) loads the maxima, sums and outputs of all of the
                // row's partials in one L2 round trip and merges them online
                // (attention.cpp:116-145); cheaper than the last-arriver chain
                for (int i = tid; i < B * D; i += kPThreads) {
                    const int b = i / D, cc = i - b * D, h = cc / dh, e = cc - h * dh;
                    const int n2 = 2 * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const float* base = a.part + size_t(b * H + h) * MC * (dh + 2);
                    float o = 0.f, Ls = 0.f, M = -INFINITY;
                    for (int c0 = 0; c0 < n2; c0 += 32) {
                        float mv[32], lv[32], ov[32];
#pragma unroll
                        for (int u = 0; u < 32; ++u) {
                            const bool ok = c0 + u < n2;
                            const float* pc = base + size_t(c0 + u) * (dh + 2);
                            mv[u] = ok ? __ldcg(pc) : -INFINITY;
                            lv[u] = ok ? __ldcg(pc + 1) : 0.f;
                            ov[u] = ok ? __ldcg(pc + 2 + e) : 0.f;
                        }
                        float Mb = M;
#pragma unroll
                        for (int u = 0; u < 32; ++u) Mb = fmaxf(Mb, mv[u]);
                        const float sc = M == -INFINITY ? 0.f : __expf(M - Mb);
                        o *= sc;
                        Ls *= sc;
#pragma unroll
                        for (int u = 0; u < 32; ++u) {
                            if (mv[u] == -INFINITY) continue;  // empty partial: never touch its output
                            const float wgt = __expf(mv[u] - Mb);
                            Ls = fmaf(wgt, lv[u], Ls);
                            o = fmaf(wgt, ov[u], o);
                        }
                        M = Mb;
                    }
                    xs[i] = o / Ls;
                }
                __syncthreads();
            }
            gemv_cols(xs, so[l].ws, B, D, so[l].ncp, so[l].c0, so[l].nc, red, [&](int b, int c, float v) {
                float& r = res[b * ncp_d + (c - so[l].c0)];
                r = r + v;  // model.cpp:184-185
                a.x2[size_t(b) * D + c] = r;
            });
            sync(t);

            // ---- LN(x2) -> W1 + b1 -> ReLU ----
            load_rows(a.x2, B * D, xs);
            __syncthreads();
            ln_smem(xs, B, D);
            __syncthreads();
            gemv_cols(xs, s1[l].ws, B, D, s1[l].ncp, s1[l].c0, s1[l].nc, red, [&](int b, int c, float v) {
                float h1 = v + s1[l].bias[c - s1[l].c0];  // model.cpp:188-194
                if (h1 < 0.f) h1 = 0.f;
                a.h1[size_t(b) * F + c] = h1;
            });
            sync(t);

            // ---- W2 + b2 + residual ----
            load_rows(a.h1, B * F, xs);
            __syncthreads();
            gemv_cols(xs, s2[l].ws, B, F, s2[l].ncp, s2[l].c0, s2[l].nc, red, [&](int b, int c, float v) {
                float& r = res[b * ncp_d + (c - s2[l].c0)];
                r = (r + v) + s2[l].bias[c - s2[l].c0];  // model.cpp:199-204
                a.x[size_t(b) * D + c] = r;
            });
            sync(t);
        }

        // ---- unembed_logits (model.cpp:238-246) + this CTA's argmax candidates ----
        if (tid < B) s_key[tid] = 0ull;
        load_rows(a.x, B * D, xs);
        __syncthreads();
        ln_smem(xs, B, D);
        __syncthreads();
        gemv_cols(xs, su.ws, B, D, su.ncp, su.c0, su.nc, red, [&](int b, int c, float v) {
            a.logits[size_t(b) * V + c] = v;
            atomicMax(&s_key[b], order_key(v, uint32_t(c)));
        });
        // the first maximum of each row among this CTA's columns; the next
        // step (or the end of the rollout) reduces the candidates of all CTAs
        if (tid < B) a.keys[size_t(blockIdx.x) * B + tid] = s_key[tid];
        sync(t);
    }
    if (blockIdx.x == 0) next_tokens(a.n_steps - 1);
}

}  // namespace

bool persist_supported(int L, int B, int D, int H, int F, int V, int P, int n_sms) {
    const int dh = D / H;
    if (L < 1 || L > 8 || B < 1 || B > kMaxB || D % 4 || F % 4 || P > 64 || n_sms < 1) return false;
    if (dh != 32 && dh != 64) return false;  // attn_task: a lane's K row and V columns in registers
    if (stage_ncp(std::max(std::max(3 * D, F), V), n_sms) > kMaxNcp) return false;
    return persist_smem_bytes(L, B, D, F, H, V, 1, n_sms) <= 200 * 1024;
}

size_t persist_smem_bytes(int L, int B, int D, int F, int H, int V, int max_chunks, int n_sms) {
    const int Kmax = F > D ? F : D;
    (void)H;
    (void)max_chunks;
    return sizeof(float) * (resident_floats(L, D, F, V, n_sms) + size_t(B) * Kmax +
                            pad4(size_t(B) * stage_ncp(D, n_sms)) + scratch_floats());
}

size_t persist_image_floats(int L, int D, int F, int V, int n_ctas) {
    return size_t(n_ctas) * resident_floats(L, D, F, V, n_ctas);
}

cudaError_t launch_persist_image(const PersistArgs& a, int n_ctas, cudaStream_t s) {
    persist_image_kernel<<<n_ctas, kPThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_decode_persist(const PersistArgs& a, int n_ctas, cudaStream_t s) {
    const size_t smem = persist_smem_bytes(a.L, a.B, a.D, a.F, a.H, a.V, a.max_chunks, n_ctas);
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem<decode_persist_kernel>(int(smem))) return e;
    if (cudaError_t e = cudaMemsetAsync(a.counters, 0, size_t(2 + a.B * a.H) * sizeof(int32_t), s)) return e;
    void* args[] = {const_cast<PersistArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(decode_persist_kernel), dim3(n_ctas),
                                       dim3(kPThreads), args, smem, s);
}

}  // namespace ep
