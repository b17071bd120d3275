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

// Attention / GEMV reduction scratch floats.
__host__ __device__ inline size_t scratch_floats(int B, int H, int max_chunks) {
    size_t v = size_t(B) * H * max_chunks + 16;
    if (v < size_t(kPThreads / 32) * kMaxB * kMaxNcp) v = size_t(kPThreads / 32) * kMaxB * kMaxNcp;
    return pad4(v);
}

// Attention page buffers: kNBuf x (K, V) of one (page, head), P x dh floats each.
constexpr int kNBuf = 2;
__host__ __device__ inline size_t att_buf_floats(int P, int dh) { return size_t(kNBuf) * 2 * P * dh; }

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

// Copy this CTA's columns of W (row-major [K][ld], columns via col_of) into ws.
template <typename ColPtr>
__device__ void load_stage(const Stage& st, ColPtr col_ptr) {
    for (int i = threadIdx.x; i < st.K * st.ncp; i += kPThreads) {
        const int k = i / st.ncp, j = i - k * st.ncp;
        float v = 0.f;
        if (j < st.nc) v = __ldg(col_ptr(st.c0 + j, k));
        st.ws[i] = v;
    }
}

__global__ void __launch_bounds__(kPThreads, 1) decode_persist_kernel(const PersistArgs a) {
    extern __shared__ __align__(16) float smem_f[];
    const int B = a.B, D = a.D, H = a.H, dh = a.dh, F = a.F, V = a.V, P = a.P, L = a.L;
    const int Kmax = F > D ? F : D;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.f / sqrtf(float(dh));
    unsigned* bar = reinterpret_cast<unsigned*>(a.counters);
    unsigned* arrive = bar + 1;

    // ---- resident weights: this CTA's columns of every stage ----
    float* wcur = smem_f;
    constexpr int kMaxL = 8;
    Stage sq[kMaxL], so[kMaxL], s1[kMaxL], s2[kMaxL];
    for (int l = 0; l < L; ++l) {
        const PersistLayer& Lw = a.layers[l];
        sq[l] = make_stage(D, 3 * D, false, wcur);
        so[l] = make_stage(D, D, false, wcur);
        s1[l] = make_stage(D, F, true, wcur);
        s2[l] = make_stage(F, D, true, wcur);
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
    const Stage su = make_stage(D, V, false, wcur);
    load_stage(su, [&](int c, int k) { return a.unembed + size_t(k) * V + c; });
    float* xs = wcur;                          // [B][Kmax] stage input rows
    const int ncp_d = so[0].ncp;               // Wo and W2 share the column split (N = D)
    float* res = xs + size_t(B) * Kmax;        // [B][ncp_d] residual stream of this CTA's columns
    float* s_att = res + pad4(size_t(B) * ncp_d);  // attention / reduction scratch
    float* red = s_att;                        // [8 warps][kMaxB][kMaxNcp]
    float* kvbuf = s_att + scratch_floats(B, H, a.max_chunks);  // [kNBuf][K | V][P][dh]
    __shared__ __align__(8) uint64_t mbar[kNBuf];
    if (tid == 0) {
        for (int i = 0; i < kNBuf; ++i) mbar_init(&mbar[i], 1);
        fence_mbar_init();
    }
    unsigned mb_phase = 0;  // parity bit per buffer
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
                for (int i = tid; i < B * D; i += kPThreads) {
                    const int b = i / D, c = i - b * D;
                    const int tok = t == 0 ? a.first[b] : __ldcg(a.out + size_t(t - 1) * B + b);
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

            // ---- attention partials: one (row, head, page) task per CTA ----
            // the task's K and V rows (nk x dh, contiguous in the page) arrive by
            // bulk async copy into a double buffer: the next task's copy is in
            // flight while this one computes
            {
                int total = 0;
                for (int b = 0; b < B; ++b) total += H * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                float* qh = s_att;        // [128]
                float* ps = s_att + 128;  // [64] scores, then probabilities
                float* po = s_att + 192;  // [8][128] PV partials of the key groups
                float* rr = s_att + 1216; // [2] max, sum
                struct Task {
                    int b, h, c, nk, page;
                };
                auto task_of = [&](int u) {
                    Task tk;
                    int b = 0, rem = u;
                    while (rem >= H * int(a.req_page_off[b + 1] - a.req_page_off[b])) {
                        rem -= H * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                        ++b;
                    }
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    tk.b = b;
                    tk.h = rem / npg;
                    tk.c = rem - tk.h * npg;
                    const PageDesc d = a.pdesc[a.req_page_off[b] + tk.c];
                    const int64_t vis = int64_t(a.pos[size_t(t) * B + b]) - d.pos + 1;
                    tk.nk = vis <= 0 ? 0 : (vis < d.n_tok ? int(vis) : d.n_tok);
                    tk.page = d.page;
                    return tk;
                };
                auto issue = [&](int i) {  // thread 0: copy task i of this CTA into buffer i % kNBuf
                    const int u = blockIdx.x + i * gridDim.x;
                    if (u >= total) return;
                    const Task tk = task_of(u);
                    if (tk.nk == 0) return;
                    const int slot = i % kNBuf;
                    const uint32_t bytes = uint32_t(tk.nk) * dh * 4;
                    float* kb = kvbuf + size_t(slot) * 2 * P * dh;
                    const size_t off = (size_t(tk.page) * H + tk.h) * P * dh;
                    mbar_arrive_expect_tx(&mbar[slot], 2 * bytes);
                    bulk_g2s(kb, Lw.kp + off, bytes, &mbar[slot]);
                    bulk_g2s(kb + size_t(P) * dh, Lw.vp + off, bytes, &mbar[slot]);
                };
                if (tid == 0) {
                    // K/V rows were written by generic stores of other CTAs
                    // (ordered by the grid barrier); the copies read them
                    // through the async proxy
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    for (int i = 0; i < kNBuf; ++i) issue(i);
                }
                const int chunk = dh / 4;
                for (int i = 0, u = blockIdx.x; u < total; ++i, u += gridDim.x) {
                    const Task tk = task_of(u);
                    const int slot = i % kNBuf, nk = tk.nk;
                    float* part = a.part + (size_t(tk.b * H + tk.h) * a.max_chunks + tk.c) * (dh + 2);
                    if (nk == 0) {
                        if (tid == 0) {
                            part[0] = -INFINITY;
                            part[1] = 0.f;
                            issue(i + kNBuf);
                        }
                        continue;
                    }
                    for (int e = tid; e < dh; e += kPThreads) qh[e] = __ldcg(a.q + size_t(tk.b) * D + tk.h * dh + e);
                    mbar_wait(&mbar[slot], (mb_phase >> slot) & 1u);
                    mb_phase ^= 1u << slot;
                    __syncthreads();
                    const float* ks = kvbuf + size_t(slot) * 2 * P * dh;
                    const float* vs = ks + size_t(P) * dh;
                    // scores: thread = (key tid / 4, quarter of d_head); the
                    // quarter's dimensions are rotated by the key (bank spread)
                    {
                        const int j = tid >> 2, qq = tid & 3;
                        float dot = 0.f;
                        if (j < nk) {
                            const float* kr = ks + size_t(j) * dh + qq * chunk;
                            const float* qr = qh + qq * chunk;
                            for (int d0 = 0; d0 < chunk; ++d0) {
                                const int dd = (d0 + j) & (chunk - 1);
                                dot = fmaf(qr[dd], kr[dd], dot);
                            }
                        }
                        dot += __shfl_xor_sync(0xffffffffu, dot, 1);
                        dot += __shfl_xor_sync(0xffffffffu, dot, 2);
                        if (qq == 0 && j < 64) ps[j] = j < nk ? dot * scale : -INFINITY;
                    }
                    __syncthreads();
                    if (warp == 0) {
                        const float s0 = ps[lane], s1v = ps[lane + 32];
                        const float m = warp_max(fmaxf(s0, s1v));
                        const float p0 = lane < nk ? __expf(s0 - m) : 0.f;
                        const float p1 = lane + 32 < nk ? __expf(s1v - m) : 0.f;
                        ps[lane] = p0;
                        ps[lane + 32] = p1;
                        const float lsum = warp_sum(p0 + p1);
                        if (lane == 0) {
                            rr[0] = m;
                            rr[1] = lsum;
                        }
                    }
                    __syncthreads();
                    // PV: thread = (dimension e, key group g); groups added in order
                    const int ng = kPThreads / dh;
                    {
                        const int e = tid % dh, g = tid / dh;
                        float o = 0.f;
                        for (int j = g; j < nk; j += ng) o = fmaf(ps[j], vs[size_t(j) * dh + e], o);
                        po[g * 128 + e] = o;
                    }
                    __syncthreads();
                    for (int e = tid; e < dh; e += kPThreads) {
                        float o = 0.f;
                        for (int gg = 0; gg < ng; ++gg) o += po[gg * 128 + e];
                        part[2 + e] = o;
                    }
                    if (tid == 0) {
                        part[0] = rr[0];
                        part[1] = rr[1];
                        issue(i + kNBuf);  // the buffer is free again (all reads done above)
                    }
                }
                __syncthreads();
            }
            sync(t);

            // ---- LSE merge of the partials (every CTA, all rows) + Wo + residual ----
            {
                float* wts = s_att;  // [B * H][max_chunks]
                for (int bh = warp; bh < B * H; bh += kPWarps) {
                    const int b = bh / H;
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const float* base = a.part + size_t(bh) * a.max_chunks * (dh + 2);
                    float M = -INFINITY;
                    for (int c = lane; c < npg; c += 32) M = fmaxf(M, __ldcg(base + size_t(c) * (dh + 2)));
                    M = warp_max(M);
                    float Ls = 0.f;
                    for (int c = lane; c < npg; c += 32) {  // L1 hits: the maxima were just read
                        const float m = base[size_t(c) * (dh + 2)];
                        const float wgt = m == -INFINITY ? 0.f : __expf(m - M);
                        wts[bh * a.max_chunks + c] = wgt;
                        Ls += wgt * base[size_t(c) * (dh + 2) + 1];
                    }
                    Ls = warp_sum(Ls);
                    for (int c = lane; c < npg; c += 32) wts[bh * a.max_chunks + c] /= Ls;
                }
                __syncthreads();
                for (int i = tid; i < B * D; i += kPThreads) {
                    const int b = i / D, cc = i - b * D, h = cc / dh, e = cc - h * dh;
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const float* base = a.part + size_t(b * H + h) * a.max_chunks * (dh + 2) + 2 + e;
                    const float* wr = wts + (b * H + h) * a.max_chunks;
                    float o = 0.f;
#pragma unroll 8
                    for (int c = 0; c < npg; ++c) o = fmaf(wr[c], __ldcg(base + size_t(c) * (dh + 2)), o);
                    xs[i] = o;
                }
            }
            __syncthreads();
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

        // ---- unembed_logits (model.cpp:238-246) ----
        load_rows(a.x, B * D, xs);
        __syncthreads();
        ln_smem(xs, B, D);
        __syncthreads();
        gemv_cols(xs, su.ws, B, D, su.ncp, su.c0, su.nc, red,
                  [&](int b, int c, float v) { a.logits[size_t(b) * V + c] = v; });

        // ---- argmax_token (model.cpp:248-255) by the last CTA to finish ----
        __shared__ int s_last;
        if (tid == 0) {
            __threadfence();
            s_last = atomicAdd(arrive, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (s_last) {
            __threadfence();
            for (int b = warp; b < B; b += kPWarps) {
                float bv = 0.f;
                int bi = V;
                for (int c = lane; c < V; c += 32) {
                    const float v = __ldcg(a.logits + size_t(b) * V + c);
                    if (bi == V || v > bv) {
                        bv = v;
                        bi = c;
                    }
                }
#pragma unroll
                for (int msk = 16; msk > 0; msk >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, bv, msk);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, msk);
                    if (oi < V && (bi == V || ov > bv || (ov == bv && oi < bi))) {
                        bv = ov;
                        bi = oi;
                    }
                }
                if (lane == 0) a.out[size_t(t) * B + b] = bi == V ? 0 : bi;
            }
            if (tid == 0) *arrive = 0;
        }
        sync(t);
    }
}

}  // namespace

bool persist_supported(int L, int B, int D, int H, int F, int V, int P, int n_sms) {
    const int dh = D / H;
    if (L < 1 || L > 8 || B < 1 || B > kMaxB || D % 4 || F % 4 || P > 64 || n_sms < 1) return false;
    if (dh != 32 && dh != 64 && dh != 128) return false;  // power-of-two quarters, 256 / dh key groups
    if (stage_ncp(std::max(std::max(3 * D, F), V), n_sms) > kMaxNcp) return false;
    return persist_smem_bytes(L, B, D, F, H, V, 1, n_sms) <= 200 * 1024;
}

size_t persist_smem_bytes(int L, int B, int D, int F, int H, int V, int max_chunks, int n_sms) {
    const int Kmax = F > D ? F : D;
    const int dh = D / H, P = 64;
    return sizeof(float) * (resident_floats(L, D, F, V, n_sms) + size_t(B) * Kmax +
                            pad4(size_t(B) * stage_ncp(D, n_sms)) + scratch_floats(B, H, max_chunks) +
                            att_buf_floats(P, dh));
}

cudaError_t launch_decode_persist(const PersistArgs& a, int n_ctas, cudaStream_t s) {
    const size_t smem = persist_smem_bytes(a.L, a.B, a.D, a.F, a.H, a.V, a.max_chunks, n_ctas);
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem<decode_persist_kernel>(int(smem))) return e;
    if (cudaError_t e = cudaMemsetAsync(a.counters, 0, 2 * sizeof(int32_t), s)) return e;
    void* args[] = {const_cast<PersistArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(decode_persist_kernel), dim3(n_ctas),
                                       dim3(kPThreads), args, smem, s);
}

}  // namespace ep
