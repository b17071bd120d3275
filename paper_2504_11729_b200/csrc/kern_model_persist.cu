// kern_model_persist.cu — K9: a whole greedy rollout of a small decoder in ONE
// persistent cooperative kernel (decode_greedy, model.cpp:285-297, for the
// BASELINE config-1 class of models: fp32, a few rows).
//
// The CUDA-graph rollout of ep_model_generate replays ~11 kernels per token;
// for config 1 (d_model 256, 2 layers) every kernel is a few microseconds of
// launch, fill and drain around well under a microsecond of L2-resident work.
// Here one CTA per SM stays resident for all n_steps tokens and the layer's
// stages are separated by grid-wide barriers instead of kernel boundaries:
//
//   per step:  [LN + Q|K|V, K/V rows -> pages]  (layer 0: embedding fused)
//              [attention partials: one (row, head, page) task per CTA]
//              [LSE merge of the partials + Wo + residual]
//              [LN + W1 + b1 + ReLU]
//              [W2 + b2 + residual]                         x n_layers
//              [LN + unembedding]  [argmax -> token of the next step]
//
// Every stage is latency-bound (a few MB of L2-resident weights, 1-8 rows),
// so work is cut for parallelism: a GEMV is split into (32-column block,
// 32-row k-chunk) warp tasks over the whole grid — each lane keeps its 32
// weight loads in flight — and the last k-chunk of a column block to finish
// (an arrival counter) adds the chunks' partial sums in chunk order
// (deterministic) and applies the epilogue. Input rows sit in shared memory
// with the LayerNorm applied (model.cpp:131-150). Attention is
// partial_attention per 64-key page with the causal rule (keys at positions
// <= the query, attention.cpp:29-33, :80-114), merged by LSE
// (attention.cpp:116-145).
#include <algorithm>
#include <cmath>
#include <cstdint>

#include <cooperative_groups.h>

#include "ep_common.cuh"
#include "model_internal.h"

namespace ep {
namespace {

namespace cg = cooperative_groups;

constexpr int kPThreads = 256;
constexpr int kPWarps = kPThreads / 32;
constexpr float kEps = 1e-5f;  // model.cpp:14

// LayerNorm of B rows of width D from global `x` into xs[B][D].
__device__ void ln_rows(const float* x, int B, int D, float* xs) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = warp; b < B; b += kPWarps) {
        const float* xr = x + size_t(b) * D;
        float s = 0.f;
        for (int c = lane; c < D; c += 32) s += __ldcg(xr + c);
        const float mean = warp_sum(s) / float(D);
        float q = 0.f;
        for (int c = lane; c < D; c += 32) {
            const float d = __ldcg(xr + c) - mean;
            q += d * d;
        }
        const float inv = 1.f / sqrtf(warp_sum(q) / float(D) + kEps);
        for (int c = lane; c < D; c += 32) xs[size_t(b) * D + c] = (__ldcg(xr + c) - mean) * inv;
    }
}

// Tasks of a GEMV y[B][N] = xs[B][K] @ W: (column block cb, k-chunk kc).
__device__ __forceinline__ int gemv_tasks(int K, int n_blocks) { return n_blocks * (K / 32); }

// Whether this CTA holds any task of the stage (it then needs xs).
__device__ __forceinline__ bool cta_has_tasks(int tasks) { return int(blockIdx.x) * kPWarps < tasks; }

// wsel(cb, W, col, ld): block cb is columns [col, col + 32) of the row-major
// [K][ld] matrix W. epi(b, cb, lane, value) for b < B, run by the last chunk.
template <typename WSel, typename Epi>
__device__ void gemv_stage(const float* xs, int B, int K, int n_blocks, float* gpart, int32_t* counters,
                           WSel wsel, Epi epi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_kc = K / 32, total = n_blocks * n_kc, N = n_blocks * 32;
    for (int task = blockIdx.x * kPWarps + warp; task < total; task += gridDim.x * kPWarps) {
        const int cb = task / n_kc, kc = task - cb * n_kc;
        const float* W;
        int col, ld;
        wsel(cb, W, col, ld);
        const float* wp = W + size_t(kc) * 32 * ld + col + lane;
        float w[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) w[i] = __ldg(wp + size_t(i) * ld);
        float acc[8];
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            acc[b] = 0.f;
            if (b < B) {
                const float* xr = xs + size_t(b) * K + kc * 32;
#pragma unroll
                for (int i = 0; i < 32; ++i) acc[b] = fmaf(xr[i], w[i], acc[b]);
            }
        }
        if (n_kc == 1) {
            for (int b = 0; b < B; ++b) epi(b, cb, lane, acc[b]);
            continue;
        }
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (b < B) __stcg(gpart + (size_t(kc) * B + b) * N + cb * 32 + lane, acc[b]);
        __threadfence();
        __syncwarp();
        int last = 0;
        if (lane == 0) last = atomicAdd(&counters[cb], 1) == n_kc - 1;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
            __threadfence();
            for (int b = 0; b < B; ++b) {
                // chunk partials: loads 8 at a time in flight, added in chunk order
                float v = 0.f;
                for (int k0 = 0; k0 < n_kc; k0 += 8) {
                    float pv[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        pv[i] = k0 + i < n_kc ? __ldcg(gpart + (size_t(k0 + i) * B + b) * N + cb * 32 + lane) : 0.f;
#pragma unroll
                    for (int i = 0; i < 8; ++i) v += pv[i];
                }
                epi(b, cb, lane, v);
            }
            if (lane == 0) counters[cb] = 0;  // ready for the next stage
        }
    }
}

__global__ void __launch_bounds__(kPThreads, 1) decode_persist_kernel(const PersistArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) float smem_f[];
    const int B = a.B, D = a.D, H = a.H, dh = a.dh, F = a.F, V = a.V, P = a.P;
    const int Kmax = F > D ? F : D;
    float* xs = smem_f;                        // [B][K] GEMV input rows
    float* s_att = smem_f + size_t(B) * Kmax;  // attention scratch (see below)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const float scale = 1.f / sqrtf(float(dh));
    int n_sync = 0;
    // debug (a.trace): CTA 0 stamps the globaltimer after every grid barrier
    auto gsync = [&](int t) {
        grid.sync();
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 8) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            a.trace[t * 32 + (n_sync & 31)] = ts;
        }
        ++n_sync;
    };

    for (int t = 0; t < a.n_steps; ++t) {
        n_sync = 0;
        if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && t < 8) {
            unsigned long long ts;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
            a.trace[t * 32 + 31] = ts;
        }
        for (int l = 0; l < a.L; ++l) {
            const PersistLayer& Lw = a.layers[l];
            // ---- LN(x) -> Q | K | V; layer 0 embeds the step's tokens first ----
            const int qkv_tasks = gemv_tasks(D, 3 * (D / 32));
            if (l == 0) {
                // model.cpp:104-129 with the fp64 sinusoid table; CTA 0 also
                // stores the embedded rows (the residual input)
                if (cta_has_tasks(qkv_tasks) || blockIdx.x == 0) {
                    for (int i = tid; i < B * D; i += kPThreads) {
                        const int b = i / D, c = i - b * D;
                        const int tok = t == 0 ? a.first[b] : __ldcg(a.out + size_t(t - 1) * B + b);
                        const int pos = a.pos[size_t(t) * B + b];
                        const float v = float(double(a.emb[size_t(tok) * D + c]) + a.pe[size_t(pos) * D + c]);
                        xs[i] = v;
                        if (blockIdx.x == 0) a.x[i] = v;
                    }
                    __syncthreads();
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
            } else if (cta_has_tasks(qkv_tasks)) {
                ln_rows(a.x, B, D, xs);
            }
            __syncthreads();
            gemv_stage(
                xs, B, D, 3 * (D / 32), a.gpart, a.counters,
                [&](int cb, const float*& W, int& col, int& ld) {
                    const int which = cb / (D / 32);
                    W = which == 0 ? Lw.wq : which == 1 ? Lw.wk : Lw.wv;
                    col = (cb - which * (D / 32)) * 32;
                    ld = D;
                },
                [&](int b, int cb, int ln, float v) {
                    const int which = cb / (D / 32);
                    const int cc = (cb - which * (D / 32)) * 32 + ln;
                    if (which == 0) {
                        a.q[size_t(b) * D + cc] = v;
                    } else {
                        const int h = cc / dh, e = cc - h * dh;
                        const size_t idx = ((size_t(a.dst_page[size_t(t) * B + b]) * H + h) * P +
                                            a.dst_slot[size_t(t) * B + b]) * dh + e;
                        (which == 1 ? Lw.kp : Lw.vp)[idx] = v;
                    }
                });
            gsync(t);

            // ---- attention partials: one (row, head, page) task per CTA ----
            {
                int total = 0;
                for (int b = 0; b < B; ++b) total += H * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                float* qh = s_att;        // [128]
                float* ps = s_att + 128;  // [64] scores, then probabilities
                float* po = s_att + 192;  // [4][128] PV partials of the key groups
                float* rr = s_att + 704;  // [2] max, sum
                for (int u = blockIdx.x; u < total; u += gridDim.x) {
                    int b = 0, rem = u;
                    while (rem >= H * int(a.req_page_off[b + 1] - a.req_page_off[b])) {
                        rem -= H * int(a.req_page_off[b + 1] - a.req_page_off[b]);
                        ++b;
                    }
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const int h = rem / npg, c = rem - h * npg;
                    const PageDesc d = a.pdesc[a.req_page_off[b] + c];
                    const int64_t qpos = a.pos[size_t(t) * B + b];
                    const int64_t vis = qpos - d.pos + 1;
                    const int nk = vis <= 0 ? 0 : (vis < d.n_tok ? int(vis) : d.n_tok);
                    float* part = a.part + (size_t(b * H + h) * a.max_chunks + c) * (dh + 2);
                    if (nk == 0) {
                        if (tid == 0) {
                            part[0] = -INFINITY;
                            part[1] = 0.f;
                        }
                        continue;
                    }
                    for (int e = tid; e < dh; e += kPThreads) qh[e] = __ldcg(a.q + size_t(b) * D + h * dh + e);
                    __syncthreads();
                    const float* kt = Lw.kp + (size_t(d.page) * H + h) * P * dh;
                    const float* vt = Lw.vp + (size_t(d.page) * H + h) * P * dh;
                    // scores: warp w takes keys w, w + 8, ...; lanes split d_head;
                    // all of the warp's key loads are in flight before the sums
                    {
                        float kv[8][4];
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int j = warp + i * kPWarps;
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const int e = lane + 32 * r;
                                kv[i][r] = (j < nk && e < dh) ? __ldcg(kt + size_t(j) * dh + e) : 0.f;
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int j = warp + i * kPWarps;
                            float dot = 0.f;
#pragma unroll
                            for (int r = 0; r < 4; ++r) {
                                const int e = lane + 32 * r;
                                if (e < dh) dot = fmaf(qh[e], kv[i][r], dot);
                            }
                            dot = warp_sum(dot);
                            if (lane == 0 && j < 64) ps[j] = j < nk ? dot * scale : -INFINITY;
                        }
                    }
                    __syncthreads();
                    if (warp == 0) {
                        const float s0 = ps[lane], s1 = ps[lane + 32];
                        const float m = warp_max(fmaxf(s0, s1));
                        const float p0 = lane < nk ? __expf(s0 - m) : 0.f;
                        const float p1 = lane + 32 < nk ? __expf(s1 - m) : 0.f;
                        ps[lane] = p0;
                        ps[lane + 32] = p1;
                        const float l = warp_sum(p0 + p1);
                        if (lane == 0) {
                            rr[0] = m;
                            rr[1] = l;
                        }
                    }
                    __syncthreads();
                    // PV: thread = (dimension e, key group g); groups added in order
                    const int ng = kPThreads / dh < 4 ? kPThreads / dh : 4;
                    const int e = tid % dh, g = tid / dh;
                    if (g < ng) {
                        float o = 0.f;
#pragma unroll 4
                        for (int j = g; j < nk; j += ng) o = fmaf(ps[j], __ldcg(vt + size_t(j) * dh + e), o);
                        po[g * 128 + e] = o;
                    }
                    __syncthreads();
                    for (int i = tid; i < dh; i += kPThreads) {
                        float o = 0.f;
                        for (int gg = 0; gg < ng; ++gg) o += po[gg * 128 + i];
                        part[2 + i] = o;
                    }
                    if (tid == 0) {
                        part[0] = rr[0];
                        part[1] = rr[1];
                    }
                    __syncthreads();
                }
            }
            gsync(t);

            // ---- LSE merge of the partials + Wo + residual ----
            if (cta_has_tasks(gemv_tasks(D, D / 32))) {
                // weights of each (row, head)'s page partials: a warp per (b, h)
                float* wts = s_att;  // [B * H][max_chunks]
                for (int bh = warp; bh < B * H; bh += kPWarps) {
                    const int b = bh / H;
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const float* base = a.part + size_t(bh) * a.max_chunks * (dh + 2);
                    float M = -INFINITY;
                    for (int c = lane; c < npg; c += 32) M = fmaxf(M, __ldcg(base + size_t(c) * (dh + 2)));
                    M = warp_max(M);
                    float L = 0.f;
                    for (int c = lane; c < npg; c += 32) {
                        const float m = __ldcg(base + size_t(c) * (dh + 2));
                        const float wgt = m == -INFINITY ? 0.f : __expf(m - M);
                        wts[bh * a.max_chunks + c] = wgt;
                        L += wgt * __ldcg(base + size_t(c) * (dh + 2) + 1);
                    }
                    L = warp_sum(L);
                    for (int c = lane; c < npg; c += 32) wts[bh * a.max_chunks + c] /= L;
                }
                __syncthreads();
                for (int i = tid; i < B * D; i += kPThreads) {
                    const int b = i / D, cc = i - b * D, h = cc / dh, e = cc - h * dh;
                    const int npg = int(a.req_page_off[b + 1] - a.req_page_off[b]);
                    const float* base = a.part + size_t(b * H + h) * a.max_chunks * (dh + 2) + 2 + e;
                    const float* wr = wts + (b * H + h) * a.max_chunks;
                    float o = 0.f;
#pragma unroll 4
                    for (int c = 0; c < npg; ++c) o = fmaf(wr[c], __ldcg(base + size_t(c) * (dh + 2)), o);
                    xs[i] = o;
                }
            }
            __syncthreads();
            gemv_stage(
                xs, B, D, D / 32, a.gpart, a.counters,
                [&](int cb, const float*& W, int& col, int& ld) {
                    W = Lw.wo;
                    col = cb * 32;
                    ld = D;
                },
                [&](int b, int cb, int ln, float v) {
                    const int c = cb * 32 + ln;
                    a.x2[size_t(b) * D + c] = __ldcg(a.x + size_t(b) * D + c) + v;  // model.cpp:184-185
                });
            gsync(t);

            // ---- LN(x2) -> W1 + b1 -> ReLU ----
            if (cta_has_tasks(gemv_tasks(D, F / 32))) ln_rows(a.x2, B, D, xs);
            __syncthreads();
            gemv_stage(
                xs, B, D, F / 32, a.gpart, a.counters,
                [&](int cb, const float*& W, int& col, int& ld) {
                    W = Lw.w1;
                    col = cb * 32;
                    ld = F;
                },
                [&](int b, int cb, int ln, float v) {
                    const int c = cb * 32 + ln;
                    float h1 = v + Lw.b1[c];  // model.cpp:188-194
                    if (h1 < 0.f) h1 = 0.f;
                    a.h1[size_t(b) * F + c] = h1;
                });
            gsync(t);

            // ---- W2 + b2 + residual ----
            if (cta_has_tasks(gemv_tasks(F, D / 32)))
                for (int i = tid; i < B * F; i += kPThreads) xs[i] = __ldcg(a.h1 + i);
            __syncthreads();
            gemv_stage(
                xs, B, F, D / 32, a.gpart, a.counters,
                [&](int cb, const float*& W, int& col, int& ld) {
                    W = Lw.w2;
                    col = cb * 32;
                    ld = D;
                },
                [&](int b, int cb, int ln, float v) {
                    const int c = cb * 32 + ln;
                    a.x[size_t(b) * D + c] = (__ldcg(a.x2 + size_t(b) * D + c) + v) + Lw.b2[c];  // model.cpp:199-204
                });
            gsync(t);
        }

        // ---- unembed_logits (model.cpp:238-246) ----
        if (cta_has_tasks(gemv_tasks(D, V / 32))) ln_rows(a.x, B, D, xs);
        __syncthreads();
        gemv_stage(
            xs, B, D, V / 32, a.gpart, a.counters,
            [&](int cb, const float*& W, int& col, int& ld) {
                W = a.unembed;
                col = cb * 32;
                ld = V;
            },
            [&](int b, int cb, int ln, float v) { a.logits[size_t(b) * V + cb * 32 + ln] = v; });
        gsync(t);

        // ---- argmax_token (model.cpp:248-255): the next step's token ----
        if (blockIdx.x == 0) {
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
        }
        gsync(t);
    }
}

}  // namespace

bool persist_supported(int B, int D, int H, int F, int V, int P) {
    const int dh = D / H;
    return B >= 1 && B <= 8 && D % 32 == 0 && F % 32 == 0 && V % 32 == 0 && dh <= 128 && P <= 64;
}

size_t persist_smem_bytes(int B, int D, int F, int H, int max_chunks) {
    const int Kmax = F > D ? F : D;
    const size_t att = std::max<size_t>(712, size_t(B) * H * max_chunks);
    return sizeof(float) * (size_t(B) * Kmax + att);
}

size_t persist_gpart_floats(int B, int D, int F, int V) {
    const int Kmax = F > D ? F : D, Nmax = std::max(std::max(3 * D, F), V);
    return size_t(Kmax / 32) * B * Nmax;
}

cudaError_t launch_decode_persist(const PersistArgs& a, int n_ctas, cudaStream_t s) {
    const size_t smem = persist_smem_bytes(a.B, a.D, a.F, a.H, a.max_chunks);
    if (smem > 48 * 1024)
        if (cudaError_t e = ensure_smem<decode_persist_kernel>(int(smem))) return e;
    void* args[] = {const_cast<PersistArgs*>(&a)};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(decode_persist_kernel), dim3(n_ctas),
                                       dim3(kPThreads), args, smem, s);
}

}  // namespace ep
