// kern_peer.cu — cross-GPU split-KV combine over NVLink peer memory
// (BASELINE config 4).
//
// The reference merges any ordered partition of a row's keys with
// merge_partials (/root/reference/proj/core/src/attention.cpp:116-156). With
// the partition across the GPUs of one box, every rank holds the fp32
// (o, lse) of its KV shard; this ONE kernel (per rank) replaces
// all-gather + merge. CTA c of every rank owns the same row slice:
//
//   1. push: the slice's o rows and lse go into every peer's receive buffer
//      as 16-byte {value, flag, value, flag} words (flag = step epoch) with
//      plain volatile stores over NVLink — a low-latency "data carries its
//      own flag" protocol: no fences, no separate flag round trip;
//   2. merge: one warp per row polls the peers' words of its row until both
//      flags equal the epoch, then folds the W partials in rank (= KV
//      segment) order — bit-identical on every rank.
//
// Receive buffers are double-buffered by epoch parity: a rank pushes step
// s+2 into the buffer it pushed step s into only after its own step s+1
// combine received the peers' step s+1 words, which each peer sends only
// after its step s combine (and its reads of our step s words) retired.
// Each CTA keeps its own epoch counter (read at entry, written at exit), so
// the launch has fixed arguments (CUDA-graph capturable), no atomics, no
// host round trip. Spins are bounded (globaltimer, 20 s) and trap instead of
// hanging the GPU when a peer never arrives.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>

#include "ep_common.cuh"
#include "ep_internal.h"

namespace ep {
namespace {

constexpr int kMaxWorld = 8;
constexpr int kPeerThreads = 256;
constexpr int kMaxSlices = 128;
constexpr int kMaxUnitsPerLane = 5;  // (d/2 + 1) <= 32 * 5  for d <= 256

struct PeerArgs {
    int32_t world, rank, rows, d, nslices, rows_max;
    int64_t src_units;       // 16-byte words per source slot: rows_max * (d/2 + 1)
    const float* o_local;    // [rows][d]
    const float* lse_local;  // [rows] natural log
    uint4* recv[kMaxWorld];  // peer p's receive area [2][world][src_units] (mapped here)
    const uint4* my_recv;    // own receive area
    uint32_t* epoch;         // own [nslices], one per CTA
    void* out;
    int32_t out_dtype;
    float* out_lse;
    unsigned long long* trace;  // debug (EP_PEER_TRACE): CTA 0 phase timestamps, [64][8]
};

__global__ void __launch_bounds__(kPeerThreads) splitkv_combine_kernel(const PeerArgs a) {
    const int c = blockIdx.x;
    const int tid = threadIdx.x;
    const int W = a.world, me = a.rank, D = a.d, H = D / 2;  // H data words per row, + 1 lse word
    const int rps = (a.rows + a.nslices - 1) / a.nslices;
    const int r0 = min(a.rows, c * rps), r1 = min(a.rows, r0 + rps);
    const uint32_t ep = a.epoch[c] + 1u;
    const size_t par_off = size_t(ep & 1u) * W * a.src_units;
    unsigned long long* tr = (a.trace && c == 0 && tid == 0) ? a.trace + (ep & 63u) * 8 : nullptr;
    if (tr) tr[0] = globaltimer();

    // 1. push rows [r0, r1) into slot [me] of every peer's buffer (parity ep&1)
    const int units = (r1 - r0) * (H + 1);
    for (int u = tid; u < units; u += kPeerThreads) {
        const int r = r0 + u / (H + 1), k = u % (H + 1);
        float2 v;
        if (k < H) v = __ldcg(reinterpret_cast<const float2*>(a.o_local + size_t(r) * D) + k);
        else v = make_float2(__ldcg(a.lse_local + r), 0.f);
        const size_t off = par_off + size_t(me) * a.src_units + size_t(r) * (H + 1) + k;
        for (int p = 0; p < W; ++p)
            if (p != me) st_ll(a.recv[p] + off, v.x, v.y, ep);
    }
    if (tr) tr[1] = globaltimer();

    // 2. merge, one warp per row: lane owns words lane, lane+32, ... of the row
    const int warp = tid >> 5, lane = tid & 31;
    for (int r = r0 + warp; r < r1; r += kPeerThreads / 32) {
        float lse_p[kMaxWorld];
        float M = -INFINITY;
        for (int p = 0; p < W; ++p) {
            float l;
            if (p == me) {
                l = __ldcg(a.lse_local + r);
            } else {
                float2 x = make_float2(0.f, 0.f);
                if (lane == 0)
                    x = ld_ll(a.my_recv + par_off + size_t(p) * a.src_units + size_t(r) * (H + 1) + H, ep);
                l = __shfl_sync(0xffffffffu, x.x, 0);
            }
            lse_p[p] = l;
            M = fmaxf(M, l);
        }
        float2 acc[kMaxUnitsPerLane];
#pragma unroll
        for (int i = 0; i < kMaxUnitsPerLane; ++i) acc[i] = make_float2(0.f, 0.f);
        float L = 0.f;
        for (int p = 0; p < W; ++p) {
            const float wt = (M == -INFINITY || lse_p[p] == -INFINITY) ? 0.f : expf(lse_p[p] - M);
            L += wt;
            const uint4* src = a.my_recv + par_off + size_t(p) * a.src_units + size_t(r) * (H + 1);
            const float2* loc = reinterpret_cast<const float2*>(a.o_local + size_t(r) * D);
#pragma unroll
            for (int i = 0; i < kMaxUnitsPerLane; ++i) {
                const int k = lane + 32 * i;
                if (k < H) {
                    // peers' words are always consumed (they carry the flag)
                    const float2 x = p == me ? __ldcg(loc + k) : ld_ll(src + k, ep);
                    acc[i].x += wt * x.x;
                    acc[i].y += wt * x.y;
                }
            }
        }
        const float inv = L > 0.f ? 1.f / L : 0.f;
#pragma unroll
        for (int i = 0; i < kMaxUnitsPerLane; ++i) {
            const int k = lane + 32 * i;
            if (k >= H) continue;
            if (a.out_dtype == EP_BF16) {
                reinterpret_cast<__nv_bfloat162*>(a.out)[size_t(r) * H + k] =
                    __floats2bfloat162_rn(acc[i].x * inv, acc[i].y * inv);
            } else {
                reinterpret_cast<float2*>(a.out)[size_t(r) * H + k] =
                    make_float2(acc[i].x * inv, acc[i].y * inv);
            }
        }
        if (lane == 0 && a.out_lse) a.out_lse[r] = L > 0.f ? M + logf(L) : -INFINITY;
    }
    if (tr) tr[2] = globaltimer();
    if (tid == 0) a.epoch[c] = ep;
}

}  // namespace
}  // namespace ep

struct ep_peer_group_s {
    ep_handle h = nullptr;
    int32_t world = 0, rank = 0, rows_max = 0, d = 0, nslices = 0;
    void* base = nullptr;       // own allocation
    size_t bytes = 0;
    void* peer[ep::kMaxWorld] = {};
    bool peer_is_ipc[ep::kMaxWorld] = {};
    bool connected = false;
    unsigned long long* trace = nullptr;  // EP_PEER_TRACE=1: [64][8] device timestamps
    int mode = 0;  // 0 unused, 1 combine kernel (ep_splitkv_combine_dev), 2 fused K1 (ep_spliced_attention_splitkv)
    // per source rank: rows_max rows of d/2 {value, flag} data words + 1 lse word
    size_t src_units() const { return size_t(rows_max) * (d / 2 + 1); }
    size_t recv_bytes() const { return size_t(2) * world * src_units() * 16; }
    size_t epoch_off() const { return (recv_bytes() + 255) & ~size_t(255); }
    // fused mode: one epoch per (request, kv-head) unit (<= rows_max units)
    size_t unit_epoch_off() const { return (epoch_off() + size_t(nslices) * sizeof(uint32_t) + 255) & ~size_t(255); }
    ~ep_peer_group_s() {
        if (h) cudaSetDevice(h->device);
        for (int p = 0; p < world; ++p)
            if (peer[p] && peer_is_ipc[p]) cudaIpcCloseMemHandle(peer[p]);
        if (trace) {
            if (const char* f = std::getenv("EP_PEER_TRACE_FILE")) {
                unsigned long long hbuf[64 * 8];
                if (cudaMemcpy(hbuf, trace, sizeof(hbuf), cudaMemcpyDeviceToHost) == cudaSuccess) {
                    std::string path = std::string(f) + "." + std::to_string(rank);
                    if (FILE* fp = std::fopen(path.c_str(), "wb")) {
                        std::fwrite(hbuf, sizeof(hbuf), 1, fp);
                        std::fclose(fp);
                    }
                }
            }
            cudaFree(trace);
        }
        if (base) cudaFree(base);
    }
};

using ep::fail;

namespace ep {
int peer_link_fill(ep_peer_group g, int64_t n_units, int64_t rows, int d, const int32_t* cta_unit_ptr,
                   PeerLink* out) {
    if (!g->connected && g->world > 1) return fail(EP_EINVAL, "ep_spliced_attention_splitkv: group not connected");
    if (g->mode == 1)
        return fail(EP_EINVAL, "ep_spliced_attention_splitkv: group is used by ep_splitkv_combine_dev "
                               "(one combine protocol per group)");
    if (d != g->d) return fail(EP_EINVAL, "ep_spliced_attention_splitkv: group d != the plan's d_head");
    if (rows > g->rows_max || n_units > g->rows_max)
        return fail(EP_EINVAL, "ep_spliced_attention_splitkv: plan rows " + std::to_string(rows) +
                                   " exceed the group's rows_max " + std::to_string(g->rows_max));
    g->mode = 2;
    PeerLink l{};
    l.world = g->world;
    l.rank = g->rank;
    l.src_units = int64_t(g->src_units());
    for (int p = 0; p < g->world; ++p) l.recv[p] = static_cast<uint4*>(g->peer[p]);
    l.epoch = reinterpret_cast<uint32_t*>(static_cast<char*>(g->base) + g->unit_epoch_off());
    l.cta_unit_ptr = cta_unit_ptr;
    *out = l;
    return EP_OK;
}
}  // namespace ep

extern "C" {

int ep_peer_group_create(ep_handle h, int32_t world, int32_t rank, int32_t rows_max, int32_t d,
                         ep_peer_group* out) {
    if (!h || !out) return fail(EP_EINVAL, "ep_peer_group_create: null argument");
    *out = nullptr;
    if (world < 1 || world > ep::kMaxWorld || rank < 0 || rank >= world)
        return fail(EP_EINVAL, "ep_peer_group_create: world must be 1..8 and 0 <= rank < world");
    if (rows_max <= 0 || d <= 0 || d > 256 || d % 2)
        return fail(EP_EINVAL, "ep_peer_group_create: rows_max > 0 and d even, 2 <= d <= 256");
    std::unique_ptr<ep_peer_group_s> g(new (std::nothrow) ep_peer_group_s());
    if (!g) return fail(EP_ENOMEM, "ep_peer_group_create");
    g->h = h;
    g->world = world;
    g->rank = rank;
    g->rows_max = rows_max;
    g->d = d;
    g->nslices = rows_max < ep::kMaxSlices ? rows_max : ep::kMaxSlices;
    g->bytes = g->unit_epoch_off() + size_t(rows_max) * sizeof(uint32_t);
    EP_CUDA_TRY(cudaSetDevice(h->device), "ep_peer_group_create");
    EP_CUDA_TRY(cudaMalloc(&g->base, g->bytes), "ep_peer_group_create alloc");
    EP_CUDA_TRY(cudaMemset(g->base, 0, g->bytes), "ep_peer_group_create memset");
    EP_CUDA_TRY(cudaDeviceSynchronize(), "ep_peer_group_create sync");
    g->peer[rank] = g->base;
    if (const char* t = std::getenv("EP_PEER_TRACE"); t && *t == '1') {
        EP_CUDA_TRY(cudaMalloc(&g->trace, 64 * 8 * sizeof(unsigned long long)), "ep_peer_group_create trace");
        EP_CUDA_TRY(cudaMemset(g->trace, 0, 64 * 8 * sizeof(unsigned long long)), "ep_peer_group_create trace");
    }
    *out = g.release();
    return EP_OK;
}

int ep_peer_group_export(ep_peer_group g, void* ipc_handle) {
    if (!g || !ipc_handle) return fail(EP_EINVAL, "ep_peer_group_export: null argument");
    static_assert(sizeof(cudaIpcMemHandle_t) == EP_IPC_HANDLE_BYTES, "ipc handle size");
    EP_CUDA_TRY(cudaSetDevice(g->h->device), "ep_peer_group_export");
    cudaIpcMemHandle_t hd;
    EP_CUDA_TRY(cudaIpcGetMemHandle(&hd, g->base), "ep_peer_group_export");
    std::memcpy(ipc_handle, &hd, sizeof(hd));
    return EP_OK;
}

int ep_peer_group_base(ep_peer_group g, void** base) {
    if (!g || !base) return fail(EP_EINVAL, "ep_peer_group_base: null argument");
    *base = g->base;
    return EP_OK;
}

int ep_peer_group_connect_ipc(ep_peer_group g, const void* handles) {
    if (!g || !handles) return fail(EP_EINVAL, "ep_peer_group_connect_ipc: null argument");
    if (g->connected) return fail(EP_EINVAL, "ep_peer_group_connect_ipc: already connected");
    EP_CUDA_TRY(cudaSetDevice(g->h->device), "ep_peer_group_connect_ipc");
    for (int p = 0; p < g->world; ++p) {
        if (p == g->rank) continue;
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, static_cast<const char*>(handles) + size_t(p) * EP_IPC_HANDLE_BYTES, sizeof(hd));
        EP_CUDA_TRY(cudaIpcOpenMemHandle(&g->peer[p], hd, cudaIpcMemLazyEnablePeerAccess),
                    "ep_peer_group_connect_ipc open");
        g->peer_is_ipc[p] = true;
    }
    g->connected = true;
    return EP_OK;
}

int ep_peer_group_connect_ptrs(ep_peer_group g, void* const* bases) {
    if (!g || !bases) return fail(EP_EINVAL, "ep_peer_group_connect_ptrs: null argument");
    if (g->connected) return fail(EP_EINVAL, "ep_peer_group_connect_ptrs: already connected");
    EP_CUDA_TRY(cudaSetDevice(g->h->device), "ep_peer_group_connect_ptrs");
    for (int p = 0; p < g->world; ++p) {
        if (p == g->rank) continue;
        if (!bases[p]) return fail(EP_EINVAL, "ep_peer_group_connect_ptrs: null peer base");
        cudaPointerAttributes at{};
        EP_CUDA_TRY(cudaPointerGetAttributes(&at, bases[p]), "ep_peer_group_connect_ptrs attributes");
        if (at.type != cudaMemoryTypeDevice)
            return fail(EP_EINVAL, "ep_peer_group_connect_ptrs: peer base is not device memory");
        if (at.device != g->h->device) {
            int can = 0;
            EP_CUDA_TRY(cudaDeviceCanAccessPeer(&can, g->h->device, at.device), "ep_peer_group_connect_ptrs");
            if (!can) return fail(EP_EUNSUPPORTED, "ep_peer_group_connect_ptrs: no peer access between devices");
            const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return ep::cuda_fail(e, "ep_peer_group_connect_ptrs enable peer");
        }
        g->peer[p] = bases[p];
    }
    g->connected = true;
    return EP_OK;
}

int ep_splitkv_combine_dev(ep_handle h, ep_peer_group g, int32_t rows, const float* o_part,
                           const float* lse_part, int32_t out_dtype, void* out, float* out_lse,
                           ep_stream stream) {
    if (!h || !g || !o_part || !lse_part || !out)
        return fail(EP_EINVAL, "ep_splitkv_combine_dev: null argument");
    if (!g->connected && g->world > 1) return fail(EP_EINVAL, "ep_splitkv_combine_dev: group not connected");
    if (rows < 0 || rows > g->rows_max) return fail(EP_EINVAL, "ep_splitkv_combine_dev: rows > rows_max");
    if (g->mode == 2)
        return fail(EP_EINVAL, "ep_splitkv_combine_dev: group is used by ep_spliced_attention_splitkv "
                               "(one combine protocol per group)");
    g->mode = 1;
    if (out_dtype != EP_F32 && out_dtype != EP_BF16)
        return fail(EP_EUNSUPPORTED, "ep_splitkv_combine_dev: out dtype");
    if ((reinterpret_cast<uintptr_t>(o_part) & 7) != 0 || (reinterpret_cast<uintptr_t>(out) & 7) != 0)
        return fail(EP_EINVAL, "ep_splitkv_combine_dev: o_part and out must be 8-byte aligned");
    ep::PeerArgs a{};
    a.world = g->world;
    a.rank = g->rank;
    a.rows = rows;
    a.d = g->d;
    a.nslices = g->nslices;
    a.rows_max = g->rows_max;
    a.src_units = int64_t(g->src_units());
    a.o_local = o_part;
    a.lse_local = lse_part;
    for (int p = 0; p < g->world; ++p) a.recv[p] = static_cast<uint4*>(g->peer[p]);
    a.my_recv = static_cast<const uint4*>(g->base);
    a.epoch = reinterpret_cast<uint32_t*>(static_cast<char*>(g->base) + g->epoch_off());
    a.out = out;
    a.out_dtype = out_dtype;
    a.out_lse = out_lse;
    a.trace = g->trace;
    ep::splitkv_combine_kernel<<<g->nslices, ep::kPeerThreads, 0, static_cast<cudaStream_t>(stream)>>>(a);
    EP_CUDA_TRY(cudaGetLastError(), "ep_splitkv_combine_dev launch");
    h->launches++;
    return EP_OK;
}

int ep_peer_group_destroy(ep_peer_group g) {
    // (the plan / kernels using g must have completed)
    delete g;
    return EP_OK;
}

}  // extern "C"
