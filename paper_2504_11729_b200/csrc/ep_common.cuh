// ep_common.cuh — sm_100a device helpers shared by the kernels: mbarrier,
// bulk-async (TMA) copies, warp reductions, packed-fp32 math, bf16 unpacking.
#pragma once

#include <atomic>
#include <cstdint>
#include <utility>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

// Checked build (python -m paper_2504_11729_b200.build --checked ->
// _lib/libep_b200_checked.so, -DEP_CHECKED): device-side bounds checks on
// every index the kernels derive from plan / table data and bounded
// mbarrier / flag spins, each trapping with the failing condition, file and
// line. The GPU test suite runs against it (EP_LIB=...) as this repo's
// stand-in for compute-sanitizer (closed on this GPU pool). Release builds
// compile the checks away.
#ifdef EP_CHECKED
#include <cstdio>
#define EP_DCHECK(cond)                                                                                   \
    do {                                                                                                  \
        if (!(cond)) {                                                                                    \
            printf("EP_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__,   \
                   int(blockIdx.x), int(threadIdx.x));                                                   \
            __trap();                                                                                     \
        }                                                                                                 \
    } while (0)
#else
#define EP_DCHECK(cond) \
    do {                \
    } while (0)
#endif

namespace ep {

// Opts kernel Kern into at least `bytes` of dynamic shared memory on the
// current device (the attribute is per device context and a process may
// drive several GPUs); raised only when a launch needs more than before.
template <auto Kern>
inline cudaError_t ensure_smem(int bytes) {
    static std::atomic<int> done[64] = {};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::atomic<int>& d = done[dev & 63];
    if (d.load(std::memory_order_acquire) >= bytes) return cudaSuccess;
    e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) {
        int cur = d.load(std::memory_order_relaxed);
        while (cur < bytes && !d.compare_exchange_weak(cur, bytes, std::memory_order_release)) {
        }
    }
    return e;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

// ------------------------------------------------------------- mbarrier --

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef EP_CHECKED
    // a protocol bug (an arrival that never comes) traps instead of hanging
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (!mbar_try_wait(bar, parity)) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 5000000000ull) {
            printf("EP_DCHECK: mbarrier wait > 5 s (block %d thread %d parity %u)\n", int(blockIdx.x),
                   int(threadIdx.x), parity);
            __trap();
        }
    }
#else
    while (!mbar_try_wait(bar, parity)) {
    }
#endif
}

// ------------------------------------------------- bulk async copy (TMA) --

// 1-D bulk copy global -> shared, completion signalled on an mbarrier as
// transaction bytes (SASS: UBLKCP). bytes % 16 == 0, both addresses 16B aligned.
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_gmem, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Same with an L2 evict-first policy: streamed KV is read exactly once.
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst_smem, const void* src_gmem,
                                                     uint32_t bytes, uint64_t* bar,
                                                     uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
        "%2, [%3], %4;" ::"r"(smem_u32(dst_smem)),
        "l"(src_gmem), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Bulk prefetch of [src, src + bytes) into L2 (bytes % 16 == 0).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// Named barrier over a subset of warps (id 0 is __syncthreads).
// gpu-scope acquire load / release store of a flag word (cross-CTA handoff)
__device__ __forceinline__ unsigned int ld_acquire_gpu(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n_threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n_threads) : "memory");
}

// ---------------------------------------------------------------- math --

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    return __ffma2_rn(a, b, c);
}

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// max(a, b, c) in one instruction (sm_100 FMNMX3); NaN handling as fmaxf
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float fast_log2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Two packed bf16 (low half = element 2i) -> float2 without cvt: a bf16 is the
// high 16 bits of the fp32 with the same value.
__device__ __forceinline__ float2 bf16x2_to_float2(uint32_t w) {
    // PRMT and LOP3 both issue on the ALU pipe, leaving the FMA pipe (which
    // an IMAD.SHL would use) to the FFMA2s.
    uint32_t lo;
    asm("prmt.b32 %0, %1, 0, 0x1044;" : "=r"(lo) : "r"(w));
    float2 r;
    r.x = __uint_as_float(lo);
    r.y = __uint_as_float(w & 0xffff0000u);
    return r;
}

template <int WIDTH = 32>
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int m = WIDTH / 2; m > 0; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
    return v;
}

template <int WIDTH = 32, typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int m = WIDTH / 2; m > 0; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    return v;
}

// ------------------------------------- NVLink low-latency {value, flag} --
// A 16-byte word {v0, flag, v1, flag} written with one vector store over
// peer memory carries its own flag: the reader polls until both flags equal
// the step epoch (no fence, no separate flag round trip). Used by the split-KV
// combine (kern_peer.cu) and the fused split-KV decode (K1 + merge.cuh).

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void st_ll(uint4* p, float v0, float v1, uint32_t flag) {
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "r"(__float_as_uint(v0)), "r"(flag), "r"(__float_as_uint(v1)), "r"(flag)
                 : "memory");
}

// Poll one LL word until both halves carry `flag`; trap after 20 s.
__device__ __forceinline__ float2 ld_ll(const uint4* p, uint32_t flag) {
    uint4 w;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(p) : "memory");
    if (w.y != flag || w.w != flag) {
        const uint64_t t0 = globaltimer();
        do {
            asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(p) : "memory");
            if (globaltimer() - t0 > 20000000000ull) __trap();
        } while (w.y != flag || w.w != flag);
    }
    return make_float2(__uint_as_float(w.x), __uint_as_float(w.z));
}

// ----------------------------------------------------------- dtype I/O --

template <typename T>
__device__ __forceinline__ float to_f32(T x);
template <>
__device__ __forceinline__ float to_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 x) {
    return __bfloat162float(x);
}

template <typename T>
__device__ __forceinline__ T from_f32(float x);
template <>
__device__ __forceinline__ float from_f32<float>(float x) {
    return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}


// Launch with programmatic dependent launch (PDL): the kernel may be
// scheduled while its stream predecessor drains; it must execute
// griddepcontrol.wait before touching the predecessor's data.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_with_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
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

}  // namespace ep
