// umma.cuh — thin inline-PTX layer for sm_100a tensor cores (tcgen05/TMEM),
// TMA tensor copies and proxy fences, used by kern_verify.cu.
#pragma once

#include <cstdint>
#include <cuda.h>

#include "ep_common.cuh"

namespace ep {
namespace umma {

// ---------------------------------------------------------------- TMEM --

// One warp allocates `cols` TMEM columns (power of two >= 32) and writes the
// base address to shared memory.
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

__device__ __forceinline__ void fence_before_sync() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Generic-proxy shared-memory writes -> visible to the async proxy (MMA/TMA).
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 32 lanes x 32 columns of 32-bit: thread t of the warp gets TMEM lane
// (taddr.lane + t), columns [taddr.col, taddr.col + 32).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
          "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
          "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
        "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
        "r"(r[29]), "r"(r[30]), "r"(r[31]));
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
        "r"(r[15]));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// One lane of the (converged) warp returns true (elect.sync). Used so a whole
// warp runs an MMA-issue loop with warp-uniform operands (uniform registers,
// no R2UR waterfall) while exactly one lane issues.
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

// ----------------------------------------------------------- descriptors --

// Shared-memory matrix descriptor, SWIZZLE_128B (layout type 2), sm100
// version 1. Addresses/offsets in bytes; the 128B-swizzle atoms (8 rows x
// 128 B) must be 1024-byte aligned (base_offset 0).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                    uint32_t sbo_bytes) {
    uint64_t d = 0;
    d |= uint64_t((saddr >> 4) & 0x3FFF);
    d |= uint64_t((lbo_bytes >> 4) & 0x3FFF) << 16;
    d |= uint64_t((sbo_bytes >> 4) & 0x3FFF) << 32;
    d |= uint64_t(1) << 46;  // version (Blackwell)
    d |= uint64_t(2) << 61;  // SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f16: BF16 x BF16 -> F32, dense.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N, bool a_mn_major, bool b_mn_major) {
    return (1u << 4)                              // c_format = F32
           | (1u << 7)                            // a_format = BF16
           | (1u << 10)                           // b_format = BF16
           | (uint32_t(a_mn_major) << 15) | (uint32_t(b_mn_major) << 16)
           | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]; issued by ONE thread.
__device__ __forceinline__ void mma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem] (A in TMEM: lane = row, two 16-bit K
// elements per 32-bit column); issued by ONE thread.
__device__ __forceinline__ void mma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Batched issue: one asm block per MMA chain so the descriptor bases are moved
// to uniform registers once and each MMA only adds an immediate offset
// (the start-address field of a smem descriptor is bits [0,14) in 16-byte
// units; offsets never carry out of it for smem addresses < 256 KB).
//
// QK^T chain of kverify: 8 x (M128 N64 K16), A = Q tile (two 64-column SW128
// halves 16 KB apart), B = K block (two halves 8 KB apart), k-step 32 bytes.
__device__ __forceinline__ void mma_chain_qk8(uint32_t tmem_d, uint64_t dq, uint64_t dk,
                                              uint32_t idesc) {
#define EP_QK_STEP(OA, OB) \
    "add.s64 a, %1, " #OA ";\n\tadd.s64 b, %2, " #OB ";\n\t" \
    "tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, t;\n\t"
    asm volatile(
        "{\n\t.reg .b64 a, b;\n\t.reg .pred f, t;\n\t"
        "setp.ne.b32 f, 0, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, f;\n\t"
        EP_QK_STEP(2, 2) EP_QK_STEP(4, 4) EP_QK_STEP(6, 6)
        EP_QK_STEP(1024, 512) EP_QK_STEP(1026, 514) EP_QK_STEP(1028, 516) EP_QK_STEP(1030, 518)
        "}" ::"r"(tmem_d), "l"(dq), "l"(dk), "r"(idesc));
#undef EP_QK_STEP
}

// QK^T chain with A = Q from TMEM (64 columns: two bf16 per column, +8
// columns per 16-element k-step) and B = K block (two SW128 halves 8 KB apart).
__device__ __forceinline__ void mma_chain_qk8_ts(uint32_t tmem_d, uint32_t tq, uint64_t dk,
                                                 uint32_t idesc) {
#define EP_QKT_STEP(OA, OB) \
    "add.u32 x, %1, " #OA ";\n\tadd.s64 b, %2, " #OB ";\n\t" \
    "tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %3, t;\n\t"
    asm volatile(
        "{\n\t.reg .b64 b;\n\t.reg .b32 x;\n\t.reg .pred f, t;\n\t"
        "setp.ne.b32 f, 0, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, f;\n\t"
        EP_QKT_STEP(8, 2) EP_QKT_STEP(16, 4) EP_QKT_STEP(24, 6)
        EP_QKT_STEP(32, 512) EP_QKT_STEP(40, 514) EP_QKT_STEP(48, 516) EP_QKT_STEP(56, 518)
        "}" ::"r"(tmem_d), "r"(tq), "l"(dk), "r"(idesc));
#undef EP_QKT_STEP
}

// PV chain: 4 x (M128 N128 K16) with A from TMEM (ta: +8 columns per k-step)
// and B = V block MN-major (+2048 bytes = +128 units per k-step). `first`
// clears the accumulator on the first MMA.
__device__ __forceinline__ void mma_chain_pv4(uint32_t tmem_d, uint32_t ta, uint64_t dv,
                                              uint32_t idesc, uint32_t first) {
#define EP_PV_STEP(OA, OB) \
    "add.u32 x, %1, " #OA ";\n\tadd.s64 b, %2, " #OB ";\n\t" \
    "tcgen05.mma.cta_group::1.kind::f16 [%0], [x], b, %3, t;\n\t"
    asm volatile(
        "{\n\t.reg .b64 b;\n\t.reg .b32 x;\n\t.reg .pred f, t;\n\t"
        "setp.eq.b32 f, %4, 0;\n\tsetp.eq.b32 t, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, f;\n\t"
        EP_PV_STEP(8, 128) EP_PV_STEP(16, 256) EP_PV_STEP(24, 384)
        "}" ::"r"(tmem_d), "r"(ta), "l"(dv), "r"(idesc), "r"(first));
#undef EP_PV_STEP
}

// Arrive once on `bar` when all previously issued tcgen05 ops of this thread
// complete (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------- TMA --

__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(tmap) : "memory");
}

// 2-D tiled TMA load: box at (c0 = inner coordinate, c1 = row) -> smem.
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 3-D tiled TMA load: box at (c0, c1, c2) -> smem.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// ------------------------------------------------------ CTA pair (2-SM) --
// cta_group::2: the two CTAs of a cluster of 2 (one TPC) run one MMA of
// M = 256 — each holds its 128 rows of A and of the accumulator, and half of
// B's N columns; the even CTA (rank 0) issues the MMAs for both. The smem
// operands sit at the same offsets in both CTAs.

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The shared::cluster address of `p` (own shared memory) in CTA `rank` of the cluster.
__device__ __forceinline__ uint32_t mapa_shared(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* smem_dst, uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(smem_dst)),
                 "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols));
}

// D[tmem, both CTAs] (+)= A[smem, both] * B[smem, both]; issued by ONE thread of rank 0.
__device__ __forceinline__ void mma_bf16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Arrive on the mbarrier at `bar`'s offset in every CTA of `mask` once the
// pair's prior MMAs complete.
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// TMA 2-D tile into this CTA's shared memory, completion bytes counted on an
// mbarrier that may live in the peer CTA (bar_cluster: shared::cluster address).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const void* tmap, int c0, int c1, uint32_t bar_cluster,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster), "l"(policy)
        : "memory");
}

}  // namespace umma
}  // namespace ep
