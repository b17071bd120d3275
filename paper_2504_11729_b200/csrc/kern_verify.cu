// kern_verify.cu — K3: multi-row (speculative-verify) spliced attention on
// the sm_100a tensor cores.
//
// Reference: the verify construction of SURVEY §8a a16 — prefill of
// [last, d1..dk] against the cache (model.cpp:211-236), i.e. transformer_layer's
// attention block (model.cpp:161-182) with n_q = k+1 causal rows: cached
// segments fully visible, the draft segment causal (attention.cpp:29-33).
// With GQA the R = group * n_q rows of one kv-head (20 for k=4, 36 for k=8)
// share every K/V byte; at 20-36 FLOP/B that is beyond the CUDA cores, so:
//
//   QK^T : S[128 x 64]  (TMEM, fp32) = Q[128 x 128] (smem) . K[64 keys x 128]^T
//   PV   : O[128 x 128] (TMEM, fp32) += (P_hi + P_lo)[128 x 64] (TMEM, 2 x bf16) . V[64 x 128]
//          (P_hi alone when the caller asked for bf16 output: prefill tiles)
//
// tcgen05.mma M=128 (rows >= R are padding; the M=128 issue rate equals
// M=64's), operands staged by TMA with 128B swizzle straight from the paged
// pool (the [page][head][token][d] tile is a 2-D tensor of 128-element rows).
// Warp roles (128 threads, one CTA per SM, persistent over the planner's page
// ranges like K1):
//   warp 8 lane 0 : TMA producer of the K ring (5 stages, freed after QK)
//   warp 10 lane 0: TMA producer of the V ring (3 stages, freed after PV)
//   warp 9        : QK MMA issuer (one elected lane); owns the TMEM allocation
//   warp 11       : PV MMA issuer
//   warps 0-7     : softmax + epilogue. Query rows are spread over the four
//                   TMEM lane quarters (row v -> M row 32*(v%4) + v/4) so all
//                   four SMSPs work, and each row's 64 keys are split between
//                   warps q and q+4: tcgen05.ld of 32 scores, causal/tail mask,
//                   exp2, P written as bf16 hi+lo, swizzled. Rescaling is lazy
//                   (FA4-style): the row max only moves when it grows by > 2^8,
//                   then O is rescaled in TMEM (tcgen05.ld/st); else P <= 256.
// QK of block i+1 is issued before PV of block i so the tensor core overlaps
// the softmax. Items that split a (request, kv-head) merge by LSE through the
// same per-unit counter protocol as K1.
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ep_common.cuh"
#include "ep_internal.h"
#include "merge.cuh"
#include "umma.cuh"

namespace ep {
namespace {

constexpr int kBT = 64;        // keys per block
constexpr int kD = 128;        // head dim
constexpr int kM = 128;        // UMMA M (rows, padded)
constexpr int kKStages = 7;  // K ring: a K block is free right after its QK
constexpr int kVStages = 7;  // V ring: a V block is free after its PV
constexpr int kSoftWarps = 8;  // 2 ping-pong groups x 4 TMEM lane quarters
constexpr int kSoftThreads = kSoftWarps * 32;
constexpr int kProdWarp = 8, kMmaWarp = 9, kProdVWarp = 10, kPvWarp = 11;
constexpr int kThreads = 384;
constexpr int kMaxRows = 128;     // valid query rows per tile (one M = 128 MMA tile)
constexpr float kLazy = 8.0f;     // log2 headroom before the max is moved

constexpr int kKVHalf = kBT * 128;         // 8 KB: 64 rows x 64 bf16
constexpr int kBlkBytes = 2 * kKVHalf;     // one K (or V) block: two 64-column halves
constexpr int OFF_STAGE = 0;
constexpr int OFF_VST = OFF_STAGE + kKStages * kBlkBytes;
constexpr int OFF_XM = OFF_VST + kVStages * kBlkBytes;  // [2 groups][128] row max of each group
constexpr int OFF_XL = OFF_XM + 2 * kM * 4; // [2 groups][128] row sum of each group
constexpr int OFF_BAR = OFF_XL + 2 * kM * 4;
constexpr int kNumBars = 2 * kKStages + 2 * kVStages + 2 + 2 + 2 + 2 + 2;
constexpr int OFF_MISC = OFF_BAR + kNumBars * 8;
constexpr int kSmem = OFF_MISC + 32;  // dynamic smem base must be 1024-aligned (checked)
// TMEM columns (512): O of group 0 / 1 (128 each, fp32), S of group 0 / 1
// (64 each, fp32) whose columns are overwritten by that group's P as bf16 hi
// (32 columns: two bf16 per 32-bit column) and lo (32), then the item's Q
// tile (64 columns, bf16). Q and P are the A operands of the MMAs, so the
// tensor core reads only K and V from shared memory. With a single bf16 P
// (bf16 output) P gets its own 32 columns per group (kColP), so the QK of a
// group's next block can overwrite S as soon as the softmax has read it,
// instead of after the PV that consumes P.
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColO = 0, kColS = 256, kColQ = 384, kColP = 448;

// Tiles of <= 64 rows (verify: 20 / 36 rows per kv-head) issue M = 64 MMAs —
// half the tensor work of M = 128. With cta_group::1 an M = 64 operand / result
// row m lives in TMEM lane 32 * (m / 16) + m % 16, i.e. lanes 0-15 of each
// lane quarter, where the softmax threads of lanes 0-15 already keep rows
// v = 4 * lane + quarter < 64 — the thread <-> row mapping does not change.
constexpr uint32_t kIdescQK128 = umma::idesc_bf16_f32(kM, kBT, false, false);
constexpr uint32_t kIdescPV128 = umma::idesc_bf16_f32(kM, kD, false, true);
constexpr uint32_t kIdescQK64 = umma::idesc_bf16_f32(64, kBT, false, false);
constexpr uint32_t kIdescPV64 = umma::idesc_bf16_f32(64, kD, false, true);

struct Bars {
    uint64_t* full_k;   // [KS] K block landed
    uint64_t* empty_k;  // [KS] K block consumed (commit after its QK)
    uint64_t* full_v;   // [VS] V block landed
    uint64_t* empty_v;  // [VS] V block consumed (commit after its PV)
    uint64_t* s_full;   // [2 groups] QK result in TMEM
    uint64_t* p_full;   // [2] P written (+ O rescaled)
    uint64_t* pv_done;  // [2] PV finished (P buffer free, O updated)
    uint64_t* q_ready;  // Q tile of the item in smem
    uint64_t* o_free;   // epilogue read O
    uint64_t* s_free;   // [2] softmax read S (single-P mode: S may be overwritten)
};

// Debug trace (a.trace != null, CTA 0 only): clock64 per event and block.
constexpr int kTraceBlocks = 1024;
enum TraceEv { TR_KISSUE = 0, TR_VISSUE, TR_QK, TR_PV, TR_S_SEEN, TR_P_DONE,
              TR_QK_START, TR_QK_FULLK, TR_QK_DONE, TR_PV_START, TR_PV_PFULL, TR_PV_DONE, TR_N };
// Per-item events (indexed by the CTA's item number), softmax warp 0.
enum ItemEv { IT_START = TR_N, IT_QDONE, IT_LASTPV, IT_EPI, IT_OUT, IT_END };  // 18 rows in total
__device__ __forceinline__ void trace(const DecodeArgs& a, int ev, uint32_t gi) {
    if (a.trace && blockIdx.x == 0 && gi < kTraceBlocks && (threadIdx.x & 31) == 0) {
        long long t;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
        a.trace[ev * kTraceBlocks + gi] = (unsigned long long)t;
    }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&v);
}

// Walks the 64-token blocks of a work item in order: page by page.
struct BlockWalker {
    const PageDesc* pd;
    int lp, lp1, t0;
    PageDesc cur;
    int64_t num_pages = -1;  // checked build: page ids in range
    __device__ void load() {
        cur = pd[lp];
        EP_DCHECK(num_pages < 0 || (cur.page >= 0 && cur.page < num_pages && cur.n_tok >= 1));
    }
    __device__ void init(const PageDesc* p, int lp0, int lp1_, int64_t n_pages = -1) {
        pd = p;
        lp = lp0;
        lp1 = lp1_;
        t0 = 0;
        num_pages = n_pages;
        if (lp < lp1) load();
    }
    // current block: valid rows and absolute position of its first key
    __device__ int nv() const { return min(kBT, cur.n_tok - t0); }
    __device__ int64_t pos() const { return cur.pos + t0; }
    __device__ void next() {
        t0 += kBT;
        if (t0 >= cur.n_tok) {
            t0 = 0;
            if (++lp < lp1) load();
        }
    }
};

// Softmax layout: query row v of a (request, kv-head) lives in M row
// 32*(v%4) + v/4, so the valid rows spread over all four TMEM lane quarters
// (a warp reads only quarter warp%4, i.e. its own SMSP). Ping-pong: warps
// 0-3 (group 0) take the even key blocks of an item, warps 4-7 (group 1) the
// odd ones, each group with its own online-softmax state, S and P buffers and
// O accumulator in TMEM; the two states merge by LSE in the epilogue. While
// one group waits on TMEM loads / barriers the other computes, and the tensor
// core always has the other group's QK or PV to run.
__global__ void __launch_bounds__(kThreads, 1)
    verify_attention_kernel(const DecodeArgs a, const __grid_constant__ CUtensorMap tmap_k,
                            const __grid_constant__ CUtensorMap tmap_v, int rows) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // PDL: the predecessor has completed
    uint8_t* smem = smem_raw;
    if (threadIdx.x == 0 && (smem_u32(smem) & 1023u) != 0) __trap();  // SW128 atoms need 1 KB alignment
    uint8_t* sStage = smem + OFF_STAGE;
    float* xm = reinterpret_cast<float*>(smem + OFF_XM);
    float* xl = reinterpret_cast<float*>(smem + OFF_XL);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    constexpr int kRB = 2 * kKStages + 2 * kVStages;
    Bars B{bar, bar + kKStages, bar + 2 * kKStages, bar + 2 * kKStages + kVStages,
           bar + kRB, bar + kRB + 2, bar + kRB + 4, bar + kRB + 6, bar + kRB + 7, bar + kRB + 8};
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + OFF_MISC);
    int* s_flag = reinterpret_cast<int*>(smem + OFF_MISC + 16);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it0 = a.cta_item_ptr[blockIdx.x], it1 = a.cta_item_ptr[blockIdx.x + 1];
    const int Hkv = a.n_kv_heads, P = a.page_tokens;
    const bool m64 = rows <= 64;
    const uint32_t kIdescQK = m64 ? kIdescQK64 : kIdescQK128;
    const uint32_t kIdescPV = m64 ? kIdescPV64 : kIdescPV128;
    if (a.trace && threadIdx.x == 0 && blockIdx.x < kTraceBlocks)  // debug: per-CTA start (ns)
        a.trace[18 * kTraceBlocks + 2 * blockIdx.x] = globaltimer_ns();
    const int G = a.n_q_heads / Hkv;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kKStages; ++s) {
            mbar_init(&B.full_k[s], 1);
            mbar_init(&B.empty_k[s], 1);
        }
        for (int s = 0; s < kVStages; ++s) {
            mbar_init(&B.full_v[s], 1);
            mbar_init(&B.empty_v[s], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&B.s_full[i], 1);
            mbar_init(&B.p_full[i], 4);
            mbar_init(&B.pv_done[i], 1);
            mbar_init(&B.s_free[i], 4);
        }
        mbar_init(B.q_ready, kSoftWarps);
        mbar_init(B.o_free, kSoftWarps);
        fence_mbar_init();
    }
    if (warp == kMmaWarp) umma::tmem_alloc(tmem_slot, kTmemCols);
    if (warp == kProdWarp && lane == 0) umma::tma_prefetch_desc(&tmap_k);
    if (warp == kProdVWarp && lane == 0) umma::tma_prefetch_desc(&tmap_v);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *tmem_slot;

    if (warp == kProdWarp || warp == kProdVWarp) {
        // ========================= producers (K ring, V ring) =========================
        if (lane == 0) {
            const bool is_k = warp == kProdWarp;
            const int ns = is_k ? kKStages : kVStages;
            uint64_t* fullb = is_k ? B.full_k : B.full_v;
            uint64_t* emptyb = is_k ? B.empty_k : B.empty_v;
            uint8_t* ring = smem + (is_k ? OFF_STAGE : OFF_VST);
            const CUtensorMap* tm = is_k ? &tmap_k : &tmap_v;
            // K/V of verify tiles (<= 64 rows) stream once; the 128-row
            // tiles (prefill chunks, shared prefixes) re-read each block from
            // L2 for many tiles, so they are not marked evict-first (same-box
            // A/B: cloud prefill 0.800 -> 0.771 ms, edge 1.403 -> 1.363 ms;
            // an L2 bulk prefetch of the next item's Q rows was slower)
            const uint64_t pol = rows > 64 ? l2_policy_evict_normal() : l2_policy_evict_first();
            uint32_t gi = 0;
            for (int it = it0; it < it1; ++it) {
                const WorkItem w = a.items[it];
                BlockWalker wk;
                wk.init(a.pdesc + a.req_page_off[w.b], w.lp0, w.lp1, a.num_pages);
                for (int i = 0; i < w.nblk; ++i, ++gi, wk.next()) {
                    const int st = gi % ns;
                    mbar_wait(&emptyb[st], ((gi / ns) & 1) ^ 1);
                    trace(a, is_k ? TR_KISSUE : TR_VISSUE, gi);
                    mbar_arrive_expect_tx(&fullb[st], kBlkBytes);
                    const int row = int((int64_t(wk.cur.page) * Hkv + w.g) * P + wk.t0);
                    uint8_t* dst = ring + st * kBlkBytes;
                    umma::tma_load_3d(dst, tm, 0, row, 0, &fullb[st], pol);  // both d-halves
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ============================== QK issuer ===============================
        // The whole warp runs the loop (operands stay warp-uniform); one
        // elected lane issues each MMA / commit. QK and PV have separate issuing
        // warps, so neither's barrier waits stall the other's MMAs (a UTCHMMA
        // blocks its issuer while the tensor queue is full). Descriptors are
        // built once; per MMA only the 14-bit start-address field moves.
        const uint64_t dk = umma::smem_desc_sw128(smem_u32(sStage), 16, 1024);
        const bool two_part = a.pv_parts > 1;
        // S[grp] may be overwritten once the previous block of the group has
        // been read by the softmax (single P: s_free) or, when P aliases S
        // (hi+lo), once its PV completed (pv_done). Every phase is waited in
        // order, so the parities never alias.
        uint64_t* sbar = two_part ? B.pv_done : B.s_free;
        uint32_t gi = 0, n = 0;
        uint32_t nqk[2] = {0, 0};
        if (two_part) {
            // hi+lo P aliases S: QK(i+2) must follow PV(i). One warp issues both
            // in the order QK(0) QK(1) | PV(i) QK(i+2) ...; the tensor pipe runs
            // in issue order, so QK(i+2) needs no wait for PV(i)'s completion.
            const uint64_t dv = umma::smem_desc_sw128(smem_u32(smem + OFF_VST), kKVHalf, 1024);
            uint32_t cpv[2] = {0, 0};
            auto issue_qk = [&](int i, uint32_t g_i) {
                const int st = g_i % kKStages, grp = i & 1;
                trace(a, TR_QK_START, g_i);
                mbar_wait(&B.full_k[st], (g_i / kKStages) & 1);
                trace(a, TR_QK, g_i);
                umma::fence_after_sync();
                const uint64_t kd0 = dk + ((st * kBlkBytes) >> 4);
                if (umma::elect_one())
                    umma::mma_chain_qk8_ts(tmem + kColS + grp * kBT, tmem + kColQ, kd0, kIdescQK);
                if (umma::elect_one()) {
                    umma::mma_commit(&B.s_full[grp]);
                    umma::mma_commit(&B.empty_k[st]);
                }
                __syncwarp();
                trace(a, TR_QK_DONE, g_i);
            };
            auto issue_pv = [&](int i, uint32_t g_i) {
                const int grp = i & 1;
                trace(a, TR_PV_START, g_i);
                mbar_wait(&B.p_full[grp], cpv[grp] & 1);
                if (i == 0) mbar_wait(B.o_free, (n & 1) ^ 1);
                const uint32_t vs = g_i % kVStages;
                mbar_wait(&B.full_v[vs], (g_i / kVStages) & 1);
                trace(a, TR_PV, g_i);
                umma::fence_after_sync();
                const uint64_t bd0 = dv + ((vs * kBlkBytes) >> 4);
                const uint32_t ta0 = tmem + kColS + grp * kBT, td = tmem + kColO + grp * kD;
                if (umma::elect_one()) {
                    umma::mma_chain_pv4(td, ta0, bd0, kIdescPV, i < 2 ? 1u : 0u);
                    umma::mma_chain_pv4(td, ta0 + 32, bd0, kIdescPV, 0u);
                }
                if (umma::elect_one()) {
                    umma::mma_commit(&B.pv_done[grp]);
                    umma::mma_commit(&B.empty_v[vs]);
                }
                __syncwarp();
                trace(a, TR_PV_DONE, g_i);
                ++cpv[grp];
            };
            for (int it = it0; it < it1; ++it, ++n) {
                const WorkItem w = a.items[it];
                mbar_wait(B.q_ready, n & 1);
                for (int i = 0; i < 2 && i < w.nblk; ++i) issue_qk(i, gi + i);
                for (int i = 0; i < w.nblk; ++i) {
                    issue_pv(i, gi + i);
                    if (i + 2 < w.nblk) issue_qk(i + 2, gi + i + 2);
                }
                gi += uint32_t(w.nblk);
            }
        } else
        for (int it = it0; it < it1; ++it, ++n) {
            const WorkItem w = a.items[it];
            mbar_wait(B.q_ready, n & 1);
            for (int i = 0; i < w.nblk; ++i) {
                const int grp = i & 1;
                const uint32_t g_i = gi + i;
                const int st = g_i % kKStages;
                trace(a, TR_QK_START, g_i);
                if (nqk[grp] > 0) mbar_wait(&sbar[grp], (nqk[grp] - 1) & 1);
                mbar_wait(&B.full_k[st], (g_i / kKStages) & 1);
                trace(a, TR_QK, g_i);
                umma::fence_after_sync();
                const uint64_t kd0 = dk + ((st * kBlkBytes) >> 4);
                const uint32_t ts = tmem + kColS + grp * kBT;
                static_assert(kKVHalf == 8192, "offsets baked into mma_chain_qk8_ts");
                if (umma::elect_one()) umma::mma_chain_qk8_ts(ts, tmem + kColQ, kd0, kIdescQK);
                if (umma::elect_one()) {
                    umma::mma_commit(&B.s_full[grp]);
                    umma::mma_commit(&B.empty_k[st]);
                }
                __syncwarp();
                trace(a, TR_QK_DONE, g_i);
                ++nqk[grp];
            }
            gi += uint32_t(w.nblk);
        }
    } else if (warp == kPvWarp) {
        // ======================= PV issuer (single-P mode) =======================
        const uint64_t dv = umma::smem_desc_sw128(smem_u32(smem + OFF_VST), kKVHalf, 1024);
        const bool two_part = a.pv_parts > 1;
        uint32_t gi = 0, n = 0;
        uint32_t cpv[2] = {0, 0};
        for (int it = two_part ? it1 : it0; it < it1; ++it, ++n) {
            const WorkItem w = a.items[it];
            for (int i = 0; i < w.nblk; ++i) {
                const int grp = i & 1;
                const uint32_t g_i = gi + i;
                trace(a, TR_PV_START, g_i);
                mbar_wait(&B.p_full[grp], cpv[grp] & 1);
                trace(a, TR_PV_PFULL, g_i);
                if (i == 0) mbar_wait(B.o_free, (n & 1) ^ 1);  // previous item's epilogue read O
                const uint32_t vs = g_i % kVStages;
                mbar_wait(&B.full_v[vs], (g_i / kVStages) & 1);
                trace(a, TR_PV, g_i);
                umma::fence_after_sync();
                const uint64_t bd0 = dv + ((vs * kBlkBytes) >> 4);
                const uint32_t ta0 = two_part ? tmem + kColS + grp * kBT : tmem + kColP + grp * 32;
                const uint32_t td = tmem + kColO + grp * kD;
                // P = hi + lo (two bf16 tiles in TMEM): O += P_hi V + P_lo V keeps
                // the probabilities at ~2^-17 relative instead of bf16's 2^-9.
                if (umma::elect_one()) {
                    umma::mma_chain_pv4(td, ta0, bd0, kIdescPV, i < 2 ? 1u : 0u);
                    if (two_part) umma::mma_chain_pv4(td, ta0 + 32, bd0, kIdescPV, 0u);
                }
                if (umma::elect_one()) {
                    umma::mma_commit(&B.pv_done[grp]);
                    umma::mma_commit(&B.empty_v[vs]);
                }
                __syncwarp();
                trace(a, TR_PV_DONE, g_i);
                ++cpv[grp];
            }
            gi += uint32_t(w.nblk);
        }
    } else {
        // ========================= softmax + epilogue =========================
        const int quarter = warp & 3, grp = warp >> 2;  // TMEM lane quarter, ping-pong group
        const int m = quarter * 32 + lane;               // M row = TMEM lane
        const int v = lane * 4 + quarter;                // query row index of this M row
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        const uint32_t tS = tmem + kColS + grp * kBT + lane_off;
        const uint32_t tP = tmem + kColP + grp * 32 + lane_off;  // single-P mode
        const uint32_t tOg = tmem + kColO + grp * kD + lane_off;
        const float scale = a.q_scale;  // log2(e)/sqrt(d)
        const bool two_part = a.pv_parts > 1;
        const uint32_t pair_bar = 1 + quarter;  // named barrier of warps q and q+4
        uint32_t cnt = 0, n = 0;  // blocks processed by this group (all items)
        uint32_t gi0 = 0;         // global index of the item's first block
        for (int it = it0; it < it1; ++it, ++n) {
            if (threadIdx.x == 0) trace(a, IT_START, n);
            const WorkItem w = a.items[it];
            const int nrows = w.pad > 0 ? w.pad : rows;  // valid rows of this item's tile
            const bool valid_row = v < nrows;
            // Row v of the tile: request rq0 + v / (G n_q), query row qi, head h.
            // A tile spans several requests in the shared-prefix (cascade) pass.
            const int rpr = G * a.n_q;
            const int rq = w.rq0 + v / rpr, qi = (v % rpr) / G, h = w.g * G + v % G;
            const int64_t q0 = w.q0min;
            const int64_t my_qpos = (valid_row ? a.q_pos[rq] : q0) + qi;

            // ---- Q tile -> TMEM (A operand of QK): group g writes d-half g ----
            {
                const uint8_t* src = static_cast<const uint8_t*>(a.q) +
                                     (((q_row_base(a, rq) + qi) * a.n_q_heads + h) * kD + grp * 64) * 2;
                uint32_t qv[32];
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint4 val = make_uint4(0, 0, 0, 0);
                    if (valid_row) val = *reinterpret_cast<const uint4*>(src + c * 16);
                    qv[4 * c] = val.x;
                    qv[4 * c + 1] = val.y;
                    qv[4 * c + 2] = val.z;
                    qv[4 * c + 3] = val.w;
                }
                umma::tmem_st32(tmem + kColQ + grp * 32 + lane_off, qv);
                umma::tmem_wait_st();
                umma::fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(B.q_ready);
                if (threadIdx.x == 0) trace(a, IT_QDONE, n);
            }

            float m_used = -INFINITY, l = 0.f;
            BlockWalker wk;
            wk.init(a.pdesc + a.req_page_off[w.b], w.lp0, w.lp1, a.num_pages);
            if (grp == 1) wk.next();
            for (int i = grp; i < w.nblk; i += 2) {
                const int nv = wk.nv();
                const int64_t pos = wk.pos();
                const uint32_t gi = gi0 + i;

                // ---- the 64 scores of this row ----
                mbar_wait(&B.s_full[grp], cnt & 1);
                if (threadIdx.x == grp * 128) trace(a, TR_S_SEEN, gi);
                umma::fence_after_sync();
                uint32_t sr[64];
                umma::tmem_ld32(tS, *reinterpret_cast<uint32_t(*)[32]>(sr));
                umma::tmem_ld32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
                umma::tmem_wait_ld();
                if (!two_part) {  // S is in registers: the next QK may overwrite it
                    umma::fence_before_sync();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&B.s_free[grp]);
                }

                if (!(nv == kBT && pos + kBT - 1 <= q0)) {
                    // keys j < lim are valid and visible: one 32-bit compare per key
                    const int64_t vis = my_qpos - pos + 1;
                    const int lim = vis < 0 ? 0 : int(vis < int64_t(nv) ? vis : int64_t(nv));
#pragma unroll
                    for (int j = 0; j < 64; ++j)
                        if (j >= lim) sr[j] = __float_as_uint(-INFINITY);
                }
                // row max: 8 independent chains of 3-input maxima (FMNMX3),
                // then a 3-input tree
                float mx[8];
#pragma unroll
                for (int c = 0; c < 8; ++c) mx[c] = __uint_as_float(sr[c]);
#pragma unroll
                for (int j = 8; j < 64; j += 16)
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        mx[c] = fmax3(mx[c], __uint_as_float(sr[j + c]),
                                      j + 8 + c < 64 ? __uint_as_float(sr[j + 8 + c]) : -INFINITY);
                const float hmax = fmax3(fmax3(mx[0], mx[1], mx[2]), fmax3(mx[3], mx[4], mx[5]), fmaxf(mx[6], mx[7]));
                const float bmax = valid_row ? hmax * scale : -INFINITY;
                // lazy max: move it only when the block exceeds it by > 2^kLazy
                float corr = 1.f;
                const bool move = bmax > m_used + kLazy;
                if (move) {
                    corr = m_used == -INFINITY ? 0.f : fast_exp2(m_used - bmax);
                    m_used = bmax;
                }
                const float mu = m_used == -INFINITY ? 0.f : m_used;
                float2 rsa[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                 make_float2(0.f, 0.f)};  // 4 independent row-sum chains
                uint32_t pk[32], pl[32];
                if (two_part) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[2 * j]), __uint_as_float(sr[2 * j + 1])),
                                                     make_float2(scale, scale), make_float2(-mu, -mu));
                        const float p0 = fast_exp2(x2.x);
                        const float p1 = fast_exp2(x2.y);
                        const float2 p2 = make_float2(p0, p1);
                        rsa[j & 3] = __fadd2_rn(rsa[j & 3], p2);
                        pk[j] = pack_bf16(p0, p1);
                        const float2 hi = bf16x2_to_float2(pk[j]);
                        const float2 lo = __fadd2_rn(p2, make_float2(-hi.x, -hi.y));
                        pl[j] = pack_bf16(lo.x, lo.y);
                    }
                } else {
                    // single bf16 P (bf16 output): the row sum keeps the fp32
                    // probabilities, so the lse stays fp32-accurate; RN rounding
                    // of P is unbiased, so the output scale error averages out
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float2 x2 = __ffma2_rn(make_float2(__uint_as_float(sr[2 * j]), __uint_as_float(sr[2 * j + 1])),
                                                     make_float2(scale, scale), make_float2(-mu, -mu));
                        const float p0 = fast_exp2(x2.x);
                        const float p1 = fast_exp2(x2.y);
                        pk[j] = pack_bf16(p0, p1);
                        rsa[j & 3] = __fadd2_rn(rsa[j & 3], make_float2(p0, p1));
                    }
                }
                const float2 rs2 = __fadd2_rn(__fadd2_rn(rsa[0], rsa[1]), __fadd2_rn(rsa[2], rsa[3]));
                l = l * corr + (rs2.x + rs2.y);

                // P/O of this group are free once its previous PV completed.
                mbar_wait(&B.pv_done[grp], (cnt & 1) ^ 1);
                if (i >= 2 && __any_sync(0xffffffffu, move)) {
                    umma::fence_after_sync();
#pragma unroll
                    for (int cblk = 0; cblk < 4; ++cblk) {
                        uint32_t o[32];
                        umma::tmem_ld32(tOg + cblk * 32, o);
                        umma::tmem_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) o[j] = __float_as_uint(__uint_as_float(o[j]) * corr);
                        umma::tmem_st32(tOg + cblk * 32, o);
                    }
                    umma::tmem_wait_st();
                }
                // P row -> TMEM over this group's S columns (A operand of the PV
                // MMAs): hi tile then lo tile.
                if (two_part) {
                    umma::tmem_st32(tS, pk);
                    umma::tmem_st32(tS + 32, pl);
                } else {
                    umma::tmem_st32(tP, pk);
                }
                umma::tmem_wait_st();
                if (nv < kBT) {
                    // Tail rows of V in the stage are stale page slots: zero them
                    // so 0 * garbage cannot reach the PV accumulator.
                    const int st = gi % kVStages;
                    mbar_wait(&B.full_v[st], (gi / kVStages) & 1);
                    uint8_t* vs = smem + OFF_VST + st * kBlkBytes;
                    const int n_chunks = (kBT - nv) * 8;
                    for (int c = (threadIdx.x & 127); c < 2 * n_chunks; c += 128) {
                        const int hsel = c / n_chunks, cc = c % n_chunks;
                        *reinterpret_cast<uint4*>(vs + hsel * kKVHalf + nv * 128 + cc * 16) =
                            make_uint4(0, 0, 0, 0);
                    }
                }
                if (nv < kBT) umma::fence_proxy_async_smem();  // the zeroed V rows -> the MMA's proxy
                umma::fence_before_sync();
                __syncwarp();
                if (lane == 0) mbar_arrive(&B.p_full[grp]);
                if (threadIdx.x == grp * 128) trace(a, TR_P_DONE, gi);
                ++cnt;
                wk.next();
                if (i + 1 < w.nblk) wk.next();
            }
            gi0 += uint32_t(w.nblk);

            // ---- epilogue: merge the two groups' (m, l, O) by LSE ----
            if (grp < w.nblk) {  // this group ran at least one block: wait its last PV
                mbar_wait(&B.pv_done[grp], (cnt & 1) ^ 1);
            }
            if (threadIdx.x == 0) trace(a, IT_LASTPV, n);
            xm[grp * kM + m] = m_used;
            xl[grp * kM + m] = l;
            named_bar_sync(pair_bar, 64);
            // Past the pair barrier the partner warp (same lane quarter, other
            // group) has also waited for its last PV: both O tiles are final.
            const float m0v = xm[m], m1v = xm[kM + m], l0v = xl[m], l1v = xl[kM + m];
            const float M = fmaxf(m0v, m1v);
            const float w0 = (l0v > 0.f) ? fast_exp2(m0v - M) : 0.f;
            const float w1 = (l1v > 0.f) ? fast_exp2(m1v - M) : 0.f;
            const float L = w0 * l0v + w1 * l1v;
            const bool empty_row = !(L > 0.f);
            const float inv = empty_row ? 0.f : 1.f / L;
            const float lse2 = empty_row ? -INFINITY : M + fast_log2(L);
            const float a0 = w0 * inv, a1 = w1 * inv;
            umma::fence_after_sync();
            float o[64];  // this thread's columns [64 grp, 64 grp + 64) of the merged row
#pragma unroll
            for (int cblk = 0; cblk < 2; ++cblk) {
                uint32_t r0[32], r1[32];
                umma::tmem_ld32(tmem + kColO + grp * 64 + cblk * 32 + lane_off, r0);
                umma::tmem_ld32(tmem + kColO + kD + grp * 64 + cblk * 32 + lane_off, r1);
                umma::tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    const float x0 = a0 > 0.f ? __uint_as_float(r0[j]) * a0 : 0.f;
                    const float x1 = a1 > 0.f ? __uint_as_float(r1[j]) * a1 : 0.f;
                    o[cblk * 32 + j] = x0 + x1;
                }
            }
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) mbar_arrive(B.o_free);
            if (threadIdx.x == 0) trace(a, IT_EPI, n);

            const int unit = w.b * Hkv + w.g;
            const int u0 = a.unit_item_ptr[unit], n_items = a.unit_item_ptr[unit + 1] - u0;
            if (valid_row) {
                if (n_items == 1) {
                    const size_t orow = (q_row_base(a, rq) + qi) * a.n_q_heads + h;
                    if (a.o_dtype == EP_BF16) {
                        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(a.o) + orow * kD + grp * 64);
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            dst[c] = make_uint4(pack_bf16(o[8 * c], o[8 * c + 1]), pack_bf16(o[8 * c + 2], o[8 * c + 3]),
                                                pack_bf16(o[8 * c + 4], o[8 * c + 5]), pack_bf16(o[8 * c + 6], o[8 * c + 7]));
                    } else {
                        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.o) + orow * kD + grp * 64);
#pragma unroll
                        for (int c = 0; c < 16; ++c)
                            dst[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                    }
                    if (grp == 0 && a.lse) a.lse[orow] = lse2 * kLn2;
                } else {
                    float4* dst = reinterpret_cast<float4*>(a.o_part + (size_t(it) * rows + v) * kD + grp * 64);
#pragma unroll
                    for (int c = 0; c < 16; ++c)
                        dst[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                    if (grp == 0) a.lse_part[size_t(it) * rows + v] = lse2;
                }
            }
            if (threadIdx.x == 0) trace(a, IT_OUT, n);
            if (n_items > 1) {
                // Fused K2: the last CTA to finish one of this unit's items merges
                // them in page (= segment) order (attention.cpp:128-144).
                __threadfence();
                named_bar_sync(5, kSoftThreads);
                if (threadIdx.x == 0) *s_flag = atomicAdd(&a.unit_counter[unit], 1) == n_items - 1;
                named_bar_sync(5, kSoftThreads);
                if (*s_flag) {
                    __threadfence();
                    merge_unit_rows<kD>(a, u0, n_items, rows, nrows, warp, kSoftWarps, [&](int r) {
                        const int rq2 = w.rq0 + r / rpr, qi2 = (r % rpr) / G, h2 = w.g * G + r % G;
                        return (q_row_base(a, rq2) + qi2) * a.n_q_heads + h2;
                    });
                    if (threadIdx.x == 0) a.unit_counter[unit] = 0;
                }
                named_bar_sync(5, kSoftThreads);
            }
            if (threadIdx.x == 0) trace(a, IT_END, n);
        }
    }

    umma::fence_before_sync();
    __syncthreads();
    if (warp == kMmaWarp) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, kTmemCols);
    }
    if (a.trace && threadIdx.x == 0 && blockIdx.x < kTraceBlocks) {  // debug: per-CTA end (ns), work
        a.trace[18 * kTraceBlocks + 2 * blockIdx.x + 1] = globaltimer_ns();
        unsigned long long nb = 0;
        for (int it = it0; it < it1; ++it) nb += a.items[it].nblk;
        a.trace[20 * kTraceBlocks + 2 * blockIdx.x] = it1 - it0;
        a.trace[20 * kTraceBlocks + 2 * blockIdx.x + 1] = nb;
    }
}

}  // namespace

bool verify_supported(int kv_dtype, int d_head, int rows) {
    return kv_dtype == EP_BF16 && d_head == kD && rows >= 1 && rows <= kMaxRows;
}

cudaError_t launch_verify_attention(int n_ctas, const DecodeArgs& a, const CUtensorMap& tk,
                                    const CUtensorMap& tv, int rows, cudaStream_t s) {
    if (cudaError_t e = ensure_smem<verify_attention_kernel>(kSmem)) return e;
    if (n_ctas > 0) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(n_ctas);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, verify_attention_kernel, a, tk, tv, rows);
    }
    return cudaGetLastError();
}

}  // namespace ep
