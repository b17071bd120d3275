// gemm_probe.cu — isolates the K4 score-GEMM mainloop (TMA ring + tcgen05
// 1-SM MMAs, K-major bf16 A [rows x K] and W [vocab x K], 128B swizzle) to
// find what bounds its per-k-block time. Modes:
//   0 full: TMA fills, MMAs consume, commit frees the stage
//   1 tma-only: the MMA thread waits each fill and frees the stage directly
//   2 mma-only: no loads; MMAs run on whatever is in shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//        -I paper_2504_11729_b200/csrc tools/gemm_probe.cu -o gpurun_out/gemm_probe
// Usage: gemm_probe rows vocab K tn stages mode [ctas_per_sm]
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace ep;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);

static void encode(CUtensorMap* map, void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {inner * 2};
    const cuuint32_t box[2] = {bi, bo};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        printf("encode failed %d\n", int(r));
        exit(1);
    }
}

struct Args {
    int tn, stages, nk, mode, variant;
    uint32_t idesc, idesc_half, idesc_m64;
    float* out;
    unsigned long long* t;  // [issue start, issue end, accumulator ready] (clock64)
};

constexpr int kTK = 64, kABytes = 128 * kTK * 2;

__global__ void __launch_bounds__(128) probe_kernel(const Args a, const __grid_constant__ CUtensorMap ta,
                                                    const __grid_constant__ CUtensorMap tw) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int TN = a.tn, NS = a.stages, kStage = kABytes + TN * kTK * 2;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * kStage);
    uint64_t* empty = full + 16;
    uint64_t* acc = empty + 16;
    uint32_t* slot = reinterpret_cast<uint32_t*>(acc + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * 128, n0 = blockIdx.y * TN;
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(acc, 1);
        fence_mbar_init();
    }
    if (warp == 1) umma::tmem_alloc(slot, 512);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = *slot;
    if (warp == 0) {
        if (lane == 0 && a.mode != 2) {
            for (int kb = 0; kb < a.nk; ++kb) {
                const int s = kb % NS;
                mbar_wait(&empty[s], ((kb / NS) & 1) ^ 1);
                mbar_arrive_expect_tx(&full[s], kABytes + TN * kTK * 2);
                uint8_t* dst = smem + s * kStage;
                umma::tma_load_2d(dst, &ta, kb * kTK, m0, &full[s], l2_policy_evict_last());
                umma::tma_load_2d(dst + kABytes, &tw, kb * kTK, n0, &full[s], l2_policy_evict_last());
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t base = smem_u32(smem);
            if (blockIdx.x == 0 && blockIdx.y == 0) a.t[0] = clock64();
            for (int kb = 0; kb < a.nk; ++kb) {
                const int s = kb % NS;
                if (a.mode != 2) mbar_wait(&full[s], (kb / NS) & 1);
                if (!(a.variant & 16)) umma::fence_after_sync();
                if (a.mode == 1) {
                    mbar_arrive(&empty[s]);
                    continue;
                }
                const uint32_t aa = base + s * kStage, ba = aa + kABytes;
                if ((a.variant & 15) == 1) {  // two N/2 MMAs into separate accumulators
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk) {
                        const uint64_t ad = umma::smem_desc_sw128(aa + kk * 32, 16, 1024);
                        umma::mma_bf16_ss(tmem, ad, umma::smem_desc_sw128(ba + kk * 32, 16, 1024), a.idesc_half,
                                          (kb | kk) ? 1u : 0u);
                        umma::mma_bf16_ss(tmem + TN / 2, ad,
                                          umma::smem_desc_sw128(ba + (TN / 2) * 128 + kk * 32, 16, 1024),
                                          a.idesc_half, (kb | kk) ? 1u : 0u);
                    }
                } else if ((a.variant & 15) == 2) {  // alternate accumulators per k-block
                    const uint32_t d = tmem + uint32_t(kb & 1) * TN;
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk)
                        umma::mma_bf16_ss(d, umma::smem_desc_sw128(aa + kk * 32, 16, 1024),
                                          umma::smem_desc_sw128(ba + kk * 32, 16, 1024), a.idesc,
                                          (kb >= 2 || kk) ? 1u : 0u);
                } else if ((a.variant & 15) == 3) {  // alternate accumulators per K16 step
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk)
                        umma::mma_bf16_ss(tmem + uint32_t(kk & 1) * TN, umma::smem_desc_sw128(aa + kk * 32, 16, 1024),
                                          umma::smem_desc_sw128(ba + kk * 32, 16, 1024), a.idesc,
                                          (kb || kk >= 2) ? 1u : 0u);
                } else if ((a.variant & 15) == 4) {  // A from TMEM (columns 256 +)
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk)
                        umma::mma_bf16_ts(tmem, tmem + 256 + kk * 8, umma::smem_desc_sw128(ba + kk * 32, 16, 1024),
                                          a.idesc, (kb | kk) ? 1u : 0u);
                } else if ((a.variant & 15) == 5) {  // M = 64
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk)
                        umma::mma_bf16_ss(tmem, umma::smem_desc_sw128(aa + kk * 32, 16, 1024),
                                          umma::smem_desc_sw128(ba + kk * 32, 16, 1024), a.idesc_m64,
                                          (kb | kk) ? 1u : 0u);
                } else {
#pragma unroll
                    for (int kk = 0; kk < kTK / 16; ++kk)
                        umma::mma_bf16_ss(tmem, umma::smem_desc_sw128(aa + kk * 32, 16, 1024),
                                          umma::smem_desc_sw128(ba + kk * 32, 16, 1024), a.idesc,
                                          (kb | kk) ? 1u : 0u);
                }
                if (!(a.variant & 32) || kb == a.nk - 1) umma::mma_commit(&empty[s]);
            }
            if (blockIdx.x == 0 && blockIdx.y == 0) a.t[1] = clock64();
            if (a.mode == 1) mbar_arrive(acc);
            else umma::mma_commit(acc);
        }
    } else if (warp >= 2) {
        mbar_wait(acc, 0);
        umma::fence_after_sync();
        if (threadIdx.x == 64 && blockIdx.x == 0 && blockIdx.y == 0) a.t[2] = clock64();
        if (warp == 2) {
            uint32_t r[32];
            umma::tmem_ld32(tmem + ((uint32_t(warp & 3) * 32) << 16), r);
            umma::tmem_wait_ld();
            float s = 0.f;
            for (int i = 0; i < 32; ++i) s += __uint_as_float(r[i]);
            if (s == 12345.f) a.out[blockIdx.x] = s;
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (warp == 1) {
        umma::fence_after_sync();
        umma::tmem_dealloc(tmem, 512);
    }
}

int main(int argc, char** argv) {
    if (argc < 7) {
        printf("usage: gemm_probe rows vocab K tn stages mode\n");
        return 1;
    }
    const int rows = atoi(argv[1]), vocab = atoi(argv[2]), K = atoi(argv[3]), tn = atoi(argv[4]),
              stages = atoi(argv[5]), mode = atoi(argv[6]), variant = argc > 7 ? atoi(argv[7]) : 0;
    void *A, *W;
    float* out;
    cudaMalloc(&A, size_t(rows) * K * 2);
    cudaMalloc(&W, size_t(vocab) * K * 2);
    cudaMalloc(&out, 4096);
    unsigned long long* t;
    cudaMallocManaged(&t, 64);
    cudaMemset(A, 0x3c, size_t(rows) * K * 2);
    cudaMemset(W, 0x3c, size_t(vocab) * K * 2);
    CUtensorMap ta, tw;
    encode(&ta, A, K, rows, 64, 128);
    encode(&tw, W, K, vocab, 64, tn);
    Args a{tn,    stages, K / kTK, mode, variant, umma::idesc_bf16_f32(128, tn, false, false),
           umma::idesc_bf16_f32(128, tn / 2, false, false), umma::idesc_bf16_f32(64, tn, false, false), out, t};
    const int smem = stages * (kABytes + tn * kTK * 2) + 1024 + 512;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dim3 grid((rows + 127) / 128, (vocab + tn - 1) / tn);
    for (int i = 0; i < 5; ++i) probe_kernel<<<grid, 128, smem>>>(a, ta, tw);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int it = 50;
    cudaEventRecord(e0);
    for (int i = 0; i < it; ++i) probe_kernel<<<grid, 128, smem>>>(a, ta, tw);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaError_t err = cudaGetLastError();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1000.0 / it;
    probe_kernel<<<grid, 128, smem>>>(a, ta, tw);
    cudaDeviceSynchronize();
    const double issue = double(t[1] - t[0]) / a.nk, done = double(t[2] - t[0]) / a.nk;
    const double flop = 2.0 * grid.x * 128.0 * grid.y * tn * K;
    printf("v%d rows=%d vocab=%d K=%d tn=%d stages=%d mode=%d grid=%dx%d smem=%d: %.2f us/launch, %.3f us/kblock, "
           "%.0f TF/s (padded); cta0 clk/kblock issue %.0f done %.0f %s\n",
           variant, rows, vocab, K, tn, stages, mode, grid.x, grid.y, smem, us, us / (K / kTK), flop / us * 1e-6, issue, done,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    return 0;
}
