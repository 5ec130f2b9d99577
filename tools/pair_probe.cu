// pair_probe.cu -- CTA-pair (cta_group::2) mechanics and throughput on B200: a cluster of
// 2 CTAs, each TMA-loading half of A (128 rows) and half of B (128 rows) into its own
// shared memory, the leader issuing tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 64),
// a multicast commit to both CTAs, each CTA reading its 128 TMEM lanes.  Checks D = A B^T
// against a host GEMM, then times back-to-back MMAs (pair vs single CTA).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pair_probe.cu -o tools/pair_probe -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2006_08861_b200/csrc/tc_ptx.cuh"
using namespace ol::tc;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

struct Smem {
    alignas(1024) __half a[128 * 64];
    alignas(1024) __half b[128 * 64];
    uint64_t full, tfull;
    uint32_t tmem;
};

template <bool kPair, int NB = 128>
__global__ void __launch_bounds__(256, 1) probe(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                                                 float *D, int reps, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem &s = *reinterpret_cast<Smem *>(raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = kPair ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        mbar_init(&s.full, 1);
        mbar_init(&s.tfull, 1);
        fence_mbar_init();
    }
    if (warp == 1) { if (kPair) tmem_alloc2<512>(&s.tmem); else tmem_alloc<512>(&s.tmem); }
    tc_fence_before();
    if (kPair) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    if (threadIdx.x == 0) {
        const uint32_t bytes = sizeof(s.a) + sizeof(s.b);
        if (rank == 0) mbar_expect_tx(&s.full, (kPair ? 2 : 1) * bytes);
        if (kPair) {
            tma_load_2d_pair(s.a, &ma, &s.full, 0, (int)rank * 128);
            tma_load_2d_pair(s.b, &mb, &s.full, 0, (int)rank * 128);
        } else {
            tma_load_2d(s.a, &ma, &s.full, 0, 0);
            tma_load_2d(s.b, &mb, &s.full, 0, 0);
        }
    }
    if (rank == 0 && threadIdx.x == 32) {
        mbar_wait(&s.full, 0);
        tc_fence_after();
        const uint32_t idesc = idesc_f16_f32(kPair ? 256 : 128, kPair ? 2 * NB : NB);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r)
            for (int k = 0; k < 4; ++k) {
                const uint64_t da = desc_sw128_kmajor(smem_u32(s.a) + k * 32), db = desc_sw128_kmajor(smem_u32(s.b) + k * 32);
                if (kPair) mma_f16_pair(tmem, da, db, idesc, k > 0 ? 1u : 0u);
                else mma_f16(tmem, da, db, idesc, k > 0 ? 1u : 0u);
            }
        if (kPair) mma_commit_pair(&s.tfull, 3); else mma_commit(&s.tfull);
        mbar_wait(&s.tfull, 0);
        cyc[0] = clock64() - t0;
    }
    // every CTA: warps 4..7 read the 128 lanes x N columns of D
    const int ncol = kPair ? 256 : 128;
    if (warp >= 4) {
        mbar_wait(&s.tfull, 0);
        tc_fence_after();
        const int q = warp & 3;
        for (int c = 0; c < ncol; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + c, v);
            tmem_ld_wait_regs(v);
            for (int j = 0; j < 32; ++j) D[(size_t)(rank * 128 + q * 32 + lane) * ncol + c + j] = __uint_as_float(v[j]);
        }
    }
    tc_fence_before();
    if (kPair) cluster_sync(); else __syncthreads();
    if (warp == 1) { if (kPair) tmem_dealloc2<512>(tmem); else tmem_dealloc<512>(tmem); }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}
static CUtensorMap make_map(void *ptr, uint64_t rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {64, rows};
    cuuint64_t strides[1] = {64 * sizeof(__half)};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    if (encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ptr, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n"); exit(1);
    }
    return m;
}

template <bool kPair, int NB = 128>
static void run(const CUtensorMap &ma, const CUtensorMap &mb, float *dD, long long *dc, int reps, int grid, size_t smem) {
    CK(cudaFuncSetAttribute(probe<kPair, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kPair ? 2 : 1; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, probe<kPair, NB>, ma, mb, dD, reps, dc));
    CK(cudaDeviceSynchronize());
}

int main() {
    const int R = 256;
    std::vector<__half> A(R * 64), B(R * 64);
    std::vector<float> Af(R * 64), Bf(R * 64);
    srand(3);
    for (int i = 0; i < R * 64; ++i) { A[i] = __float2half((rand() % 2001 - 1000) / 1000.f); Af[i] = __half2float(A[i]); }
    for (int i = 0; i < R * 64; ++i) { B[i] = __float2half((rand() % 2001 - 1000) / 1000.f); Bf[i] = __half2float(B[i]); }
    __half *dA, *dB; float *dD; long long *dc;
    CK(cudaMalloc(&dA, R * 64 * 2)); CK(cudaMalloc(&dB, R * 64 * 2)); CK(cudaMalloc(&dD, R * R * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), R * 64 * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), R * 64 * 2, cudaMemcpyHostToDevice));
    CUtensorMap ma = make_map(dA, R), mb = make_map(dB, R);
    const size_t smem = sizeof(Smem) + 1024;
    // correctness (1 rep) for the pair
    run<true>(ma, mb, dD, dc, 1, 2, smem);
    std::vector<float> D(R * R);
    CK(cudaMemcpy(D.data(), dD, R * R * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < R; ++i)
        for (int j = 0; j < R; ++j) {
            double ref = 0;
            for (int k = 0; k < 64; ++k) ref += (double)Af[i * 64 + k] * Bf[j * 64 + k];
            maxerr = fmax(maxerr, fabs(ref - D[i * R + j]));
        }
    printf("pair M256 N256 K64: max abs err vs host GEMM %.3e (D[0][0]=%f D[255][255]=%f)\n", maxerr, D[0], D[R * R - 1]);
    long long cyc;
    const int reps = 4096;
    run<true>(ma, mb, dD, dc, reps, 2, smem);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("pair:   %.1f cycles per M256xN256xK64 (per SM: M128xN256xK64)\n", (double)cyc / reps);
    run<false>(ma, mb, dD, dc, reps, 1, smem);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("single: %.1f cycles per M128xN128xK64\n", (double)cyc / reps);
    run<true, 80>(ma, mb, dD, dc, reps, 2, smem);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("pair N=160: %.1f cycles per M256xN160xK64 (ideal 320)\n", (double)cyc / reps);
    run<true, 64>(ma, mb, dD, dc, reps, 2, smem);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("pair N=128: %.1f cycles per M256xN128xK64 (ideal 256)\n", (double)cyc / reps);
    return 0;
}
