// tc_probe.cu -- standalone check of the tcgen05 / TMA / TMEM mechanics the
// tensor-core scan relies on (descriptors, swizzle, TMEM layout), plus
// micro-measurements of MMA and TMEM-load throughput on one SM.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo tools/tc_probe.cu -o tools/tc_probe -lcuda
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

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
    } while (0)

constexpr int M = 128, NQ = 256, K = 64;

struct Smem {
    alignas(1024) __half a[M * K];
    alignas(1024) __half b[NQ * K];
    uint64_t bar_tma, bar_mma;
    uint32_t tmem;
};

__global__ void probe_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                             float *D, int reps, long long *cycles, int mode) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem &s = *reinterpret_cast<Smem *>(raw);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        mbar_init(&s.bar_tma, 1);
        mbar_init(&s.bar_mma, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<256>(&s.tmem);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    if (threadIdx.x == 0) {
        mbar_expect_tx(&s.bar_tma, sizeof(s.a) + sizeof(s.b));
        tma_load_2d(s.a, &ma, &s.bar_tma, 0, 0);
        tma_load_2d(s.b, &mb, &s.bar_tma, 0, 0);
    }
    mbar_wait(&s.bar_tma, 0);
    const uint32_t idesc = idesc_f16_f32(M, NQ);
    long long t0 = clock64();
    uint32_t phase = 0;
    if (mode == 0 || mode == 1) {
        for (int r = 0; r < (mode == 0 ? 1 : reps); ++r) {
            if (threadIdx.x == 0) {
                tc_fence_after();
                for (int k = 0; k < K / 16; ++k) {
                    uint64_t da = desc_sw128_kmajor(smem_u32(s.a) + k * 32);
                    uint64_t db = desc_sw128_kmajor(smem_u32(s.b) + k * 32);
                    mma_f16(tmem, da, db, idesc, k > 0 ? 1u : 0u);
                }
                if (mode == 0 || (r % 16) == 15 || r == reps - 1) mma_commit(&s.bar_mma);
            }
            if (mode == 0 || (r % 16) == 15 || r == reps - 1) {
                mbar_wait(&s.bar_mma, phase);
                phase ^= 1;
            }
        }
        tc_fence_after();
    }
    if (mode == 4 || mode == 5) {   // N=128 (mode 4) / N=256 (mode 5) rounds of 10 / 5 MMAs
        const int NN = mode == 4 ? 128 : 256;
        const uint32_t id2 = idesc_f16_f32(M, NN);
        for (int r = 0; r < reps; ++r) {
            if (threadIdx.x == 0) {
                tc_fence_after();
                const int nm = mode == 4 ? 10 : 5;
                for (int i = 0; i < nm; ++i) {
                    uint64_t da = desc_sw128_kmajor(smem_u32(s.a) + (i % 4) * 32);
                    uint64_t db = desc_sw128_kmajor(smem_u32(s.b) + (i % 4) * 32);
                    mma_f16(tmem + (mode == 4 ? (i / 5) * 128 : 0), da, db, id2, (i % 5) > 0 ? 1u : 0u);
                }
                if ((r % 16) == 15 || r == reps - 1) mma_commit(&s.bar_mma);
            }
            if ((r % 16) == 15 || r == reps - 1) { mbar_wait(&s.bar_mma, phase); phase ^= 1; }
        }
        tc_fence_after();
    }
    long long t1 = clock64();
    if (mode == 2) {  // TMEM load throughput: all 4 warps read all 256 columns, reps times
        uint32_t acc = 0;
        for (int r = 0; r < reps; ++r) {
            for (int c = 0; c < NQ; c += 32) {
                uint32_t v[32];
                tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc ^= v[j];
            }
        }
        t1 = clock64();
        if (acc == 0x12345678) D[0] = 1;  // keep
    }
    if (mode == 3) {  // 8 warps: quarter = warp % 4, half = warp / 4; 4 loads in flight per wait
        uint32_t acc = 0;
        const uint32_t q = warp % 4, h = warp / 4;
        for (int r = 0; r < reps; ++r) {
            uint32_t v0[32], v1[32], v2[32], v3[32];
            uint32_t base = tmem + ((q * 32) << 16) + h * 128;
            tmem_ld32(base + 0, v0);
            tmem_ld32(base + 32, v1);
            tmem_ld32(base + 64, v2);
            tmem_ld32(base + 96, v3);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v0[j] + v1[j] + v2[j] + v3[j];
        }
        t1 = clock64();
        if (acc == 0x12345678) D[0] = 1;
    }
    if (threadIdx.x == 0) cycles[0] = t1 - t0;
    // write D out: thread = row (TMEM lane), 8 chunks of 32 columns
    if (mode == 0 && warp < 4) {
        for (int c = 0; c < NQ; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c, v);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * NQ + c + j] = __uint_as_float(v[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<256>(tmem);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

static CUtensorMap make_map(void *ptr, uint64_t rows, uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {K, rows};
    cuuint64_t strides[1] = {K * sizeof(__half)};
    cuuint32_t box[2] = {K, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, ptr, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
    return m;
}

int main() {
    std::vector<__half> A(M * K), B(NQ * K);
    std::vector<float> Af(M * K), Bf(NQ * K);
    srand(1);
    for (int i = 0; i < M * K; ++i) { A[i] = __float2half((rand() % 1000) / 1000.f); Af[i] = __half2float(A[i]); }
    for (int i = 0; i < NQ * K; ++i) { B[i] = __float2half((rand() % 1000) / 1000.f); Bf[i] = __half2float(B[i]); }
    __half *dA, *dB;
    float *dD;
    long long *dc;
    CK(cudaMalloc(&dA, A.size() * 2));
    CK(cudaMalloc(&dB, B.size() * 2));
    CK(cudaMalloc(&dD, M * NQ * 4));
    CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice));
    CUtensorMap ma = make_map(dA, M, M), mb = make_map(dB, NQ, NQ);
    size_t smem = sizeof(Smem) + 1024;
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    probe_kernel<<<1, 128, smem>>>(ma, mb, dD, 1, dc, 0);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(M * NQ);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0;
    for (int i = 0; i < M; ++i)
        for (int j = 0; j < NQ; ++j) {
            double ref = 0;
            for (int k = 0; k < K; ++k) ref += (double)Af[i * K + k] * Bf[j * K + k];
            maxerr = fmax(maxerr, fabs(ref - D[i * NQ + j]) / fmax(1e-6, fabs(ref)));
        }
    printf("correctness: max rel err %.3e  (D[0][0]=%f)\n", maxerr, D[0]);
    long long cyc;
    int reps = 4096;
    probe_kernel<<<1, 128, smem>>>(ma, mb, dD, reps, dc, 1);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    double flops = 2.0 * M * NQ * K * reps;
    printf("mma: %lld cycles for %d x (128x256x64): %.1f flop/cycle/SM (%.1f cycles per 128x256x64)\n", cyc,
           reps, flops / cyc, (double)cyc / reps);
    reps = 256;
    probe_kernel<<<1, 128, smem>>>(ma, mb, dD, reps, dc, 2);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("tmem ld (4 warps, wait after each x32): %lld cycles for %d x 128 KB: %.1f B/cycle\n", cyc, reps,
           128.0 * 1024 * reps / cyc);
    // many CTAs: aggregate MMA throughput
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    reps = 8192;
    cudaEventRecord(e0);
    probe_kernel<<<148, 128, smem>>>(ma, mb, dD, reps, dc, 1);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("148 CTAs mma: %.3f ms -> %.1f TFLOP/s fp16\n", ms, 2.0 * M * NQ * K * reps * 148 / ms / 1e9);
    cudaEventRecord(e0);
    probe_kernel<<<148, 128, smem>>>(ma, mb, dD, 2048, dc, 2);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
    printf("148 CTAs tmem ld: %.3f ms -> %.1f TB/s total\n", ms, 128.0 * 1024 * 2048 * 148 / ms / 1e9);
    for (int mode = 4; mode <= 5; ++mode) {
        reps = 2048;
        probe_kernel<<<1, 128, smem>>>(ma, mb, dD, reps, dc, mode);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
        printf("mode %d (%s): %.1f cycles per round (32768 x K80 pairs)\n", mode,
               mode == 4 ? "10 x M128N128K16" : "5 x M128N256K16", (double)cyc / reps);
    }
    CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    reps = 256;
    probe_kernel<<<1, 256, smem>>>(ma, mb, dD, reps, dc, 3);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("tmem ld (8 warps, 4 x32 in flight): %lld cycles for %d x 128 KB: %.1f B/cycle\n", cyc, reps,
           128.0 * 1024 * reps / cyc);
    cudaEventRecord(e0);
    probe_kernel<<<148, 256, smem>>>(ma, mb, dD, 2048, dc, 3);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
    printf("148 CTAs tmem ld 8 warps: %.3f ms -> %.1f TB/s total\n", ms, 128.0 * 1024 * 2048 * 148 / ms / 1e9);
    return 0;
}
