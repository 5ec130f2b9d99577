// pipe_probe2.cu -- round 2: which MMA -> TMEM -> epilogue pipeline shape reads the
// accumulators fastest?  One CTA, one thread issues K = 32 (2 x K16) MMAs M = 128 x N = TC into
// NB TMEM buffers of TC columns; G groups of 16/G epilogue warps take tiles round-robin; every
// warp reads CW = TC * 4 * G / 16 columns of its 32 lanes per tile (x16 loads, up to 64
// registers per round, one tcgen05.wait::ld per round), releases the buffer, then does the
// compare math (an FMNMX3 chain, like tcscan).  Prints cycles per 256 accumulator columns
// (128 KB): tcscan today is NB = 2, TC = 256, G = 2 (843 cycles in round 1).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pipe_probe2.cu -o tools/pipe_probe2
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_08861_b200/csrc/tc_ptx.cuh"
using namespace ol::tc;

__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t *r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}
template <int N>
__device__ __forceinline__ void wait_ld(uint32_t (&r)[N]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < N; ++i) asm volatile("" : "+r"(r[i]));
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

struct Smem {
    alignas(1024) __half a[128 * 64];
    alignas(1024) __half b[256 * 64];
    uint64_t tfull[8], tempty[8], dummy[8];
    alignas(16) float2 bnd[16][8];
    uint32_t tau[128];
    uint32_t tmem;
};

template <int NB, int TC, int G, bool SPIN, int LDG = 0>
__global__ void __launch_bounds__(640, 1) probe(int mma, int tiles, long long *out, const float2 *gsrc, int extra) {
    constexpr int WPG = 16 / G;            // warps per group
    constexpr int CW = TC * 4 / WPG;       // columns per warp per tile
    constexpr int R1 = CW > 64 ? 64 : CW;  // first round
    constexpr int R2 = CW - R1;
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem &s = *reinterpret_cast<Smem *>(raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) s.a[i] = __float2half(0.001f * (i % 7));
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) s.b[i] = __float2half(0.001f * (i % 5));
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], WPG); }
        for (int i = 0; i < 8; ++i) mbar_init(&s.dummy[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 128; i += blockDim.x) s.tau[i] = 0x3f000000u;
    for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) s.bnd[i / 8][i % 8] = make_float2(0.5f, 0.001f);
    if (warp == 0) tmem_alloc<512>(&s.tmem);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    long long t0 = clock64();
    if (warp == 0) {
        if (lane == 0) {
            const uint32_t idesc = idesc_f16_f32(128, TC);
            for (int t = 0; t < tiles; ++t) {
                const int buf = t % NB;
                if (t >= NB) mbar_wait(&s.tempty[buf], ((t / NB) - 1) & 1);
                tc_fence_after();
                if (mma)
                    for (int k = 0; k < 2; ++k) {
                        if (extra & 4)   // the 64-byte plane (tcscan at kf = 32): SW64 K-major operands
                            mma_f16(tmem + buf * TC, desc_sw64_kmajor(smem_u32(s.a) + k * 32),
                                    desc_sw64_kmajor(smem_u32(s.b) + k * 32), idesc, k ? 1u : 0u);
                        else
                            mma_f16(tmem + buf * TC, desc_sw128_kmajor(smem_u32(s.a) + k * 32),
                                    desc_sw128_kmajor(smem_u32(s.b) + k * 32), idesc, k ? 1u : 0u);
                    }
                if (LDG == 3) mma_commit(&s.dummy[t & 7]);   // a second commit per tile (tcscan frees the TMA stage)
                mma_commit(&s.tfull[buf]);
            }
        }
    } else if (warp <= 16) {
        const int ew = warp - 1, q = warp & 3;
        const int grp = ew / WPG, slice = (ew % WPG) >> 2;
        float m0 = 0.f, m1 = 0.f;
        float2 pA = make_float2(0.f, 0.f), pB = pA;   // LDG variants: a load consumed 2 own tiles later
        for (int t = grp; t < tiles; t += G) {
            if (LDG == 1) {   // load issued at tile start, consumed two own tiles later (ping-pong registers)
                float2 &p = ((t / G) & 1) ? pB : pA;
                m0 += p.x;
                p = __ldg(&gsrc[(t * 16 + ew) * 4 + (lane & 3)]);
            }
            if (LDG == 2 && lane == 0) m1 += __ldcg(&gsrc[t]).x;   // load consumed in the same tile
            const int buf = t % NB;
            if (SPIN) mbar_wait(&s.tfull[buf], (t / NB) & 1);
            else mbar_wait_sleep(&s.tfull[buf], (t / NB) & 1);
            tc_fence_after();
            float th0 = 0.f, th1 = 0.f;
            uint32_t gt = 0;
            if (extra & 1) {
                const int ql = q * 32 + lane;
                if (slice == 0 && grp == 0) gt = __ldcg(reinterpret_cast<const uint32_t *>(gsrc) + ql);
                const float h = 0.5f * (1.0f - __uint_as_float(((volatile uint32_t *)s.tau)[ql]) * 1.0000076f);
                const float4 *bp = reinterpret_cast<const float4 *>(&s.bnd[t & 15][slice * 4]);
                const float4 b01 = bp[0], b23 = bp[1];
                th0 = __fadd_rd(h, __fsub_rd(b01.x, __fmul_ru(0.5f, b01.y)));
                th1 = __fadd_rd(h, __fsub_rd(b23.z, __fmul_ru(0.5f, b23.w)));
            }
            const uint32_t ta = tmem + ((q * 32) << 16) + buf * TC + slice * CW;
            uint32_t v[R1];
#pragma unroll
            for (int c = 0; c < R1; c += 16) ld16(ta + c, v + c);
            wait_ld(v);
            if (R2 == 0) { tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]); }
#pragma unroll
            for (int j = 0; j + 3 < R1; j += 4) {
                m0 = max3f(m0, __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
                m1 = max3f(m1, __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
            }
            if ((extra & 1) && fmaxf(m0, m1) >= th0 + 1e30f) out[2] = 1;
            if (R2 > 0) {
                uint32_t w[R2 > 0 ? R2 : 1];
#pragma unroll
                for (int c = 0; c < R2; c += 16) ld16(ta + R1 + c, w + c);
                wait_ld(w);
                tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]);
#pragma unroll
                for (int j = 0; j + 3 < R2; j += 4) {
                    m0 = max3f(m0, __uint_as_float(w[j]), __uint_as_float(w[j + 1]));
                    m1 = max3f(m1, __uint_as_float(w[j + 2]), __uint_as_float(w[j + 3]));
                }
                if ((extra & 1) && fmaxf(m0, m1) >= th1 + 1e30f) out[2] = 1;
            }
            if ((extra & 1) && gt != 0 && gt < ((volatile uint32_t *)s.tau)[q * 32 + lane]) atomicMin(&s.tau[q * 32 + lane], gt);
        }
        if (m0 + m1 == 1234.5f) out[3] = 1;
    } else if (warp >= 17 && (extra & 2)) {
        // idle warps like tcscan's exact warps: poll + nanosleep with backoff
        uint32_t nap = 32;
        while (clock64() - t0 < 2000000000ll && !(((volatile uint32_t *)s.tau)[0] == 0xdeadbeefu)) {
            if (((volatile uint32_t *)s.tau)[1] == 0xdeadbeefu) break;
            if (clock64() - t0 > (long long)tiles * 460) break;
            __nanosleep(nap); if (nap < 1024) nap <<= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int NB, int TC, int G, bool SPIN, int LDG = 0>
void run(long long *d, const char *name, int extra = 0, int grid = 1) {
    size_t smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(probe<NB, TC, G, SPIN, LDG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    static float2 *g = nullptr;
    if (!g) { cudaMalloc(&g, sizeof(float2) * 1 << 20); cudaMemset(g, 0, sizeof(float2) * 1 << 20); }
    const int tiles = 960;
    for (int mma = 0; mma <= 1; ++mma) {
        long long h[4] = {0, 0, 0, 0};
        probe<NB, TC, G, SPIN, LDG><<<grid, (extra & 2) ? 32 * 20 : 32 * 17, smem>>>(mma, tiles, d, g, extra);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("NB=%d TC=%3d G=%d %s ldg=%d extra=%d grid=%d mma=%d %-28s: %6.0f cycles per 256 columns\n", NB, TC, G,
               SPIN ? "spin " : "sleep", LDG, extra, grid, mma, name, (double)h[0] / tiles * 256.0 / TC);
    }
}

int main() {
    long long *d;
    cudaMalloc(&d, 64);
    run<2, 256, 2, false, 0>(d, "SW128 operands", 0, 1);
    run<2, 256, 2, false, 0>(d, "SW64 operands", 4, 1);
    run<2, 256, 2, false, 3>(d, "148 CTAs + both, SW128", 3, 148);
    run<2, 256, 2, false, 3>(d, "148 CTAs + both, SW64", 7, 148);
    return 0;
}
