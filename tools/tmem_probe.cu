// tmem_probe.cu -- tcgen05.ld (TMEM -> registers) throughput on one SM, by load shape
// and warp count, with and without a concurrent stream of tcgen05.mma writing the
// other half of TMEM (the tensor-core scan's epilogue regime).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tmem_probe.cu -o tools/tmem_probe -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_08861_b200/csrc/tc_ptx.cuh"
using namespace ol::tc;

#define R8(b) "=r"(r[b]), "=r"(r[b + 1]), "=r"(r[b + 2]), "=r"(r[b + 3]), "=r"(r[b + 4]), "=r"(r[b + 5]), "=r"(r[b + 6]), "=r"(r[b + 7])
__device__ __forceinline__ void ld64(uint32_t t, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,"
        "%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : R8(0), R8(8), R8(16), R8(24), R8(32), R8(40), R8(48), R8(56)
        : "r"(t));
}

struct Smem {
    alignas(1024) __half a[128 * 64];
    alignas(1024) __half b[256 * 64];
    uint64_t bar;
    uint32_t tmem;
    uint32_t stop;
};

// mode 0: x32 x2 per wait; 1: x64 per wait; 2: x32 x4 per wait.  mma: 1 = thread 0 of
// the last warp issues back-to-back 128x256x16 MMAs into columns 256..511.
__global__ void probe(int mode, int mma, int reps, long long *out) {
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem &s = *reinterpret_cast<Smem *>(raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) s.a[i] = __float2half(0.001f * (i % 7));
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) s.b[i] = __float2half(0.001f * (i % 5));
    if (threadIdx.x == 0) { s.stop = 0; mbar_init(&s.bar, 1); fence_mbar_init(); }
    if (warp == 0) tmem_alloc<512>(&s.tmem);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem;
    const int loaders = mma ? nw - 1 : nw;
    long long t0 = clock64();
    if (warp < loaders) {
        const uint32_t q = warp & 3, part = warp >> 2;   // lanes 32q.., a slice of columns
        const uint32_t parts = (loaders + 3) / 4;
        const uint32_t cols = 256 / parts;
        uint32_t acc = 0;
        unsigned long long nbytes = 0;
        for (int r = 0; r < reps; ++r) {
            for (uint32_t c = 0; c < cols; c += (mode == 2 ? 128 : 64)) {
                nbytes += 32ull * 4 * (mode == 2 ? 128 : 64);
                const uint32_t ta = tmem + ((q * 32) << 16) + part * cols + c;
                if (mode == 1) {
                    uint32_t v[64];
                    ld64(ta, v);
                    tmem_ld_wait_regs(*reinterpret_cast<uint32_t(*)[32]>(v));
                    reg_fence(*reinterpret_cast<uint32_t(*)[32]>(v + 32));
                    for (int j = 0; j < 64; ++j) acc += v[j];
                } else if (mode == 0) {
                    uint32_t v0[32], v1[32];
                    tmem_ld32(ta, v0);
                    tmem_ld32(ta + 32, v1);
                    tmem_ld_wait_regs(v0);
                    reg_fence(v1);
                    for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
                } else {
                    uint32_t v0[32], v1[32], v2[32], v3[32];
                    tmem_ld32(ta, v0); tmem_ld32(ta + 32, v1); tmem_ld32(ta + 64, v2); tmem_ld32(ta + 96, v3);
                    tmem_ld_wait_regs(v0); reg_fence(v1); reg_fence(v2); reg_fence(v3);
                    for (int j = 0; j < 32; ++j) acc += (v0[j] ^ v1[j]) + (v2[j] ^ v3[j]);
                }
            }
        }
        if (acc == 0x12345u) out[4] = acc;
        if ((threadIdx.x & 31) == 0) {
            atomicAdd((unsigned long long *)&out[0], (unsigned long long)(clock64() - t0));
            atomicAdd((unsigned long long *)&out[3], nbytes);
        }
        __syncwarp();
        if (threadIdx.x == 0) atomicExch(&s.stop, 1u);
    } else if (threadIdx.x == blockDim.x - 32) {
        const uint32_t idesc = idesc_f16_f32(128, 256);
        long long n = 0;
        while (!*(volatile uint32_t *)&s.stop) {
            for (int k = 0; k < 16; ++k, ++n)
                mma_f16(tmem + 256, desc_sw128_kmajor(smem_u32(s.a) + (k & 3) * 32),
                        desc_sw128_kmajor(smem_u32(s.b) + (k & 3) * 32), idesc, (k & 3) ? 1u : 0u);
        }
        mma_commit(&s.bar);
        mbar_wait(&s.bar, 0);
        out[1] = n;
        out[2] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long *d;
    cudaMalloc(&d, 64);
    size_t smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const char *names[] = {"x32 x2 / wait", "x64 / wait", "x32 x4 / wait"};
    for (int mma = 0; mma <= 1; ++mma)
        for (int nw : {8, 16})
            for (int mode = 0; mode < 3; ++mode) {
                long long h[4] = {0, 0, 0, 0};
                cudaMemset(d, 0, 64);
                const int reps = 400;
                probe<<<1, 32 * (nw + mma), smem>>>(mode, mma, reps, d);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
                const double cyc = (double)h[0] / nw;          // mean per loading warp
                const double bytes = (double)h[3];
                printf("mma=%d warps=%2d %-14s: %.1f B/cycle  (%.0f cycles per 128 KB)\n", mma, nw, names[mode],
                       bytes / cyc, 131072.0 / (bytes / cyc));
                if (mma) printf("      concurrent MMAs: %lld in %lld cycles = %.1f cycles per 128x256x16\n", h[1], h[2],
                                (double)h[2] / (h[1] ? h[1] : 1));
            }
    return 0;
}
