// pipe_probe.cu -- the tensor-core scan's TMEM pipeline in isolation: one thread issues
// (optionally) 4 MMAs 128x256x16 per tile into a double-buffered accumulator and commits
// tfull[buf]; epilogue warps wait tfull, tcgen05.ld their share, arrive tempty[buf].
// Compares "all warps on every tile" with "two groups on alternate tiles" (2 x 256-column
// buffers, each warp two 64-column chunks) and "two groups on alternate tiles over 4 x 128-column
// buffers" (design 2: each warp one 64-column chunk, released before its math); kst = K/16 steps.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/pipe_probe.cu -o tools/pipe_probe -lcuda
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../paper_2006_08861_b200/csrc/tc_ptx.cuh"
using namespace ol::tc;

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}

__device__ __forceinline__ void reg_fence16(uint32_t (&r)[16]) {
    asm volatile("" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                      "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]));
}

struct Smem {
    alignas(1024) __half a[128 * 64];
    alignas(1024) __half b[256 * 64];
    uint64_t tfull[4], tempty[4];
    uint32_t tmem;
};

// design 0: E warps all load every tile, each 256*4/E columns... (E = 16: 64 columns)
// design 1: two groups of E/2 warps on alternate tiles, each warp 128 columns in two 64-col chunks
__global__ void __launch_bounds__(544, 1) probe(int design, int E, int mma, int tiles, int NB, int kst, long long *out) {
    const int TC = NB == 3 ? 160 : 512 / NB;   // columns per tile (NB = 3: 3 x 160 columns)
    extern __shared__ __align__(1024) unsigned char raw[];
    Smem &s = *reinterpret_cast<Smem *>(raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) s.a[i] = __float2half(0.001f * (i % 7));
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) s.b[i] = __float2half(0.001f * (i % 5));
    const int arrivals = design == 0 ? E : E / 2;
    if (threadIdx.x == 0) {
        for (int i = 0; i < (design == 5 ? 4 : NB); ++i) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], arrivals); }
        fence_mbar_init();
    }
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
            if (design == 5) {   // each tile as two N = 128 halves, each with its own handshake
                const uint32_t idh = idesc_f16_f32(128, 128);
                for (int t = 0; t < tiles; ++t) {
                    const int buf = t & 1;
                    for (int hb = 0; hb < 2; ++hb) {
                        if (t >= 2) mbar_wait(&s.tempty[2 * hb + buf], ((t >> 1) - 1) & 1);
                        tc_fence_after();
                        if (mma)
                            for (int k = 0; k < kst; ++k)
                                mma_f16(tmem + buf * 256 + hb * 128, desc_sw128_kmajor(smem_u32(s.a) + k * 32),
                                        desc_sw128_kmajor(smem_u32(s.b) + hb * 128 * 128 + k * 32), idh, k ? 1u : 0u);
                        mma_commit(&s.tfull[2 * hb + buf]);
                    }
                }
                out[1] = clock64() - t0;
            } else
            for (int t = 0; t < tiles; ++t) {
                const int buf = t % NB;
                if (t >= NB) mbar_wait(&s.tempty[buf], ((t / NB) - 1) & 1);
                tc_fence_after();
                if (mma)
                    for (int k = 0; k < kst; ++k)
                        mma_f16(tmem + buf * TC, desc_sw128_kmajor(smem_u32(s.a) + k * 32),
                                desc_sw128_kmajor(smem_u32(s.b) + k * 32), idesc, k ? 1u : 0u);
                mma_commit(&s.tfull[buf]);
            }
            out[1] = clock64() - t0;
        }
    } else if (warp <= E) {
        const int ew = warp - 1, q = warp & 3;
        uint32_t acc = 0;
        if (design == 0) {
            const int part = ew >> 2, cols = TC / (E / 4);
            for (int t = 0; t < tiles; ++t) {
                const int buf = t % NB;
                mbar_wait(&s.tfull[buf], (t / NB) & 1);
                tc_fence_after();
                for (int c = 0; c < cols; c += 64) {
                    uint32_t v0[32], v1[32];
                    const uint32_t ta = tmem + ((q * 32) << 16) + buf * TC + part * cols + c;
                    tmem_ld32(ta, v0);
                    if (cols - c >= 64) { tmem_ld32(ta + 32, v1); tmem_ld_wait_regs(v0); reg_fence(v1); }
                    else { tmem_ld_wait_regs(v0); for (int j = 0; j < 32; ++j) v1[j] = 0; }
                    for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&s.tempty[buf]);
            }
        } else if (design == 3) {
            // 3 buffers of 160 columns, two groups on alternate tiles: the MMA can run one tile
            // ahead of both groups; each warp reads 80 columns (x32 + x32 + x16, one wait)
            const int grp = ew / (E / 2), half = (ew % (E / 2)) >> 2;
            for (int t = grp; t < tiles; t += 2) {
                const int buf = t % 3;
                mbar_wait(&s.tfull[buf], (t / 3) & 1);
                tc_fence_after();
                uint32_t v0[32], v1[32], v2[16];
                const uint32_t ta = tmem + ((q * 32) << 16) + buf * TC + half * 80;
                tmem_ld32(ta, v0); tmem_ld32(ta + 32, v1); tmem_ld16(ta + 64, v2);
                tmem_ld_wait_regs(v0); reg_fence(v1); reg_fence16(v2);
                tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]);
                for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
                for (int j = 0; j < 16; ++j) acc += v2[j];
            }
        } else if (design == 5) {
            const int grp = ew / (E / 2), half = (ew % (E / 2)) >> 2;
            for (int t = grp; t < tiles; t += 2) {
                const int buf = t & 1;
                uint32_t v0[32], v1[32];
                for (int hb = 0; hb < 2; ++hb) {
                    mbar_wait(&s.tfull[2 * hb + buf], (t >> 1) & 1);
                    tc_fence_after();
                    const uint32_t ta = tmem + ((q * 32) << 16) + buf * 256 + hb * 128 + half * 64;
                    tmem_ld32(ta, v0); tmem_ld32(ta + 32, v1);
                    tmem_ld_wait_regs(v0); reg_fence(v1);
                    tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[2 * hb + buf]);
                    for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
                }
            }
        } else if (design == 2) {
            const int grp = ew / (E / 2), half = (ew % (E / 2)) >> 2;   // E/2 = 8: half in {0, 1}
            for (int t = grp; t < tiles; t += 2) {
                const int buf = t % NB;
                mbar_wait(&s.tfull[buf], (t / NB) & 1);
                tc_fence_after();
                uint32_t v0[32], v1[32];
                const uint32_t ta = tmem + ((q * 32) << 16) + buf * TC + half * 64;
                tmem_ld32(ta, v0); tmem_ld32(ta + 32, v1);
                tmem_ld_wait_regs(v0); reg_fence(v1);
                tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]);
                for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
            }
        } else {
            const int grp = ew / (E / 2), half = (ew % (E / 2)) >> 2;   // E/2 = 8: half in {0, 1}
            for (int t = grp; t < tiles; t += 2) {
                const int buf = t & 1;
                mbar_wait(&s.tfull[buf], (t >> 1) & 1);
                tc_fence_after();
                if (design == 4) {   // the handoff alone: no accumulator reads
                    tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]);
                    continue;
                }
                for (int c = 0; c < 128; c += 64) {
                    uint32_t v0[32], v1[32];
                    const uint32_t ta = tmem + ((q * 32) << 16) + buf * 256 + half * 128 + c;
                    tmem_ld32(ta, v0); tmem_ld32(ta + 32, v1);
                    tmem_ld_wait_regs(v0); reg_fence(v1);
                    if (c == 64) { tc_fence_before(); __syncwarp(); if (lane == 0) mbar_arrive(&s.tempty[buf]); }
                    for (int j = 0; j < 32; ++j) acc += v0[j] ^ v1[j];
                }
            }
        }
        if (acc == 0x1234567u) out[3] = acc;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) out[0] = clock64() - t0;
    if (warp == 0) tmem_dealloc<512>(tmem);
}

int main() {
    long long *d;
    cudaMalloc(&d, 64);
    size_t smem = sizeof(Smem) + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles = 400;
    for (int kst : {4, 2, 1})
        for (int mma = 0; mma <= 1; ++mma) {
            if (!mma && kst < 4) continue;
            for (int design = 0; design <= 5; ++design) {
                const int NB = design == 2 ? 4 : design == 3 ? 3 : 2, E = 16;
                long long h[4] = {0, 0, 0, 0};
                probe<<<1, 32 * (1 + E), smem>>>(design, E, mma, tiles, NB, kst, d);
                cudaError_t e = cudaGetLastError();
                if (e == cudaSuccess) e = cudaDeviceSynchronize();
                if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
                e = cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) { printf("copy error %s\n", cudaGetErrorString(e)); return 1; }
                printf("[total %lld, mma thread %lld] ", h[0], h[1]);
                printf("K=%d mma=%d NB=%d %-34s: %.0f cycles per 128 KB of accumulators\n", kst * 16, mma, NB,
                       design == 0 ? "all 16 warps on every tile" : design == 1 ? "two groups, 2 x 256-col buffers" : design == 2 ? "two groups, 4 x 128-col buffers" : design == 3 ? "two groups, 3 x 160-col buffers" : design == 4 ? "two groups, handoff only (no reads)" : "two groups, 2 x 256, half handshakes",
                       (double)h[0] / tiles * 256.0 / (NB == 3 ? 160 : 512 / NB));   // per 256 columns (128 KB)
            }
        }
    return 0;
}
