// extract.cu -- GPU descriptor extraction (NEXT-3 in SURVEY §8f, kernel NK9): the
// step before the hot path, for query ingestion at video rate and for building
// large databases on the device.
//
// P:121 "The FFT magnitude of the one-dimensional omnidirectional vector is used as
// a rotation-invariant omnidirectional feature"; S:53 fixes the unnormalised forward
// DFT X[k] = sum_w x[w] e^{-2 pi i k w / W}, bins k = 1..K (DC dropped), descriptor
// m / ||m|| if ||m|| > 1e-12, else all-zero and flagged degenerate (reading R4).
// Binary64 throughout, like the oracle; the angle of term (k, w) is reduced exactly
// to 2 pi ((k w) mod W) / W and taken from a per-CTA table of sincospi(2 j / W).
// Parity with the oracle is within a few ulps of binary64 (summation order of the
// norm differs); the fp32 descriptor is RN32 of the binary64 value.
#include "ol_internal.h"

namespace ol {

constexpr int kExtractWarps = 8;   // profiles per CTA (one warp each)

// One warp per profile; lane l computes bins l + 1 and l + 33.
__global__ void __launch_bounds__(32 * kExtractWarps)
extract_kernel(const double *prof, uint64_t n, uint32_t W, float *out32, double *out64, uint8_t *degenerate) {
    extern __shared__ double ex_smem[];
    double *tc = ex_smem, *ts = ex_smem + W;                 // cos / sin of 2 pi j / W
    double *pw = ex_smem + 2 * W + (threadIdx.x >> 5) * W;   // this warp's profile
    for (uint32_t j = threadIdx.x; j < W; j += blockDim.x) {
        double sn, cs;
        sincospi(2.0 * (double)j / (double)W, &sn, &cs);     // 2 j / W exact for W <= 2^52
        tc[j] = cs;
        ts[j] = sn;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t p = (uint64_t)blockIdx.x * kExtractWarps + (threadIdx.x >> 5); p < n;
         p += (uint64_t)gridDim.x * kExtractWarps) {
        for (uint32_t w = lane; w < W; w += 32) pw[w] = prof[p * W + w];
        __syncwarp();
        double m[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t k = lane + 1 + 32 * h;
            double re = 0.0, im = 0.0;
            uint32_t r = 0;                                    // (k w) mod W, exactly
            for (uint32_t w = 0; w < W; ++w) {
                re = fma(pw[w], tc[r], re);
                im = fma(-pw[w], ts[r], im);
                r += k;
                if (r >= W) r -= W;
            }
            m[h] = sqrt(re * re + im * im);
        }
        double n2 = m[0] * m[0] + m[1] * m[1];
        for (int o = 16; o; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        const double norm = sqrt(n2);
        const bool deg = !(norm > 1e-12);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double c = deg ? 0.0 : m[h] / norm;
            const uint64_t o = p * kK + lane + 32 * h;
            if (out64) out64[o] = c;
            if (out32) out32[o] = __double2float_rn(c);
        }
        if (degenerate && lane == 0) degenerate[p] = deg ? 1 : 0;
        __syncwarp();
    }
}

size_t extract_smem_bytes(uint32_t W) { return sizeof(double) * W * (2 + kExtractWarps); }

cudaError_t launch_extract(const double *prof, uint64_t n, uint32_t W, float *out32, double *out64,
                           uint8_t *degenerate, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t smem = extract_smem_bytes(W);
    cudaError_t e = cudaFuncSetAttribute(extract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint64_t blocks = (n + kExtractWarps - 1) / kExtractWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    extract_kernel<<<(unsigned)blocks, 32 * kExtractWarps, smem, s>>>(prof, n, W, out32, out64, degenerate);
    return cudaGetLastError();
}

}  // namespace ol
