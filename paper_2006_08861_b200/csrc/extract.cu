// extract.cu -- GPU descriptor extraction (NEXT-3 in SURVEY §8f, kernel NK9): the
// step before the hot path, for query ingestion at video rate and for building
// large databases on the device.
//
// P:121 "The FFT magnitude of the one-dimensional omnidirectional vector is used as
// a rotation-invariant omnidirectional feature"; S:53 fixes the unnormalised forward
// DFT X[k] = sum_w x[w] e^{-2 pi i k w / W}, bins k = 1..K (DC dropped), descriptor
// m / ||m|| if ||m|| > 1e-12, else all-zero and flagged degenerate (reading R4).
// Binary64 throughout, like the oracle; twiddles come from a per-CTA table of
// sincospi(2 j / W) at the exactly reduced index (k w) mod W every 8 columns and are
// advanced by one complex rotation in between.
// Parity with the oracle is within a few ulps of binary64 (summation order of the
// norm differs); the fp32 descriptor is RN32 of the binary64 value.
#define OL_TU 6
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
        // lane l: bins k = l + 1 and l + 33.  The twiddle e^{-2 pi i k w / W} advances by a
        // rotation per w; every 8 steps it is re-anchored exactly from the table at the
        // reduced index (k w0) mod W, so rounding drift stays within ~8 rotations
        const uint32_t k0 = lane + 1, k1 = lane + 33;
        const double cr0 = tc[k0 % W], sr0 = ts[k0 % W], cr1 = tc[k1 % W], sr1 = ts[k1 % W];
        double re0 = 0.0, im0 = 0.0, re1 = 0.0, im1 = 0.0;
        for (uint32_t w0 = 0; w0 < W; w0 += 8) {
            const uint32_t r0 = (uint32_t)(((uint64_t)k0 * w0) % W), r1 = (uint32_t)(((uint64_t)k1 * w0) % W);
            double c0 = tc[r0], s0 = ts[r0], c1 = tc[r1], s1 = ts[r1];
            const uint32_t jn = min(8u, W - w0);
            for (uint32_t j = 0; j < jn; ++j) {
                const double x = pw[w0 + j];
                re0 = fma(x, c0, re0);
                im0 = fma(-x, s0, im0);
                re1 = fma(x, c1, re1);
                im1 = fma(-x, s1, im1);
                const double c0n = fma(c0, cr0, -s0 * sr0), s0n = fma(s0, cr0, c0 * sr0);
                const double c1n = fma(c1, cr1, -s1 * sr1), s1n = fma(s1, cr1, c1 * sr1);
                c0 = c0n; s0 = s0n; c1 = c1n; s1 = s1n;
            }
        }
        double m[2] = {sqrt(re0 * re0 + im0 * im0), sqrt(re1 * re1 + im1 * im1)};
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

OL_CHECK_EXPORT(check_extract)

}  // namespace ol
