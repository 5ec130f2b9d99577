// extract.cu -- GPU descriptor extraction (NEXT-3 in SURVEY §8f, kernel NK9): the
// step before the hot path, for query ingestion at video rate and for building
// large databases on the device; and the NEXT-1 stored profile.
//
// P:121 "The FFT magnitude of the one-dimensional omnidirectional vector is used as
// a rotation-invariant omnidirectional feature"; S:53 fixes the unnormalised forward
// DFT X[k] = sum_w x[w] e^{-2 pi i k w / W}, bins k = 1..K (DC dropped), descriptor
// m / ||m|| if ||m|| > 1e-12, else all-zero and flagged degenerate (reading R4).
// The NEXT-1 stored profile is (x - mean x) / ||m|| (zeros if degenerate): its |DFT| on
// bins 1..K is then the descriptor itself (the Parseval link).
// Binary64 throughout, like the oracle.  Two kernels:
//  - fft_extract_kernel<R> (W = 32 R, R in {4, 8, 16}: W = 128, 256, 512): the paper's FFT.
//    One warp per profile, lane l holds x[l + 32 j]; an R-point DFT per lane over j, the
//    twiddle e^{-2 pi i l k1 / W}, then a 32-point radix-2 DIF FFT across the lanes
//    (shuffles): X[k1 + R k2] lands in lane bitrev5(k2).  ~19k flops per profile instead of
//    the direct sum's 65k, and HBM-bound (2 KB read per profile).
//  - extract_kernel (any W): the direct sum, twiddles from a per-CTA sincospi table at the
//    exactly reduced index (k w) mod W every 8 columns, advanced by a rotation in between.
// Parity with the oracle's direct sum is within a few ulps of binary64; the fp32 outputs are
// RN32 of the binary64 values.
#define OL_TU 6
#include "ol_internal.h"

namespace ol {

constexpr int kExtractWarps = 8;   // profiles per CTA (one warp each)

// One warp per profile; lane l computes bins l + 1 and l + 33.
__global__ void __launch_bounds__(32 * kExtractWarps)
extract_kernel(const double *prof, uint64_t n, uint32_t W, float *out32, double *out64, uint8_t *degenerate,
               float *prof_out) {
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
        if (prof_out) {   // NEXT-1 stored profile: (x - mean) / ||m||
            double sum = 0.0;
            for (uint32_t w = lane; w < W; w += 32) sum += pw[w];
            for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const double mean = sum / (double)W;
            for (uint32_t w = lane; w < W; w += 32)
                prof_out[p * W + w] = deg ? 0.f : __double2float_rn((pw[w] - mean) / norm);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- FFT path (W = 32 R)
template <int R>
__global__ void __launch_bounds__(32 * kExtractWarps, R <= 8 ? 3 : 1)
fft_extract_kernel(const double *prof, uint64_t n, float *out32, double *out64, uint8_t *degenerate, float *prof_out) {
    constexpr uint32_t W = 32u * R;
    __shared__ double tc[W], ts[W];   // cos / sin of 2 pi j / W
    for (uint32_t j = threadIdx.x; j < W; j += blockDim.x) {
        double sn, cs;
        sincospi(2.0 * (double)j / (double)W, &sn, &cs);
        tc[j] = cs;
        ts[j] = sn;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    // lane -> its 32-point output k2 (DIF leaves the outputs bit-reversed)
    const uint32_t k2 = __brev(lane) >> 27;
    for (uint64_t p = (uint64_t)blockIdx.x * kExtractWarps + (threadIdx.x >> 5); p < n;
         p += (uint64_t)gridDim.x * kExtractWarps) {
        double x[R];
#pragma unroll
        for (int j = 0; j < R; ++j) x[j] = __ldcs(&prof[p * W + lane + 32 * j]);   // (streamed once)
        // step 1: R-point DFT over j of x[l + 32 j] (real input: A[R - k1] = conj A[k1])
        double re[R], im[R];
        if constexpr (R == 8) {   // the 8-point real DFT by hand (~20 operations instead of 80)
            constexpr double c = 0.70710678118654752440;   // cos(pi/4) = sin(pi/4), RN
            const double a0 = x[0] + x[4], a1 = x[1] + x[5], a2 = x[2] + x[6], a3 = x[3] + x[7];
            const double b0 = x[0] - x[4], b1 = x[1] - x[5], b2 = x[2] - x[6], b3 = x[3] - x[7];
            const double s02 = a0 + a2, s13 = a1 + a3;
            re[0] = s02 + s13; im[0] = 0.0;
            re[4] = s02 - s13; im[4] = 0.0;
            re[2] = a0 - a2;   im[2] = a3 - a1;
            const double cp = c * (b1 - b3), cm = c * (b1 + b3);
            re[1] = b0 + cp;   im[1] = -(b2 + cm);
            re[3] = b0 - cp;   im[3] = b2 - cm;
        } else {
#pragma unroll
        for (int k1 = 0; k1 <= R / 2; ++k1) {
            double a = 0.0, b = 0.0;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int t = (32 * j * k1) % (int)W;   // e^{-2 pi i j k1 / R} = table[32 j k1 mod W]
                a = fma(x[j], tc[t], a);
                b = fma(-x[j], ts[t], b);
            }
            re[k1] = a;
            im[k1] = b;
        }
        }
#pragma unroll
        for (int k1 = R / 2 + 1; k1 < R; ++k1) { re[k1] = re[R - k1]; im[k1] = -im[R - k1]; }
        // step 2: twiddle e^{-2 pi i l k1 / W}
#pragma unroll
        for (int k1 = 1; k1 < R; ++k1) {
            const uint32_t t = (lane * (uint32_t)k1) % W;
            const double c = tc[t], sn = ts[t];
            const double r = re[k1], i = im[k1];
            re[k1] = fma(r, c, i * sn);       // (r + i i)(c - i sn)
            im[k1] = fma(i, c, -r * sn);
        }
        // step 3: 32-point radix-2 DIF FFT across the lanes, every k1
#pragma unroll
        // (branch-free: the upper lane of a pair computes mine + partner, times 1; the lower
        // one partner - mine, times the twiddle -- no divergence between the two halves)
        for (int h = 16; h >= 1; h >>= 1) {
            const bool lower = (lane & h) != 0;
            const uint32_t e = (lane & (h - 1)) * (W / (2 * h));   // W_{2h}^{lane mod h}
            const double c = lower ? tc[e] : 1.0, sn = lower ? ts[e] : 0.0;
            const double sg = lower ? -1.0 : 1.0;
#pragma unroll
            for (int k1 = 0; k1 < R; ++k1) {
                const double pr = __shfl_xor_sync(0xffffffffu, re[k1], h);
                const double pi = __shfl_xor_sync(0xffffffffu, im[k1], h);
                const double dr = fma(sg, re[k1], pr), di = fma(sg, im[k1], pi);   // (lower: pr - re)
                re[k1] = lower ? fma(dr, c, di * sn) : dr;
                im[k1] = lower ? fma(di, c, -dr * sn) : di;
            }
        }
        // step 4: magnitudes of bins 1..K held by this lane (k = k1 + R k2), norm, outputs
        double n2 = 0.0;
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) {
            const uint32_t k = (uint32_t)k1 + R * k2;
            if (k >= 1 && k <= (uint32_t)kK) {
                re[k1] = sqrt(re[k1] * re[k1] + im[k1] * im[k1]);
                n2 += re[k1] * re[k1];
            }
        }
        for (int o = 16; o; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        const double norm = sqrt(n2);
        const bool deg = !(norm > 1e-12);
        // one division, then products (a division per output costs as much as the whole FFT;
        // the results stay within an ulp of binary64 of m / ||m||)
        const double inv = deg ? 0.0 : 1.0 / norm;
#pragma unroll
        for (int k1 = 0; k1 < R; ++k1) {
            const uint32_t k = (uint32_t)k1 + R * k2;
            if (k >= 1 && k <= (uint32_t)kK) {
                const double c = re[k1] * inv;
                const uint64_t o = p * kK + (k - 1);
                if (out64) out64[o] = c;
                if (out32) out32[o] = __double2float_rn(c);
            }
        }
        if (degenerate && lane == 0) degenerate[p] = deg ? 1 : 0;
        if (prof_out) {   // NEXT-1 stored profile: (x - mean) / ||m||
            double sum = 0.0;
#pragma unroll
            for (int j = 0; j < R; ++j) sum += x[j];
            for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const double mean = sum / (double)W;
#pragma unroll
            for (int j = 0; j < R; ++j)
                prof_out[p * W + lane + 32 * j] = __double2float_rn((x[j] - mean) * inv);
        }
    }
}

size_t extract_smem_bytes(uint32_t W) { return sizeof(double) * W * (2 + kExtractWarps); }

cudaError_t launch_extract(const double *prof, uint64_t n, uint32_t W, float *out32, double *out64,
                           uint8_t *degenerate, float *prof_out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (W == 128 || W == 256 || W == 512) {   // the FFT
        uint64_t blocks = (n + kExtractWarps - 1) / kExtractWarps;
        if (blocks > 148 * 32) blocks = 148 * 32;
        if (W == 128) fft_extract_kernel<4><<<(unsigned)blocks, 32 * kExtractWarps, 0, s>>>(prof, n, out32, out64, degenerate, prof_out);
        else if (W == 256) fft_extract_kernel<8><<<(unsigned)blocks, 32 * kExtractWarps, 0, s>>>(prof, n, out32, out64, degenerate, prof_out);
        else fft_extract_kernel<16><<<(unsigned)blocks, 32 * kExtractWarps, 0, s>>>(prof, n, out32, out64, degenerate, prof_out);
        return cudaGetLastError();
    }
    const size_t smem = extract_smem_bytes(W);
    cudaError_t e = cudaFuncSetAttribute(extract_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint64_t blocks = (n + kExtractWarps - 1) / kExtractWarps;
    if (blocks > 148 * 16) blocks = 148 * 16;
    extract_kernel<<<(unsigned)blocks, 32 * kExtractWarps, smem, s>>>(prof, n, W, out32, out64, degenerate, prof_out);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_extract)

}  // namespace ol
