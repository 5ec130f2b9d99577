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

// 8-point complex DFT (W_8 = e^{-2 pi i / 8}) of (xr, xi), radix 2 by hand: out k -> (yr, yi)[k]
__device__ __forceinline__ void dft8(const double *xr, const double *xi, double *yr, double *yi) {
    constexpr double c = 0.70710678118654752440;   // cos(pi/4) = sin(pi/4), RN
    double ar[4], ai[4], br[4], bi[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        ar[j] = xr[j] + xr[j + 4]; ai[j] = xi[j] + xi[j + 4];
        br[j] = xr[j] - xr[j + 4]; bi[j] = xi[j] - xi[j + 4];
    }
    const double A0r = ar[0] + ar[2], A0i = ai[0] + ai[2], A2r = ar[0] - ar[2], A2i = ai[0] - ai[2];
    const double A1r = ar[1] + ar[3], A1i = ai[1] + ai[3], A3r = ar[1] - ar[3], A3i = ai[1] - ai[3];
    yr[0] = A0r + A1r; yi[0] = A0i + A1i;
    yr[4] = A0r - A1r; yi[4] = A0i - A1i;
    yr[2] = A2r + A3i; yi[2] = A2i - A3r;
    yr[6] = A2r - A3i; yi[6] = A2i + A3r;
    const double t1r = c * (br[1] + bi[1]), t1i = c * (bi[1] - br[1]);
    const double t2r = bi[2], t2i = -br[2];
    const double t3r = c * (bi[3] - br[3]), t3i = -c * (bi[3] + br[3]);
    const double B0r = br[0] + t2r, B0i = bi[0] + t2i, B2r = br[0] - t2r, B2i = bi[0] - t2i;
    const double B1r = t1r + t3r, B1i = t1i + t3i, B3r = t1r - t3r, B3i = t1i - t3i;
    yr[1] = B0r + B1r; yi[1] = B0i + B1i;
    yr[5] = B0r - B1r; yi[5] = B0i - B1i;
    yr[3] = B2r + B3i; yi[3] = B2i - B3r;
    yr[7] = B2r - B3i; yi[7] = B2i + B3r;
}

// (row r of 8 doubles, element e) -> a per-warp shared-memory slot: rows padded to 9, so a
// warp writing one element of every row, or reading rows a + 4 b, spreads over the banks, and
// every address is a per-lane base plus an immediate
__device__ __forceinline__ uint32_t sw8(uint32_t r, uint32_t e) { return r * 9 + e; }
// Z[k] slot: 4 doubles of padding per 16 (the step-C writers, lanes (k1, cp), hit 16 banks)
__device__ __forceinline__ uint32_t swz(uint32_t k) { return k + 4 * (k >> 4); }
constexpr uint32_t kZSlots = 256 + 4 * 16;

// W = 256: TWO profiles per warp as one complex sequence z = a + i b (the real-input trick:
// the FFT's twiddles and butterflies serve both), separated at the end by the symmetry of real
// inputs: A[k] = (Z[k] + conj Z[W-k]) / 2, B[k] = (Z[k] - conj Z[W-k]) / 2i.  The 256-point
// FFT as 8 x 8 x 4 with two shared-memory transposes (round 2; the first version, an 8-point
// DFT per lane and a 32-point DIF across the lanes by five shuffle stages, ran 840M profiles/s,
// this one 1,186M): n = l + 32 j, k = k1 + 8 k2 with l = a + 4 b, k2 = c + 8 d:
//   Y[l][k1]   = DFT8_j z[l + 32 j] . W_256^{l k1}            (lane l)
//   U[k1,a][c] = DFT8_b Y[a + 4 b][k1] . W_32^{a c}           (lane 4 k1 + a)
//   Z[k1 + 8 c + 64 d] = DFT4_a U[k1,a][c]                     (lane 4 k1 + c / 2, two c)
// then Z goes to shared memory, lane l separates bins l + 1 and l + 33 of both profiles from
// Z[k], Z[256 - k], and the outputs are written contiguously.
__global__ void __launch_bounds__(32 * kExtractWarps, 3)
fft3_extract256_kernel(const double *prof, uint64_t n, float *out32, double *out64, uint8_t *degenerate, float *prof_out) {
    constexpr uint32_t W = 256;
    // twiddles laid out in the order the lanes read them (a table indexed by l q mod 256 put
    // lanes of even q on the same banks: up to 8-way conflicts); the same sincospi values
    //   twA[q][l] = W_256^{l q} (step A, lane l),  twB[c][a] = W_256^{8 a c} (step B)
    __shared__ double2 twA[8][32], twB[8][4];
    __shared__ double zr[kExtractWarps][kZSlots], zi[kExtractWarps][kZSlots];
    for (uint32_t j = threadIdx.x; j < 8 * 32 + 8 * 4; j += blockDim.x) {
        const bool isA = j < 8 * 32;
        const uint32_t jb = j - 8 * 32;
        const uint32_t t = isA ? ((j & 31) * (j >> 5)) & (W - 1) : (8u * (jb & 3) * (jb >> 2)) & (W - 1);
        double sn, cs;
        sincospi(2.0 * (double)t / (double)W, &sn, &cs);
        if (isA) twA[j >> 5][j & 31] = make_double2(cs, sn);
        else twB[jb >> 2][jb & 3] = make_double2(cs, sn);
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    double *const br = zr[wi], *const bi = zi[wi];
    const uint32_t k1 = lane >> 2, a = lane & 3;   // steps B and C: (k1, a) / (k1, c pair)
    const uint64_t pairs = (n + 1) / 2;
    for (uint64_t pp = (uint64_t)blockIdx.x * kExtractWarps + wi; pp < pairs; pp += (uint64_t)gridDim.x * kExtractWarps) {
        const uint64_t pa = 2 * pp, pb = pa + 1;
        const bool hasb = pb < n;
        {   // the warp's next pair (4 KB contiguous: 128 B per lane) towards L2 while this one computes
            const uint64_t nx = 2 * (pp + (uint64_t)gridDim.x * kExtractWarps) * W + 16ull * lane;
            if (nx < n * W) asm volatile("prefetch.global.L2 [%0];" ::"l"(prof + nx));
        }
        double re[8], im[8];
        double sa = 0.0, sb = 0.0;
        int ea = 0, eb = 0;
        {   // step A: lane l, the 8-point DFT over j of z[l + 32 j], twiddled
            double xa[8], xb[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                xa[j] = __ldg(&prof[pa * W + lane + 32 * j]);
                xb[j] = hasb ? __ldg(&prof[pb * W + lane + 32 * j]) : 0.0;
            }
            if (prof_out) {
#pragma unroll
                for (int j = 0; j < 8; ++j) { sa += xa[j]; sb += xb[j]; }
            }
            // each profile scaled by a power of two to max |x| in [1, 2): exact (all later
            // operations scale exactly), so the descriptor is unchanged, and a dim profile is
            // not drowned by the rounding of a bright partner's transform (the biased exponent
            // field of the largest |x|: an integer warp max; 0 for zeros)
            uint32_t ga = 0, gb = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ga = max(ga, (uint32_t)(__double_as_longlong(xa[j]) >> 52) & 0x7ffu);
                gb = max(gb, (uint32_t)(__double_as_longlong(xb[j]) >> 52) & 0x7ffu);
            }
            ga = __reduce_max_sync(0xffffffffu, ga);
            gb = __reduce_max_sync(0xffffffffu, gb);
            ea = (ga > 1 && ga < 2046) ? (int)ga - 1023 : 0;
            eb = (gb > 1 && gb < 2046) ? (int)gb - 1023 : 0;
            const double sca = __longlong_as_double((long long)(1023 - ea) << 52);
            const double scb = __longlong_as_double((long long)(1023 - eb) << 52);
#pragma unroll
            for (int j = 0; j < 8; ++j) { xa[j] *= sca; xb[j] *= scb; }
            dft8(xa, xb, re, im);
        }
#pragma unroll
        for (int q = 1; q < 8; ++q) {   // W_256^{l q}
            const double2 w = twA[q][lane];
            const double c = w.x, sn = w.y;
            const double r = re[q], i = im[q];
            re[q] = fma(r, c, i * sn);
            im[q] = fma(i, c, -r * sn);
        }
        __syncwarp();   // (the previous pair's readers of the buffer are done)
#pragma unroll
        for (int q = 0; q < 8; ++q) { br[sw8(lane, q)] = re[q]; bi[sw8(lane, q)] = im[q]; }
        __syncwarp();
        {   // step B: lane (k1, a), the 8-point DFT over b of Y[a + 4 b][k1], twiddled by W_32^{a c}
            double xr[8], xi[8];
#pragma unroll
            for (int b = 0; b < 8; ++b) { xr[b] = br[sw8(a + 4 * b, k1)]; xi[b] = bi[sw8(a + 4 * b, k1)]; }
            dft8(xr, xi, re, im);
        }
#pragma unroll
        for (int c = 1; c < 8; ++c) {
            const double2 w = twB[c][a];
            const double cs = w.x, sn = w.y;
            const double r = re[c], i = im[c];
            re[c] = fma(r, cs, i * sn);
            im[c] = fma(i, cs, -r * sn);
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c) { br[sw8(lane, c)] = re[c]; bi[sw8(lane, c)] = im[c]; }
        __syncwarp();
        {   // step C: lane (k1, cp), the 4-point DFTs over a of U[k1, a][c], c = 2 cp, 2 cp + 1
            const uint32_t cp = a;
            double ur[2][4], ui[2][4];
#pragma unroll
            for (int e = 0; e < 2; ++e)
#pragma unroll
                for (int aa = 0; aa < 4; ++aa) {
                    ur[e][aa] = br[sw8(4 * k1 + aa, 2 * cp + e)];
                    ui[e][aa] = bi[sw8(4 * k1 + aa, 2 * cp + e)];
                }
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double x0r = ur[e][0] + ur[e][2], x0i = ui[e][0] + ui[e][2];
                const double x1r = ur[e][0] - ur[e][2], x1i = ui[e][0] - ui[e][2];
                const double x2r = ur[e][1] + ur[e][3], x2i = ui[e][1] + ui[e][3];
                const double x3r = ur[e][1] - ur[e][3], x3i = ui[e][1] - ui[e][3];
                const uint32_t k = k1 + 8 * (2 * cp + e);
                br[swz(k)] = x0r + x2r;         bi[swz(k)] = x0i + x2i;          // d = 0
                br[swz(k + 128)] = x0r - x2r;   bi[swz(k + 128)] = x0i - x2i;    // d = 2
                br[swz(k + 64)] = x1r + x3i;    bi[swz(k + 64)] = x1i - x3r;     // d = 1: X1 - i X3
                br[swz(k + 192)] = x1r - x3i;   bi[swz(k + 192)] = x1i + x3r;    // d = 3: X1 + i X3
            }
        }
        __syncwarp();
        // separate bins k = lane + 1 and lane + 33: 2 A[k] = Z[k] + conj Z[W - k],
        // 2 i B[k] = Z[k] - conj Z[W - k]
        double ma[2], mb[2], n2a = 0.0, n2b = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t k = lane + 1 + 32 * h, m = W - k;
            const double zkr = br[swz(k)], zki = bi[swz(k)], zmr = br[swz(m)], zmi = bi[swz(m)];
            const double sr = zkr + zmr, di = zki - zmi;
            const double si = zki + zmi, dr = zkr - zmr;
            ma[h] = 0.5 * sqrt(sr * sr + di * di);
            mb[h] = 0.5 * sqrt(si * si + dr * dr);
            n2a += ma[h] * ma[h];
            n2b += mb[h] * mb[h];
        }
        for (int o = 16; o; o >>= 1) {
            n2a += __shfl_xor_sync(0xffffffffu, n2a, o);
            n2b += __shfl_xor_sync(0xffffffffu, n2b, o);
        }
        const double norma = sqrt(n2a), normb = sqrt(n2b);   // (of the scaled profiles)
        const double una = __longlong_as_double((long long)(1023 + ea) << 52);
        const double unb = __longlong_as_double((long long)(1023 + eb) << 52);
        const bool dega = !(norma * una > 1e-12), degb = !(normb * unb > 1e-12);
        const double inva = dega ? 0.0 : 1.0 / norma, invb = degb ? 0.0 : 1.0 / normb;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double ca = ma[h] * inva, cb = mb[h] * invb;
            const uint64_t oa = pa * kK + lane + 32 * h, ob = pb * kK + lane + 32 * h;
            if (out64) { out64[oa] = ca; if (hasb) out64[ob] = cb; }
            if (out32) { out32[oa] = __double2float_rn(ca); if (hasb) out32[ob] = __double2float_rn(cb); }
        }
        if (degenerate && lane == 0) { degenerate[pa] = dega ? 1 : 0; if (hasb) degenerate[pb] = degb ? 1 : 0; }
        if (prof_out) {   // NEXT-1 stored profiles: (x - mean) / ||m|| (the profiles re-read: L2)
            for (int o = 16; o; o >>= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
                sb += __shfl_xor_sync(0xffffffffu, sb, o);
            }
            const double meana = sa / (double)W, meanb = sb / (double)W;
            const double sca2 = __longlong_as_double((long long)(1023 - ea) << 52), scb2 = __longlong_as_double((long long)(1023 - eb) << 52);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                prof_out[pa * W + lane + 32 * j] = __double2float_rn((__ldg(&prof[pa * W + lane + 32 * j]) - meana) * (inva * sca2));
                if (hasb) prof_out[pb * W + lane + 32 * j] = __double2float_rn((__ldg(&prof[pb * W + lane + 32 * j]) - meanb) * (invb * scb2));
            }
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
        else if (W == 256) {   // two profiles per warp
            uint64_t b2 = ((n + 1) / 2 + kExtractWarps - 1) / kExtractWarps;
            if (b2 > 148 * 32) b2 = 148 * 32;
            fft3_extract256_kernel<<<(unsigned)b2, 32 * kExtractWarps, 0, s>>>(prof, n, out32, out64, degenerate, prof_out);
        }
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
