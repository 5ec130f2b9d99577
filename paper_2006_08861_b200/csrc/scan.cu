// scan.cu -- calculateDistance + selectTopCandidates on sm_100a (Alg. 1 steps 7
// and 10; "top N ... smallest Euclidean distance").
//
// Hot loop (kernel NK2): every CTA owns one work item (a run of
// rows of one subspace) x one tile of query frames.  For each (query, row) pair
// it runs the fixed fp32 chain of R3 over the first kc coefficients (the
// "coarse" prefix, streamed from the coarse plane); the pair is pruned iff that
// partial sum already exceeds the query's threshold tau (strict; the partial of
// a non-negative RN chain never exceeds the full sum, so pruning is exact, R2).
// Survivors continue the SAME chain over the remaining K-kc coefficients from
// the fine plane and are inserted into a per-warp top-N list keyed by
// (acc bits << 32 | global frame).  tau = min(seeded bound, any list's N-th acc)
// is always >= the true N-th distance, so no true top-N pair is ever pruned.
// kc == K is the one-pass scan (NK1).
#include "ol_internal.h"

namespace ol {

__device__ __forceinline__ float chain_step(float acc, float q, float f) {
    float d = __fsub_rn(q, f);
    return __fmaf_rn(d, d, acc);
}

// Insert key into the sorted list L[0..N) (ascending; kPadKey = empty slot).
// Returns the new N-th key.
__device__ __forceinline__ u64 list_insert(u64 *L, uint32_t N, u64 key) {
    if (!(key < L[N - 1])) return L[N - 1];
    int p = (int)N - 1;
    while (p > 0 && L[p - 1] > key) { L[p] = L[p - 1]; --p; }
    L[p] = key;
    return L[N - 1];
}

size_t scan_smem_bytes(uint32_t qt, uint32_t N) {
    return sizeof(float) * qt * kK + sizeof(uint32_t) * kMaxQT + sizeof(u64) * kScanWarps * qt * N;
}

template <int KC>
__global__ void __launch_bounds__(kScanThreads) scan_kernel(ScanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t qt = a.qt, N = a.N;
    float *qs = reinterpret_cast<float *>(smem);                         // [qt][K]
    uint32_t *tau = reinterpret_cast<uint32_t *>(qs + qt * kK);          // [kMaxQT]
    u64 *lists = reinterpret_cast<u64 *>(tau + kMaxQT);                  // [warps][qt][N]

    const uint32_t item_id = blockIdx.x / a.n_qtiles;
    const uint32_t qtile = blockIdx.x % a.n_qtiles;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qtile * qt;
    const uint32_t qn = min(qt, a.nq - q0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    for (uint32_t i = threadIdx.x; i < qn * kK; i += blockDim.x)
        qs[i] = a.queries[(size_t)q0 * kK + i];
    for (uint32_t q = threadIdx.x; q < qt; q += blockDim.x)
        tau[q] = (a.tau0 && q < qn) ? a.tau0[(size_t)(q0 + q) * a.n_sub + it.sub] : kInfBits;
    for (uint32_t i = threadIdx.x; i < kScanWarps * qt * N; i += blockDim.x) lists[i] = kPadKey;
    __syncthreads();

    unsigned long long survivors = 0;
    for (uint32_t base = 0; base < it.count; base += kScanThreads) {
        const uint32_t e = base + threadIdx.x;
        const bool valid = e < it.count;
        const uint64_t row = it.row_begin + (valid ? e : 0);
        float f[KC];
        const float4 *src = reinterpret_cast<const float4 *>(a.coarse + row * KC);
#pragma unroll
        for (int k = 0; k < KC / 4; ++k) {
            float4 v = valid ? __ldg(src + k) : make_float4(0.f, 0.f, 0.f, 0.f);
            f[4 * k] = v.x; f[4 * k + 1] = v.y; f[4 * k + 2] = v.z; f[4 * k + 3] = v.w;
        }
        for (uint32_t q = 0; q < qn; ++q) {
            const float4 *qv = reinterpret_cast<const float4 *>(qs + q * kK);
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < KC / 4; ++k) {
                float4 x = qv[k];
                acc = chain_step(acc, x.x, f[4 * k]);
                acc = chain_step(acc, x.y, f[4 * k + 1]);
                acc = chain_step(acc, x.z, f[4 * k + 2]);
                acc = chain_step(acc, x.w, f[4 * k + 3]);
            }
            const bool surv = valid && __float_as_uint(acc) <= tau[q];
            if (__any_sync(0xffffffffu, surv)) {
                u64 key = kPadKey;
                if (surv) {
                    ++survivors;
                    if (KC < kK) {  // fine pass: continue the same chain
                        const float4 *fr =
                            reinterpret_cast<const float4 *>(a.fine + row * (kK - KC));
#pragma unroll
                        for (int k = 0; k < (kK - KC) / 4; ++k) {
                            float4 x = qv[KC / 4 + k];
                            float4 v = __ldg(fr + k);
                            acc = chain_step(acc, x.x, v.x);
                            acc = chain_step(acc, x.y, v.y);
                            acc = chain_step(acc, x.z, v.z);
                            acc = chain_step(acc, x.w, v.w);
                        }
                    }
                    key = ((u64)__float_as_uint(acc) << 32) | (u64)(it.frame_begin + e);
                }
                u64 *L = lists + ((size_t)warp * qt + q) * N;
                unsigned m = __ballot_sync(0xffffffffu, key < L[N - 1]);
                while (m) {
                    const int l = __ffs(m) - 1;
                    m &= m - 1;
                    if (lane == l) {
                        u64 nth = list_insert(L, N, key);
                        if (nth != kPadKey) atomicMin(&tau[q], (uint32_t)(nth >> 32));
                    }
                    __syncwarp();
                }
            }
        }
    }
    if (a.stat_survivors) {
        for (int o = 16; o; o >>= 1) survivors += __shfl_xor_sync(0xffffffffu, survivors, o);
        if (lane == 0 && survivors) atomicAdd(a.stat_survivors, survivors);
    }
    __syncthreads();
    // merge the per-warp lists of each query (8-way merge) into the item's list
    for (uint32_t q = threadIdx.x; q < qn; q += blockDim.x) {
        int h[kScanWarps];
#pragma unroll
        for (int w = 0; w < kScanWarps; ++w) h[w] = 0;
        u64 *dst = a.partial + ((size_t)(q0 + q) * a.n_items + item_id) * N;
        for (uint32_t r = 0; r < N; ++r) {
            u64 best = kPadKey;
            int bw = 0;
#pragma unroll
            for (int w = 0; w < kScanWarps; ++w) {
                u64 v = h[w] < (int)N ? lists[((size_t)w * qt + q) * N + h[w]] : kPadKey;
                if (v < best) { best = v; bw = w; }
            }
            dst[r] = best;
            if (best != kPadKey) ++h[bw];
        }
    }
}

cudaError_t launch_scan(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s) {
    switch (kc) {
#define OL_SCAN_CASE(KC)                                                                      \
    case KC:                                                                                  \
        cudaFuncSetAttribute(scan_kernel<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                             (int)smem);                                                      \
        scan_kernel<KC><<<grid, kScanThreads, smem, s>>>(a);                                  \
        break;
        OL_SCAN_CASE(8)
        OL_SCAN_CASE(16)
        OL_SCAN_CASE(32)
        OL_SCAN_CASE(64)
#undef OL_SCAN_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ tau seeding (NK3)
// tau0[q][i] = the exact N-th smallest acc over an evenly spaced sample of this
// rank's rows of subspace i (an upper bound on the true N-th acc, so pruning
// with it is exact).  One CTA per (query, subspace); bitonic sort in smem.
constexpr int kSeedThreads = 256;
constexpr int kSeedMax = 4096;

__global__ void __launch_bounds__(kSeedThreads) tau_seed_kernel(SeedArgs a) {
    __shared__ uint32_t v[kSeedMax];
    __shared__ float qs[kK];
    const uint32_t q = blockIdx.x / a.n_sub, i = blockIdx.x % a.n_sub;
    const SubInfo si = a.subs[i];
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, si.count);
    if (threadIdx.x < kK) qs[threadIdx.x] = a.queries[(size_t)q * kK + threadIdx.x];
    __syncthreads();
    if (S < a.N) {
        if (threadIdx.x == 0) a.tau0[(size_t)q * a.n_sub + i] = kInfBits;
        return;
    }
    uint32_t P = 1;
    while (P < S) P <<= 1;
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        uint32_t val = 0xFFFFFFFFu;
        if (s < S) {
            const uint64_t row = si.row_begin + (uint64_t)s * si.count / S;
            const float *c = a.coarse + row * a.kc;
            float acc = 0.f;
            for (uint32_t k = 0; k < a.kc; ++k) acc = chain_step(acc, qs[k], c[k]);
            if (a.kc < (uint32_t)kK) {
                const float *f = a.fine + row * (kK - a.kc);
                for (uint32_t k = a.kc; k < (uint32_t)kK; ++k) acc = chain_step(acc, qs[k], f[k - a.kc]);
            }
            val = __float_as_uint(acc);
        }
        v[s] = val;
    }
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
                uint32_t o = t ^ j;
                if (o > t) {
                    bool up = (t & k) == 0;
                    uint32_t x = v[t], y = v[o];
                    if ((x > y) == up) { v[t] = y; v[o] = x; }
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) a.tau0[(size_t)q * a.n_sub + i] = v[a.N - 1];
}

cudaError_t launch_tau_seed(const SeedArgs &a, cudaStream_t s) {
    tau_seed_kernel<<<a.nq * a.n_sub, kSeedThreads, 0, s>>>(a);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ upload helpers
__global__ void relayout_kernel(const float *src, uint64_t rows, int kc, float *coarse,
                                float *fine) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows * kK;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = i / kK;
        int k = (int)(i % kK);
        float v = src[i];
        if (k < kc) coarse[r * kc + k] = v;
        else fine[r * (kK - kc) + (k - kc)] = v;
    }
}

cudaError_t launch_relayout(const float *src, uint64_t rows, int kc, float *coarse, float *fine,
                            cudaStream_t s) {
    relayout_kernel<<<148 * 8, 256, 0, s>>>(src, rows, kc, coarse, fine);
    return cudaGetLastError();
}

__global__ void check_finite_kernel(const float *p, uint64_t n, int *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (!isfinite(p[i])) *flag = 1;
}

cudaError_t launch_check_finite(const float *p, uint64_t n, int *flag, cudaStream_t s) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    check_finite_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, n, flag);
    return cudaGetLastError();
}

__global__ void check_coords_kernel(const int32_t *xy, uint64_t rows, int32_t gw, int32_t gh,
                                    int *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int32_t x = xy[2 * i], y = xy[2 * i + 1];
        if (x < 0 || x >= gw || y < 0 || y >= gh) *flag = 1;
    }
}

cudaError_t launch_check_coords(const int32_t *xy, uint64_t rows, int32_t gw, int32_t gh,
                                int *flag, cudaStream_t s) {
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    check_coords_kernel<<<(unsigned)blocks, 256, 0, s>>>(xy, rows, gw, gh, flag);
    return cudaGetLastError();
}

}  // namespace ol
