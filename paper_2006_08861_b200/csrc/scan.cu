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
#define OL_TU 1
#include "ol_internal.h"
#include "tc_ptx.cuh"

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
    // (a work item's rows lie inside the planes, its subspace and frame tile exist)
    if (!OL_DCHECK(item_id < a.n_items && it.row_begin + it.count <= a.rows_pad && it.sub < a.n_sub && q0 < a.nq &&
                   qt <= kMaxQT))
        return;
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
#pragma unroll
        for (int k = 0; k < KC / 4; ++k) {
            const float4 *src = reinterpret_cast<const float4 *>(a.coarse + coarse_off(row, 4 * k, KC));
            float4 v = valid ? __ldg(src) : make_float4(0.f, 0.f, 0.f, 0.f);
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
                            reinterpret_cast<const float4 *>(a.fine + fine_off(row, KC));
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

// ---------------------------------------------------------------- small-batch scan (NK2s)
// Same contract as scan_kernel, tuned for few query frames (<= kMaxQT2), the
// HBM-bound regime: each thread owns a PAIR of rows (r, r + 256) whose coarse
// coefficients it keeps packed as f32x2 pairs, so every chain step is one FADD2
// + one FFMA2 for two rows (each lane still the exact RN fp32 chain of R3), the
// next pair's rows are loaded before the current pair is scored (register
// double buffering), and query coefficients sit duplicated (q, q) in smem so one
// LDS.128 feeds two steps.
constexpr int kMaxQT2 = 16;

__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
    return ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ uint64_t f2sub(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

template <int KC>
__device__ __forceinline__ void load_pair(const float *coarse, const WorkItem &it, uint32_t e0, float4 (&v)[2][KC / 4]) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const uint32_t e = e0 + h * kScanThreads;
        const bool ok = e < it.count;
        const uint64_t row = it.row_begin + (ok ? e : 0);
#pragma unroll
        for (int k = 0; k < KC / 4; ++k)
            v[h][k] = ok ? __ldg(reinterpret_cast<const float4 *>(coarse + coarse_off(row, 4 * k, KC)))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

// Survivors of one query for a thread's row pair: finish the chain from the fine
// plane and insert into the warp's list (ballot-serialised, see scan_kernel).
template <int KC>
__device__ __noinline__ void scan2_survivors(const ScanArgs &a, const WorkItem &it, const float *qs, u64 *lists,
                                             uint32_t *tau, uint32_t q, uint32_t q0, uint32_t qt, uint32_t N,
                                             int warp, int lane, uint32_t e0, uint32_t e1, bool s0, bool s1,
                                             uint64_t acc2, unsigned long long &survivors) {
    for (int h = 0; h < 2; ++h) {
        const bool sv = h ? s1 : s0;
        const uint32_t e = h ? e1 : e0;
        float acc = __uint_as_float(h ? (uint32_t)(acc2 >> 32) : (uint32_t)acc2);
        u64 key = kPadKey;
        if (sv) {
            ++survivors;
            if (KC < kK) {  // fine pass: continue the same chain
                const uint64_t row = it.row_begin + e;
                const float4 *fr = reinterpret_cast<const float4 *>(a.fine + fine_off(row, KC));
                const float4 *qv = reinterpret_cast<const float4 *>(qs + q * kK);
#pragma unroll
                for (int k = 0; k < (kK - KC) / 4; ++k) {
                    const float4 x = qv[KC / 4 + k], v = __ldg(fr + k);
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
                const u64 nth = list_insert(L, N, key);
                if (nth != kPadKey) {
                    const uint32_t tb = (uint32_t)(nth >> 32);
                    atomicMin(&tau[q], tb);
                    // publish: any CTA's N-th is a valid bound for all of them
                    if (a.tau0) atomicMin(&a.tau0[(size_t)(q0 + q) * a.n_sub + it.sub], tb);
                }
            }
            __syncwarp();
        }
    }
}

template <int KC>
__global__ void __launch_bounds__(kScanThreads) scan2_kernel(ScanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t qt = a.qt, N = a.N;
    float *qs = reinterpret_cast<float *>(smem);                           // [qt][K] (fine part)
    uint64_t *qd = reinterpret_cast<uint64_t *>(qs + kMaxQT2 * kK);        // [qt][KC] (q, q)
    uint32_t *tau = reinterpret_cast<uint32_t *>(qd + kMaxQT2 * KC);       // [kMaxQT2]
    u64 *lists = reinterpret_cast<u64 *>(tau + kMaxQT2);                   // [warps][qt][N]

    const uint32_t item_id = blockIdx.x / a.n_qtiles;
    const uint32_t qtile = blockIdx.x % a.n_qtiles;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qtile * qt;
    const uint32_t qn = min(qt, a.nq - q0);
    // (a work item's rows lie inside the planes, its subspace and frame tile exist)
    if (!OL_DCHECK(item_id < a.n_items && it.row_begin + it.count <= a.rows_pad && it.sub < a.n_sub && q0 < a.nq &&
                   qt <= kMaxQT))
        return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    for (uint32_t i = threadIdx.x; i < kMaxQT2 * kK; i += blockDim.x) {
        const float v = i < qn * kK ? a.queries[(size_t)q0 * kK + i] : 0.f;
        qs[i] = v;
        if ((i % kK) < (uint32_t)KC) qd[(i / kK) * KC + (i % kK)] = f2pack(v, v);
    }
    for (uint32_t q = threadIdx.x; q < kMaxQT2; q += blockDim.x)
        tau[q] = (a.tau0 && q < qn) ? a.tau0[(size_t)(q0 + q) * a.n_sub + it.sub] : kInfBits;
    for (uint32_t i = threadIdx.x; i < kScanWarps * qt * N; i += blockDim.x) lists[i] = kPadKey;
    __syncthreads();

    unsigned long long survivors = 0;
    float4 nxt[2][KC / 4];
    load_pair<KC>(a.coarse, it, threadIdx.x, nxt);
    for (uint32_t base = 0; base < it.count; base += 2 * kScanThreads) {
        uint64_t f2[KC];   // (row0[k], row1[k])
#pragma unroll
        for (int k = 0; k < KC / 4; ++k) {
            f2[4 * k] = f2pack(nxt[0][k].x, nxt[1][k].x);
            f2[4 * k + 1] = f2pack(nxt[0][k].y, nxt[1][k].y);
            f2[4 * k + 2] = f2pack(nxt[0][k].z, nxt[1][k].z);
            f2[4 * k + 3] = f2pack(nxt[0][k].w, nxt[1][k].w);
        }
        const uint32_t e0 = base + threadIdx.x, e1 = e0 + kScanThreads;
        const bool v0 = e0 < it.count, v1 = e1 < it.count;
        // import the thresholds other CTAs published (valid bounds; races only loosen)
        if (a.tau0 && threadIdx.x < qn && (base & (8 * kScanThreads - 1)) == 0)
            atomicMin(&tau[threadIdx.x], __ldcg(&a.tau0[(size_t)(q0 + threadIdx.x) * a.n_sub + it.sub]));
        if (base + 2 * kScanThreads < it.count) load_pair<KC>(a.coarse, it, e0 + 2 * kScanThreads, nxt);
        // four query chains at a time for instruction-level parallelism (qd/tau are
        // padded to kMaxQT2 frames, so the tail group reads harmless values)
        for (uint32_t qb = 0; qb < qn; qb += 4) {
            uint64_t acc2[4] = {0, 0, 0, 0};
#pragma unroll
            for (int k = 0; k < KC / 2; ++k) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const ulonglong2 x = reinterpret_cast<const ulonglong2 *>(qd + (qb + u) * KC)[k];
                    uint64_t d = f2sub(x.x, f2[2 * k]);
                    acc2[u] = f2fma(d, d, acc2[u]);
                    d = f2sub(x.y, f2[2 * k + 1]);
                    acc2[u] = f2fma(d, d, acc2[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t q = qb + u;
                if (q >= qn) break;
                const uint32_t tq = tau[q];
                const bool s0 = v0 && (uint32_t)acc2[u] <= tq, s1 = v1 && (uint32_t)(acc2[u] >> 32) <= tq;
                if (__any_sync(0xffffffffu, s0 || s1))
                    scan2_survivors<KC>(a, it, qs, lists, tau, q, q0, qt, N, warp, lane, e0, e1, s0, s1, acc2[u],
                                        survivors);
            }
        }
    }
    if (a.stat_survivors) {
        for (int o = 16; o; o >>= 1) survivors += __shfl_xor_sync(0xffffffffu, survivors, o);
        if (lane == 0 && survivors) atomicAdd(a.stat_survivors, survivors);
    }
    __syncthreads();
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
                const u64 v = h[w] < (int)N ? lists[((size_t)w * qt + q) * N + h[w]] : kPadKey;
                if (v < best) { best = v; bw = w; }
            }
            dst[r] = best;
            if (best != kPadKey) ++h[bw];
        }
    }
}

// ---------------------------------------------------------------- small-batch scan, TMA-fed
// scan2's arithmetic, but the coarse rows reach shared memory through 1-D bulk
// copies (cp.async.bulk, UBLKCP) issued by a producer warp into a kStages2-deep
// mbarrier ring, so bytes in flight no longer cost registers; the 8 consumer
// warps read their row pairs with LDS.128.
constexpr int kStages2 = 3;
constexpr int kRows2 = 2 * kScanThreads;   // rows per stage

template <int KC>
__global__ void __launch_bounds__(kScanThreads + 32) scan3_kernel(ScanArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];   // (bulk copies need 16 B)
    const uint32_t qt = a.qt, N = a.N;
    float *rows = reinterpret_cast<float *>(smem);                         // [kStages2][kRows2][KC]
    uint64_t *full = reinterpret_cast<uint64_t *>(rows + kStages2 * kRows2 * KC);
    uint64_t *empty = full + kStages2;
    float *qs = reinterpret_cast<float *>(empty + kStages2);               // [qt][K]
    uint64_t *qd = reinterpret_cast<uint64_t *>(qs + kMaxQT2 * kK);        // [qt][KC] (q, q)
    uint32_t *tau = reinterpret_cast<uint32_t *>(qd + kMaxQT2 * KC);       // [kMaxQT2]
    u64 *lists = reinterpret_cast<u64 *>(tau + kMaxQT2);                   // [warps][qt][N]

    const uint32_t item_id = blockIdx.x / a.n_qtiles;
    const uint32_t qtile = blockIdx.x % a.n_qtiles;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qtile * qt;
    const uint32_t qn = min(qt, a.nq - q0);
    // (a work item's rows lie inside the planes, its subspace and frame tile exist)
    if (!OL_DCHECK(item_id < a.n_items && it.row_begin + it.count <= a.rows_pad && it.sub < a.n_sub && q0 < a.nq &&
                   qt <= kMaxQT))
        return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n_stages_total = (it.count + kRows2 - 1) / kRows2;

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages2; ++i) { tc::mbar_init(&full[i], 1); tc::mbar_init(&empty[i], kScanWarps); }
        tc::fence_mbar_init();
    }
    for (uint32_t i = threadIdx.x; i < qn * kK; i += blockDim.x) {
        const float v = a.queries[(size_t)q0 * kK + i];
        qs[i] = v;
        if ((i % kK) < (uint32_t)KC) qd[(i / kK) * KC + (i % kK)] = f2pack(v, v);
    }
    for (uint32_t q = threadIdx.x; q < kMaxQT2; q += blockDim.x)
        tau[q] = (a.tau0 && q < qn) ? a.tau0[(size_t)(q0 + q) * a.n_sub + it.sub] : kInfBits;
    for (uint32_t i = threadIdx.x; i < kScanWarps * qt * N; i += blockDim.x) lists[i] = kPadKey;
    __syncthreads();

    if (warp == kScanWarps) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            for (uint32_t t = 0; t < n_stages_total; ++t) {
                const uint32_t st = t % kStages2;
                if (t >= kStages2) tc::mbar_wait_sleep(&empty[st], ((t / kStages2) - 1) & 1);
                // whole 32-row tiles (the plane is padded to tiles, so this stays in bounds)
                const uint32_t nrows = (min((uint32_t)kRows2, it.count - t * kRows2) + 31) & ~31u;
                const uint32_t bytes = nrows * KC * sizeof(float);
                tc::mbar_expect_tx(&full[st], bytes);
                tc::bulk_load(rows + (size_t)st * kRows2 * KC,
                              a.coarse + coarse_off(it.row_begin + (uint64_t)t * kRows2, 0, KC), bytes, &full[st]);
            }
        }
    } else {
        // ------------------------------------------------------------ consumers
        unsigned long long survivors = 0;
        for (uint32_t t = 0; t < n_stages_total; ++t) {
            const uint32_t st = t % kStages2, base = t * kRows2;
            const uint32_t e0 = base + threadIdx.x, e1 = e0 + kScanThreads;
            const bool v0 = e0 < it.count, v1 = e1 < it.count;
            if (a.tau0 && threadIdx.x < qn && (t & 7) == 0)   // import published thresholds
                atomicMin(&tau[threadIdx.x], __ldcg(&a.tau0[(size_t)(q0 + threadIdx.x) * a.n_sub + it.sub]));
            tc::mbar_wait(&full[st], (t / kStages2) & 1);
            uint64_t f2[KC];   // (row0[k], row1[k])
            {
                const float *sb = rows + (size_t)st * kRows2 * KC;
#pragma unroll
                for (int k = 0; k < KC / 4; ++k) {
                    const float4 x = v0 ? *reinterpret_cast<const float4 *>(sb + coarse_off(threadIdx.x, 4 * k, KC))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                    const float4 y = v1 ? *reinterpret_cast<const float4 *>(sb + coarse_off(threadIdx.x + kScanThreads, 4 * k, KC))
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
                    f2[4 * k] = f2pack(x.x, y.x); f2[4 * k + 1] = f2pack(x.y, y.y);
                    f2[4 * k + 2] = f2pack(x.z, y.z); f2[4 * k + 3] = f2pack(x.w, y.w);
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&empty[st]);
            for (uint32_t q = 0; q < qn; ++q) {
                const ulonglong2 *qq = reinterpret_cast<const ulonglong2 *>(qd + q * KC);
                uint64_t acc2 = 0;
#pragma unroll
                for (int k = 0; k < KC / 2; ++k) {
                    const ulonglong2 x = qq[k];
                    uint64_t d = f2sub(x.x, f2[2 * k]);
                    acc2 = f2fma(d, d, acc2);
                    d = f2sub(x.y, f2[2 * k + 1]);
                    acc2 = f2fma(d, d, acc2);
                }
                const uint32_t tq = tau[q];
                const bool s0 = v0 && (uint32_t)acc2 <= tq, s1 = v1 && (uint32_t)(acc2 >> 32) <= tq;
                if (__any_sync(0xffffffffu, s0 || s1)) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const bool sv = h ? s1 : s0;
                        const uint32_t e = h ? e1 : e0;
                        float acc = __uint_as_float(h ? (uint32_t)(acc2 >> 32) : (uint32_t)acc2);
                        u64 key = kPadKey;
                        if (sv) {
                            ++survivors;
                            if (KC < kK) {
                                const uint64_t row = it.row_begin + e;
                                const float4 *fr = reinterpret_cast<const float4 *>(a.fine + fine_off(row, KC));
                                const float4 *qv = reinterpret_cast<const float4 *>(qs + q * kK);
#pragma unroll
                                for (int k = 0; k < (kK - KC) / 4; ++k) {
                                    const float4 x = qv[KC / 4 + k], v = __ldg(fr + k);
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
                                const u64 nth = list_insert(L, N, key);
                                if (nth != kPadKey) {
                                    const uint32_t tb = (uint32_t)(nth >> 32);
                                    atomicMin(&tau[q], tb);
                                    if (a.tau0) atomicMin(&a.tau0[(size_t)(q0 + q) * a.n_sub + it.sub], tb);
                                }
                            }
                            __syncwarp();
                        }
                    }
                }
            }
        }
        if (a.stat_survivors) {
            for (int o = 16; o; o >>= 1) survivors += __shfl_xor_sync(0xffffffffu, survivors, o);
            if (lane == 0 && survivors) atomicAdd(a.stat_survivors, survivors);
        }
    }
    __syncthreads();
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
                const u64 v = h[w] < (int)N ? lists[((size_t)w * qt + q) * N + h[w]] : kPadKey;
                if (v < best) { best = v; bw = w; }
            }
            dst[r] = best;
            if (best != kPadKey) ++h[bw];
        }
    }
}

size_t scan3_smem_bytes(uint32_t qt, uint32_t N, int kc) {
    return sizeof(float) * kStages2 * kRows2 * kc + 2 * kStages2 * sizeof(uint64_t) + sizeof(float) * kMaxQT2 * kK +
           sizeof(uint64_t) * kMaxQT2 * kc + sizeof(uint32_t) * kMaxQT2 + sizeof(u64) * kScanWarps * qt * N;
}

cudaError_t launch_scan3(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s) {
    switch (kc) {
#define OL_SCAN3_CASE(KC)                                                                     \
    case KC:                                                                                  \
        cudaFuncSetAttribute(scan3_kernel<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)smem);                                                      \
        scan3_kernel<KC><<<grid, kScanThreads + 32, smem, s>>>(a);                            \
        break;
        OL_SCAN3_CASE(8)
        OL_SCAN3_CASE(16)
        OL_SCAN3_CASE(32)
#undef OL_SCAN3_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

size_t scan2_smem_bytes(uint32_t qt, uint32_t N, int kc) {
    return sizeof(float) * kMaxQT2 * kK + sizeof(uint64_t) * kMaxQT2 * kc + sizeof(uint32_t) * kMaxQT2 +
           sizeof(u64) * kScanWarps * qt * N;
}

cudaError_t launch_scan2(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s) {
    switch (kc) {
#define OL_SCAN2_CASE(KC)                                                                     \
    case KC:                                                                                  \
        cudaFuncSetAttribute(scan2_kernel<KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                             (int)smem);                                                      \
        scan2_kernel<KC><<<grid, kScanThreads, smem, s>>>(a);                                 \
        break;
        OL_SCAN2_CASE(8)
        OL_SCAN2_CASE(16)
        OL_SCAN2_CASE(32)
        OL_SCAN2_CASE(64)
#undef OL_SCAN2_CASE
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
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
// with it is exact).  One CTA per (query, subspace, split): the sample's exact fp32
// chains (float4 row loads, query in shared memory), then the N-th smallest by a
// 4-pass radix select (8-bit digits) over the acc bits (non-negative floats order as
// their bits).
constexpr int kSeedThreads = 256;
constexpr int kSeedMax = 8192;

template <int KC>
__global__ void __launch_bounds__(kSeedThreads, 2) tau_seed_kernel(SeedArgs a) {
    __shared__ uint32_t v[kSeedMax];
    __shared__ alignas(16) float qs[kK];
    __shared__ uint32_t hist[256];
    __shared__ uint32_t sel[2];   // digit, count below it
    const uint32_t split = blockIdx.x % a.splits;
    const uint32_t q = (blockIdx.x / a.splits) / a.n_sub, i = (blockIdx.x / a.splits) % a.n_sub;
    const SubInfo si = a.subs[i];
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, si.count);
    if (threadIdx.x < kK) qs[threadIdx.x] = a.queries[(size_t)q * kK + threadIdx.x];
    __syncthreads();
    if (S < a.N) return;   // the caller pre-filled +inf
    const float4 *q4 = reinterpret_cast<const float4 *>(qs);
    for (uint32_t s = threadIdx.x; s < S; s += blockDim.x) {
        // split j takes the j-th of `splits` interleaved sample grids
        const uint64_t row = si.row_begin + (((uint64_t)s * a.splits + split) * si.count) / ((uint64_t)S * a.splits);
        if (!OL_DCHECK(row < si.row_begin + si.count && row < a.rows_pad && s < (uint32_t)kSeedMax)) continue;
        float4 f[kK / 4];   // (KC is a compile-time constant: all 16 loads issue before the chain)
#pragma unroll
        for (int k4 = 0; k4 < kK / 4; ++k4)
            f[k4] = __ldg(reinterpret_cast<const float4 *>(a.fine + fine_off(row, 4 * k4)));
        float acc = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < kK / 4; ++k4) {
            const float4 x = q4[k4];
            acc = chain_step(acc, x.x, f[k4].x); acc = chain_step(acc, x.y, f[k4].y);
            acc = chain_step(acc, x.z, f[k4].z); acc = chain_step(acc, x.w, f[k4].w);
        }
        v[s] = __float_as_uint(acc);
    }
    // radix select: the N-th smallest value (1-based), digit by digit from the top
    uint32_t prefix = 0, pmask = 0, k = a.N;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t t = threadIdx.x; t < 256; t += blockDim.x) hist[t] = 0;
        __syncthreads();
        // (values share their high digits: warp-aggregated increments avoid serializing
        // on one bin)
        for (uint32_t s0 = 0; s0 < S; s0 += blockDim.x) {
            const uint32_t s = s0 + threadIdx.x;
            const uint32_t x = s < S ? v[s] : 0u;
            const bool in = s < S && (x & pmask) == prefix;
            const uint32_t d = in ? (x >> shift) & 255u : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (in && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&hist[d], (uint32_t)__popc(peers));
        }
        __syncthreads();
        if (threadIdx.x < 32) {   // one warp: 8 bins per lane, inclusive scan, first bin reaching k
            const int lane = threadIdx.x;
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) { c[j] = hist[lane * 8 + j]; tot += c[j]; }
            uint32_t incl = tot;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            uint32_t below = incl - tot;
            const bool here = below < k && k <= incl;
            if (here) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (below + c[j] >= k) { sel[0] = lane * 8 + j; sel[1] = below; break; }
                    below += c[j];
                }
            }
        }
        __syncthreads();
        prefix |= sel[0] << shift;
        pmask |= 255u << shift;
        k -= sel[1];
        __syncthreads();
    }
    // every split's N-th smallest is an upper bound of the true N-th: keep the least
    if (threadIdx.x == 0) atomicMin(&a.tau0[(size_t)q * a.n_sub + i], prefix);
}

// Two-kernel seed (the default): every sample row is loaded ONCE per block and scored
// against 32 frames (rows in registers, frames broadcast from shared memory), the
// exact chains' acc bits go to a scratch array, then one CTA per (frame, subspace,
// split) radix-selects the N-th smallest from it (8-bit digits from the top, warp-
// aggregated shared-memory histograms).  Same sample rows and the same values as
// tau_seed_kernel, far fewer bytes: rows are reused across frames.
constexpr int kSeedFrames = 32;

template <int KC>
__global__ void __launch_bounds__(256) seed_acc_kernel(SeedArgs a) {
    // frames as interleaved pairs: qd[p][k] = (q_{2p}[k], q_{2p+1}[k]), so one f32x2 FADD2 + FFMA2
    // advances two frames' chains (each lane of the pair the exact RN fp32 step of R3)
    __shared__ alignas(16) uint64_t qd[kSeedFrames / 2][kK];
    const uint32_t isp = blockIdx.x;                     // (subspace, split)
    const uint32_t i = isp / a.splits, split = isp % a.splits;
    const uint32_t f0 = blockIdx.z * kSeedFrames;
    const uint32_t nf = min((uint32_t)kSeedFrames, a.nq - f0);
    for (uint32_t t = threadIdx.x; t < (kSeedFrames / 2) * kK; t += blockDim.x) {
        const uint32_t p = t / kK, k = t % kK;
        const float lo = 2 * p < nf ? a.queries[(size_t)(f0 + 2 * p) * kK + k] : 0.f;
        const float hi = 2 * p + 1 < nf ? a.queries[(size_t)(f0 + 2 * p + 1) * kK + k] : 0.f;
        qd[p][k] = f2pack(lo, hi);
    }
    __syncthreads();
    const SubInfo si = a.subs[i];
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, si.count);
    const uint32_t smp = blockIdx.y * blockDim.x + threadIdx.x;
    if (S < a.N || smp >= S) return;
    const uint64_t row = si.row_begin + (((uint64_t)smp * a.splits + split) * si.count) / ((uint64_t)S * a.splits);
    if (!OL_DCHECK(row < si.row_begin + si.count && row < a.rows_pad && f0 + nf <= a.nq)) return;
    float4 f[kK / 4];
#pragma unroll
    for (int k4 = 0; k4 < kK / 4; ++k4)
        f[k4] = __ldg(reinterpret_cast<const float4 *>(a.fine + fine_off(row, 4 * k4)));
    const size_t fstride = (size_t)a.n_sub * a.splits * a.samples;
    uint32_t *out = a.scratch + ((size_t)f0 * a.n_sub + i) * a.splits * a.samples + (size_t)split * a.samples + smp;
    // four frames at a time: two f32x2 chains in flight
    for (uint32_t p = 0; 2 * p < nf; p += 2) {
        const ulonglong2 *qa = reinterpret_cast<const ulonglong2 *>(qd[p]);
        const ulonglong2 *qb = reinterpret_cast<const ulonglong2 *>(qd[p + 1 < kSeedFrames / 2 ? p + 1 : p]);
        uint64_t acc0 = 0, acc1 = 0;
#pragma unroll
        for (int k4 = 0; k4 < kK / 4; ++k4) {
            const float fv[4] = {f[k4].x, f[k4].y, f[k4].z, f[k4].w};
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const ulonglong2 x = qa[2 * k4 + c], y = qb[2 * k4 + c];
                const uint64_t fa = f2pack(fv[2 * c], fv[2 * c]), fb = f2pack(fv[2 * c + 1], fv[2 * c + 1]);
                uint64_t d = f2sub(x.x, fa); acc0 = f2fma(d, d, acc0);
                d = f2sub(y.x, fa); acc1 = f2fma(d, d, acc1);
                d = f2sub(x.y, fb); acc0 = f2fma(d, d, acc0);
                d = f2sub(y.y, fb); acc1 = f2fma(d, d, acc1);
            }
        }
        const uint32_t j = 2 * p;
        out[j * fstride] = (uint32_t)acc0;
        if (j + 1 < nf) out[(j + 1) * fstride] = (uint32_t)(acc0 >> 32);
        if (j + 2 < nf) out[(j + 2) * fstride] = (uint32_t)acc1;
        if (j + 3 < nf) out[(j + 3) * fstride] = (uint32_t)(acc1 >> 32);
    }
}

// One CTA per (frame, subspace, split): the N-th smallest of its S acc bits by radix
// select (4 passes of 8-bit digits, most significant first).  Every pass streams the
// job's values from L2 with all of a thread's loads in flight; counts go to one shared
// histogram (warp-aggregated increments: equal digits of a warp add once); a CTA-wide
// scan of the 256 counts finds the digit holding the k-th value.
__global__ void __launch_bounds__(256) seed_select_kernel(SeedArgs a) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t wsum[8];
    __shared__ uint32_t pick[2];
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const uint32_t job = blockIdx.x;   // (frame, subspace, split)
    const uint32_t i = (job / a.splits) % a.n_sub, q = (job / a.splits) / a.n_sub;
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, a.subs[i].count);
    if (S < a.N) return;   // (uniform over the CTA)
    const uint32_t *v = a.scratch + (size_t)job * a.samples;
    uint32_t prefix = 0, pmask = 0, k = a.N;
    for (int shift = 24; shift >= 0; shift -= 8) {
        hist[tid] = 0;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < S; t0 += 8 * 256) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 256 + tid;
                x[j] = t < S ? __ldcg(v + t) : 0u;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 256 + tid;
                const bool in = t < S && (x[j] & pmask) == prefix;
                const uint32_t d = in ? (x[j] >> shift) & 255u : 256u;
                const uint32_t peers = __match_any_sync(0xffffffffu, d);
                if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[d], (uint32_t)__popc(peers));
            }
        }
        __syncthreads();
        // inclusive scan of the 256 counts (thread = digit)
        const uint32_t c = hist[tid];
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) wsum[w] = incl;
        __syncthreads();
        for (int j = 0; j < w; ++j) incl += wsum[j];
        if (incl - c < k && k <= incl) { pick[0] = (uint32_t)tid; pick[1] = incl - c; }
        __syncthreads();
        prefix |= pick[0] << shift;
        pmask |= 255u << shift;
        k -= pick[1];
        __syncthreads();
    }
    // every split's N-th smallest is an upper bound of the true N-th: keep the least
    if (tid == 0) atomicMin(&a.tau0[(size_t)q * a.n_sub + i], prefix);
}

// N <= 32 (about one pass over the job's values instead of four): T = the N-th smallest of
// 512 evenly strided values (an upper bound of the N-th smallest of all S), then every value
// <= T -- about N x S / 512 of them -- is gathered into shared memory and the N-th smallest
// of those is the answer (keys acc bits << 32 | sample index are unique; ties in acc resolve
// to the same value).  If more than kSelBuf values are <= T, the N-th smallest of the
// gathered ones is a tighter bound: gather again below it (at most 3 rounds; the last bound
// found is valid in any case).
constexpr uint32_t kSelBuf = 2048;
__global__ void __launch_bounds__(256) seed_select_small_kernel(SeedArgs a) {
    __shared__ u64 buf[kSelBuf];
    __shared__ u64 sel[32];
    __shared__ u64 scratch[256];
    __shared__ uint32_t nbuf;
    const uint32_t job = blockIdx.x;   // (frame, subspace, split)
    const uint32_t i = (job / a.splits) % a.n_sub, q = (job / a.splits) / a.n_sub;
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, a.subs[i].count);
    if (S < a.N) return;   // (uniform over the CTA)
    const uint32_t *v = a.scratch + (size_t)job * a.samples;
    const uint32_t S0 = min(S, 512u);
    for (uint32_t t = threadIdx.x; t < S0; t += blockDim.x) {
        const uint32_t idx = (uint32_t)(((uint64_t)t * S) / S0);
        buf[t] = ((u64)__ldcg(v + idx) << 32) | idx;
    }
    __syncthreads();
    block_select32(buf, S0, a.N, sel, scratch);
    __syncthreads();
    uint32_t T = (uint32_t)(sel[a.N - 1] >> 32);
    for (int round = 0; round < 3; ++round) {
        if (threadIdx.x == 0) nbuf = 0;
        __syncthreads();
        for (uint32_t t0 = 0; t0 < S; t0 += 8 * 256) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 256 + threadIdx.x;
                x[j] = t < S ? __ldcg(v + t) : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 256 + threadIdx.x;
                if (t < S && x[j] <= T) {
                    const uint32_t pos = atomicAdd(&nbuf, 1u);
                    if (pos < kSelBuf) buf[pos] = ((u64)x[j] << 32) | t;
                }
            }
        }
        __syncthreads();
        const uint32_t nb = nbuf;
        block_select32(buf, min(nb, kSelBuf), a.N, sel, scratch);
        __syncthreads();
        T = (uint32_t)(sel[a.N - 1] >> 32);   // (N values <= it: a valid bound either way)
        __syncthreads();
        if (nb <= kSelBuf) break;              // exact: every value <= the old T was gathered
    }
    // every split's N-th smallest is an upper bound of the true N-th: keep the least
    if (threadIdx.x == 0) atomicMin(&a.tau0[(size_t)q * a.n_sub + i], T);
}

// Warp per job, 2,048 <= S <= 4,096 and N <= 32 (many mid-sized jobs: C3 split into 50 subspaces is
// 51,200 jobs of 2,500 samples).  T = the N-th smallest of 256 evenly strided values (N
// real samples: an upper bound of the N-th smallest of all S); one pass gathers every value
// <= T, compacted by ballot into the warp's shared buffer (about N x S / 256 of them); the
// N-th smallest of the gathered is the answer when they all fit (exact); otherwise the
// N-th smallest of those that fit (N real samples: a valid, tighter bound) is gathered
// below again, at most 3 rounds (or until it stops moving: ties).  Sorting networks on 32-key warp
// lists (warp_sort32 / warp_merge32), no CTA barriers.
constexpr uint32_t kWSelBuf = 512;
__global__ void __launch_bounds__(256) seed_select_gather_warp_kernel(SeedArgs a) {
    __shared__ u64 buf[8][kWSelBuf];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t job = blockIdx.x * 8 + w;   // (frame, subspace, split)
    if (job >= a.nq * a.n_sub * a.splits) return;   // (whole warps)
    const uint32_t i = (job / a.splits) % a.n_sub, q = (job / a.splits) / a.n_sub;
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, a.subs[i].count);
    if (S < a.N) return;
    const uint32_t *v = a.scratch + (size_t)job * a.samples;
    const uint32_t S0 = min(S, 256u);
    u64 run = kPadKey;
    for (uint32_t b = 0; b < S0; b += 32) {
        const uint32_t t = b + lane;
        u64 k = kPadKey;
        if (t < S0) {
            const uint32_t idx = (uint32_t)(((uint64_t)t * S) / S0);
            k = ((u64)__ldcg(v + idx) << 32) | idx;
        }
        run = warp_merge32(run, warp_sort32(k, lane), lane);
    }
    uint32_t T = (uint32_t)(__shfl_sync(0xffffffffu, run, a.N - 1) >> 32);
    uint32_t R = T;
    for (int round = 0; round < 3; ++round) {
        uint32_t nb = 0;
        for (uint32_t t0 = 0; t0 < S; t0 += 32 * 8) {
            uint32_t x[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 32 + lane;
                x[j] = t < S ? __ldcg(v + t) : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t t = t0 + j * 32 + lane;
                const bool in = t < S && x[j] <= T;
                const unsigned m = __ballot_sync(0xffffffffu, in);
                if (in) {
                    const uint32_t pos = nb + __popc(m & ((1u << lane) - 1u));
                    if (pos < kWSelBuf) buf[w][pos] = ((u64)x[j] << 32) | t;
                }
                nb += __popc(m);
            }
        }
        __syncwarp();
        const uint32_t ng = min(nb, kWSelBuf);   // >= N: N samples are <= T
        run = kPadKey;
        for (uint32_t b = 0; b < ng; b += 32) {
            const u64 k = b + lane < ng ? buf[w][b + lane] : kPadKey;
            run = warp_merge32(run, warp_sort32(k, lane), lane);
        }
        __syncwarp();
        R = (uint32_t)(__shfl_sync(0xffffffffu, run, a.N - 1) >> 32);   // (N samples <= R: valid)
        if (nb <= kWSelBuf || R == T) break;     // exact: every value <= T was gathered
        T = R;                                   // (overflow: again below the tighter bound)
    }
    // every split's N-th smallest is an upper bound of the true N-th: keep the least
    if (lane == 0) atomicMin(&a.tau0[(size_t)q * a.n_sub + i], R);
}

// Warp per job (small samples, many jobs: a CTA per job would mostly wait at barriers).
__global__ void __launch_bounds__(256) seed_select_warp_kernel(SeedArgs a) {
    __shared__ uint32_t hist[8][256];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t job = blockIdx.x * 8 + w;   // (frame, subspace, split)
    if (job >= a.nq * a.n_sub * a.splits) return;   // (whole warps only: warp-level sync below)
    const uint32_t i = (job / a.splits) % a.n_sub, q = (job / a.splits) / a.n_sub;
    const uint32_t S = (uint32_t)min((uint64_t)a.samples, a.subs[i].count);
    if (S < a.N) return;
    const uint32_t *v = a.scratch + (size_t)job * a.samples;
    uint32_t prefix = 0, pmask = 0, k = a.N;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = lane; b < 256; b += 32) hist[w][b] = 0;
        __syncwarp();
        for (uint32_t t0 = 0; t0 < S; t0 += 32) {
            const uint32_t t = t0 + lane;
            const uint32_t x = t < S ? __ldcg(v + t) : 0u;
            const bool in = t < S && (x & pmask) == prefix;
            const uint32_t d = in ? (x >> shift) & 255u : 256u;
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (in && lane == __ffs(peers) - 1) atomicAdd(&hist[w][d], (uint32_t)__popc(peers));
        }
        __syncwarp();
        uint32_t c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { c[j] = hist[w][lane * 8 + j]; tot += c[j]; }
        uint32_t incl = tot;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        uint32_t below = incl - tot, digit = 0, under = 0;
        const bool here = below < k && k <= incl;
        if (here) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (below + c[j] >= k) { digit = lane * 8 + j; under = below; break; }
                below += c[j];
            }
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, here)) - 1;
        digit = __shfl_sync(0xffffffffu, digit, src);
        under = __shfl_sync(0xffffffffu, under, src);
        prefix |= digit << shift;
        pmask |= 255u << shift;
        k -= under;
        __syncwarp();
    }
    // every split's N-th smallest is an upper bound of the true N-th: keep the least
    if (lane == 0) atomicMin(&a.tau0[(size_t)q * a.n_sub + i], prefix);
}

cudaError_t launch_tau_seed(const SeedArgs &a, cudaStream_t s) {
    if (a.scratch) {
        // 64-thread CTAs when 256 would leave SMs idle (few frames)
        const uint32_t fz = (a.nq + kSeedFrames - 1) / kSeedFrames;
        const uint32_t bt = (uint64_t)a.n_sub * a.splits * ((a.samples + 255) / 256) * fz < 2 * 148 ? 64 : 256;
        const dim3 g1(a.n_sub * a.splits, (a.samples + bt - 1) / bt, fz);
        switch (a.kc) {
            case 8: seed_acc_kernel<8><<<g1, bt, 0, s>>>(a); break;
            case 16: seed_acc_kernel<16><<<g1, bt, 0, s>>>(a); break;
            case 32: seed_acc_kernel<32><<<g1, bt, 0, s>>>(a); break;
            case 64: seed_acc_kernel<64><<<g1, bt, 0, s>>>(a); break;
            default: return cudaErrorInvalidValue;
        }
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        // one CTA per job streams large samples with its loads in flight (C4: 170 -> 28 us);
        // a warp per job is faster for small ones: gathering below a strided bound for 2,048-4,096
        // samples (C3 / 50 subspaces, 2,500 x 51,200 jobs: 0.31 vs 0.68 ms; at 8,192 samples it
        // loses), radix passes below 2,048 (C2, 500 samples x 25,000 jobs: 0.173 vs 0.198 ms for
        // the gather, 0.32 ms for the CTA per job)
        const uint32_t jobs = a.nq * a.n_sub * a.splits;
        if (a.samples >= 2048 && a.samples <= 4096 && a.N <= 32 && !a.select_old) seed_select_gather_warp_kernel<<<(jobs + 7) / 8, 256, 0, s>>>(a);
        else if (a.samples >= 2048 && a.N <= 32) seed_select_small_kernel<<<a.nq * a.n_sub * a.splits, 256, 0, s>>>(a);
        else if (a.samples >= 2048) seed_select_kernel<<<a.nq * a.n_sub * a.splits, 256, 0, s>>>(a);
        else seed_select_warp_kernel<<<(a.nq * a.n_sub * a.splits + 7) / 8, 256, 0, s>>>(a);
        return cudaGetLastError();
    }
    const unsigned grid = a.nq * a.n_sub * a.splits;
    switch (a.kc) {
        case 8: tau_seed_kernel<8><<<grid, kSeedThreads, 0, s>>>(a); break;
        case 16: tau_seed_kernel<16><<<grid, kSeedThreads, 0, s>>>(a); break;
        case 32: tau_seed_kernel<32><<<grid, kSeedThreads, 0, s>>>(a); break;
        case 64: tau_seed_kernel<64><<<grid, kSeedThreads, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ upload helpers
// [rows][64] source rows -> tiled coarse plane (rows dst_row0 ..) + row-major fine plane (full rows)
__global__ void relayout_kernel(const float *src, uint64_t rows, uint64_t dst_row0, int kc, float *coarse,
                                float *fine) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows * kK;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = i / kK, d = dst_row0 + r;
        const int k = (int)(i % kK);
        const float v = src[i];
        if (k < kc) coarse[coarse_off(d, k, kc)] = v;
        fine[fine_off(d, k)] = v;
    }
}

cudaError_t launch_relayout(const float *src, uint64_t rows, uint64_t dst_row0, int kc, float *coarse,
                            float *fine, cudaStream_t s) {
    uint64_t blocks = (rows * kK + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    relayout_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, rows, dst_row0, kc, coarse, fine);
    return cudaGetLastError();
}

// Tile-padding rows (count .. next multiple of 32) of each subspace <- its last row.
__global__ void pad_rows_kernel(const SubInfo *subs, uint32_t n_sub, int kc, float *coarse, float *fine) {
    const uint32_t i = blockIdx.x;
    const SubInfo si = subs[i];
    const uint64_t pad = (si.count + kPadRows - 1) / kPadRows * kPadRows;
    if (si.count == 0) return;
    const uint64_t src = si.row_begin + si.count - 1;
    for (uint64_t p = si.count + threadIdx.x / kK; p < pad; p += blockDim.x / kK) {
        const uint64_t dst = si.row_begin + p;
        const int k = threadIdx.x % kK;
        if (k < kc) coarse[coarse_off(dst, k, kc)] = coarse[coarse_off(src, k, kc)];
        fine[fine_off(dst, k)] = fine[fine_off(src, k)];
    }
}

cudaError_t launch_pad_rows(const SubInfo *subs, uint32_t n_sub, int kc, float *coarse, float *fine, cudaStream_t s) {
    if (n_sub == 0) return cudaSuccess;
    pad_rows_kernel<<<n_sub, 256, 0, s>>>(subs, n_sub, kc, coarse, fine);
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

__global__ void check_coords_kernel(const int32_t *xy, uint64_t rows, int32_t x0, int32_t x1, int32_t y0,
                                    int32_t y1, int *flag) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < rows;
         i += (uint64_t)gridDim.x * blockDim.x) {
        int32_t x = xy[2 * i], y = xy[2 * i + 1];
        if (x < x0 || x >= x1 || y < y0 || y >= y1) *flag = 1;
    }
}

cudaError_t launch_check_coords(const int32_t *xy, uint64_t rows, int32_t x0, int32_t x1, int32_t y0,
                                int32_t y1, int *flag, cudaStream_t s) {
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    check_coords_kernel<<<(unsigned)blocks, 256, 0, s>>>(xy, rows, x0, x1, y0, y1, flag);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_scan)

}  // namespace ol
