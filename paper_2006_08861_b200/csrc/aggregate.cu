// aggregate.cu -- Algorithm 2, 2-D multi-frame candidate aggregation
// on sm_100a (kernel NK5).  One CTA per bundle, all in shared memory:
//   1. 2-D binning (Alg. 2 steps 2-3): sort the candidates' tile keys (y, x);
//      runs of equal keys are the non-zero tiles of locationDistriArray and
//      their lengths the counts (a sparse histogram: only occupied tiles exist);
//   2. rankLocationDistribution / findTopDensityArea (steps 5-6): sort the
//      occupied tiles by (count desc, y asc, x asc) (R7) and keep TopC;
//   3. the tolerance circle of each ranked tile (step 7-8): the sum of
//      the counts of the occupied tiles whose centre lies within radius_m
//      (dx^2 + dy^2 <= (radius_m / tile_m)^2, inclusive, R11);
//   4. the first ranked tile whose circle > toler_per * total (strict)
//      wins; if none does, the ranked tile with the largest circle (earliest
//      rank on ties) flagged low-confidence (R12).
#define OL_TU 3
#include "ol_internal.h"
#include "tc_ptx.cuh"   // (cluster barrier, shared-memory addresses)

namespace ol {

using tc::cluster_sync;
using tc::smem_u32;

constexpr int kAggThreads = 512;

__device__ void bitonic_sort_u64(u64 *v, uint32_t P) {
    for (uint32_t k = 2; k <= P; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
                uint32_t o = t ^ j;
                if (o > t) {
                    bool up = (t & k) == 0;
                    u64 x = v[t], y = v[o];
                    if ((x > y) == up) { v[t] = y; v[o] = x; }
                }
            }
            __syncthreads();
        }
    }
}

// exclusive block scan of one value per thread; returns the thread's offset, *total
__device__ uint32_t block_excl_scan(uint32_t v, uint32_t *scratch, uint32_t *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) scratch[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < (int)(blockDim.x / 32) ? scratch[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        scratch[lane] = w;  // inclusive prefix over warps
    }
    __syncthreads();
    uint32_t res = x - v + (warp > 0 ? scratch[warp - 1] : 0);
    *total = scratch[blockDim.x / 32 - 1];
    __syncthreads();
    return res;
}

// Tile sort key: (y, x) with both halves biased by 2^31, so unsigned key order is the
// signed (y asc, x asc) order of the ranking tie-break (R7) for any int32 tile,
// negative ones included (the unbiased key sorted negative tiles last).
__device__ __forceinline__ u64 tile_key(int32_t x, int32_t y) {
    return ((u64)((uint32_t)y ^ 0x80000000u) << 32) | ((uint32_t)x ^ 0x80000000u);
}
__device__ __forceinline__ int32_t key_x(u64 k) { return (int32_t)((uint32_t)k ^ 0x80000000u); }
__device__ __forceinline__ int32_t key_y(u64 k) { return (int32_t)((uint32_t)(k >> 32) ^ 0x80000000u); }

// Algorithm 2 for a bundle of 1..32 candidates by one warp, lane = candidate: the steps and
// tie rules of aggregate_block below, with shuffles in place of its shared-memory sorts and
// block barriers (a bundle of C4 / C1 size costs a few hundred cycles instead of ~12k).
__device__ __noinline__ void aggregate_warp(const AggArgs &a, uint32_t b, uint32_t begin, uint32_t total) {
    constexpr uint32_t kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    ol_estimate *out = a.out + b;
    u64 k = kPadKey;
    if ((uint32_t)lane < total) {
        int32_t x, y;
        if (a.cand) { x = a.cand[begin + lane].x; y = a.cand[begin + lane].y; }
        else { x = a.xy[2 * (size_t)(begin + lane)]; y = a.xy[2 * (size_t)(begin + lane) + 1]; }
        k = tile_key(x, y);
    }
    // step 1: the 32 keys sorted ascending across the lanes; runs of equal keys are the occupied
    // tiles, a run's length its count
    k = warp_sort32(k, lane);
    const u64 prev = __shfl_up_sync(kAll, k, 1);
    const bool start = (uint32_t)lane < total && (lane == 0 || k != prev);
    const uint32_t starts = __ballot_sync(kAll, start);
    const uint32_t nd = __popc(starts);
    uint32_t cnt = 0;
    if (start) {
        const uint32_t later = lane == 31 ? 0u : starts & ~((2u << lane) - 1u);
        cnt = (later ? (uint32_t)(__ffs(later) - 1) : total) - (uint32_t)lane;
    }
    // step 2: rank = #tiles before it in (count desc, (y, x) asc) order; lanes of run starts are
    // in (y, x) order already
    uint32_t rank = 0;
    for (int j = 0; j < (int)total; ++j) {   // (run starts lie below total; warp-uniform bound)
        const uint32_t cj = __shfl_sync(kAll, cnt, j);
        if (((starts >> j) & 1u) && (cj > cnt || (cj == cnt && j < lane))) ++rank;
    }
    const uint32_t nr = min(a.top_c, nd);
    const bool ranked = start && rank < nr;
    // step 3: the tolerance circle of every ranked tile
    const int64_t cx = key_x(k), cy = key_y(k);
    uint32_t circ = 0;
    for (int j = 0; j < (int)total; ++j) {
        const u64 kj = __shfl_sync(kAll, k, j);
        const uint32_t cj = __shfl_sync(kAll, cnt, j);
        if ((starts >> j) & 1u) {
            const int64_t dx = (int64_t)key_x(kj) - cx;
            const int64_t dy = (int64_t)key_y(kj) - cy;
            if ((double)(dx * dx + dy * dy) <= a.r2) circ += cj;
        }
    }
    // step 4: the first ranked tile whose circle > toler_per * total, else the largest circle
    // (earliest rank on ties), low confidence
    const double thresh = a.toler_per * (double)total;
    const uint32_t chosen = __reduce_min_sync(kAll, ranked && (double)circ > thresh ? rank : 0xFFFFFFFFu);
    const uint32_t best = 63u - (__reduce_max_sync(kAll, ranked ? (circ << 6) | (63u - rank) : 0u) & 63u);
    const uint32_t low = chosen == 0xFFFFFFFFu ? 1u : 0u;
    const uint32_t win = low ? best : chosen;
    if (ranked && rank == win) {
        out->x = key_x(k);
        out->y = key_y(k);
        out->x_m = a.tile_m * (double)out->x;
        out->y_m = a.tile_m * (double)out->y;
        out->confidence = (double)circ / (double)total;
        out->low_confidence = low;
        out->n_ranked = nr;
        out->total = total;
        out->_pad = 0;
    }
    if (ranked) {
        ol_ranked_tile rt;
        rt.x = key_x(k); rt.y = key_y(k); rt.count = cnt; rt.circle = circ;
        out->ranked[rank] = rt;
    }
    for (uint32_t r = lane; r < OL_MAX_TOP_C; r += 32)
        if (r >= nr) out->ranked[r] = ol_ranked_tile{0, 0, 0, 0};
}

// Algorithm 2 for bundle b, by the whole CTA (kAggThreads threads); smem: the dynamic shared
// memory (2 x cap u64 + cap u32).  Shared by aggregate_kernel and micro_kernel.  Bundles of
// at most 32 candidates go to aggregate_warp (warp 0; the other warps return).
__device__ __noinline__ void aggregate_block(const AggArgs &a, uint32_t b, unsigned char *smem) {
    __shared__ uint32_t scratch[32];
    __shared__ uint32_t circ[OL_MAX_TOP_C];
    __shared__ uint32_t red[kAggThreads / 32];
    uint32_t begin, total;
    if (a.cand) { begin = b * a.per_bundle; total = a.per_bundle; }
    else { begin = a.offsets[b]; total = a.offsets[b + 1] - begin; }
    ol_estimate *out = a.out + b;
    const uint32_t cap = a.cap ? a.cap : (uint32_t)kAggMax;   // shared-memory entries
    if (total == 0 || total > cap) {
        if (threadIdx.x == 0) { *a.err_empty = total == 0 ? 1 : 2; out->total = total; }
        return;
    }
    if (total <= 32 && !a.block_only) {
        if (threadIdx.x < 32) aggregate_warp(a, b, begin, total);
        return;
    }
    uint32_t P = 1;
    while (P < total) P <<= 1;
    if (!OL_DCHECK(P <= cap && cap <= (uint32_t)kAggMax)) return;   // the sort fits the shared arrays
    u64 *keys = reinterpret_cast<u64 *>(smem);          // [P]  sorted candidate tiles
    u64 *dtile = keys + cap;                            // [P]  occupied tiles
    uint32_t *dcount = reinterpret_cast<uint32_t *>(dtile + cap);  // [P]
    for (uint32_t t = threadIdx.x; t < P; t += blockDim.x) {
        u64 k = kPadKey;
        if (t < total) {
            int32_t x, y;
            if (a.cand) { x = a.cand[begin + t].x; y = a.cand[begin + t].y; }
            else { x = a.xy[2 * (size_t)(begin + t)]; y = a.xy[2 * (size_t)(begin + t) + 1]; }
            k = tile_key(x, y);
        }
        keys[t] = k;
    }
    __syncthreads();
    // step 1: binning by sort
    bitonic_sort_u64(keys, P);
    const uint32_t per = (P + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = threadIdx.x * per, hi = min(lo + per, total);
    uint32_t mine = 0;
    for (uint32_t t = lo; t < hi; ++t) mine += (t == 0 || keys[t] != keys[t - 1]);
    uint32_t nd;
    uint32_t pos = block_excl_scan(mine, scratch, &nd);
    uint32_t *first = reinterpret_cast<uint32_t *>(dcount);  // temporarily: run starts
    for (uint32_t t = lo; t < hi; ++t)
        if (t == 0 || keys[t] != keys[t - 1]) { dtile[pos] = keys[t]; first[pos] = t; ++pos; }
    __syncthreads();
    uint32_t cnt[16];  // per <= kAggMax / kAggThreads
    const uint32_t dper = (nd + blockDim.x - 1) / blockDim.x;
    for (uint32_t j = 0; j < dper; ++j) {
        uint32_t d = threadIdx.x * dper + j;
        cnt[j] = d < nd ? ((d + 1 < nd ? first[d + 1] : total) - first[d]) : 0;
    }
    __syncthreads();
    for (uint32_t j = 0; j < dper; ++j) {
        uint32_t d = threadIdx.x * dper + j;
        if (d < nd) dcount[d] = cnt[j];
    }
    __syncthreads();
    // step 2: rank occupied tiles (count desc; ties by (y, x) = position in dtile)
    uint32_t PD = 1;
    while (PD < nd) PD <<= 1;
    for (uint32_t d = threadIdx.x; d < PD; d += blockDim.x)
        keys[d] = d < nd ? (((u64)(0xFFFFFFFFu - dcount[d]) << 32) | d) : kPadKey;
    __syncthreads();
    bitonic_sort_u64(keys, PD);
    const uint32_t nr = min(a.top_c, nd);
    // step 3: tolerance circles
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint32_t r = 0; r < nr; ++r) {
        const u64 c = dtile[(uint32_t)keys[r]];
        const int64_t cx = key_x(c), cy = key_y(c);
        uint32_t s = 0;
        for (uint32_t d = threadIdx.x; d < nd; d += blockDim.x) {
            const u64 t = dtile[d];
            const int64_t dx = (int64_t)key_x(t) - cx;
            const int64_t dy = (int64_t)key_y(t) - cy;
            if ((double)(dx * dx + dy * dy) <= a.r2) s += dcount[d];
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            for (int w = 0; w < kAggThreads / 32; ++w) tot += red[w];
            circ[r] = tot;
        }
        __syncthreads();
    }
    // step 4: decision
    if (threadIdx.x == 0) {
        const double thresh = a.toler_per * (double)total;
        int chosen = -1, best = 0;
        for (uint32_t r = 0; r < nr; ++r) {
            if (chosen < 0 && (double)circ[r] > thresh) chosen = (int)r;
            if (circ[r] > circ[best]) best = (int)r;
        }
        uint32_t low = 0;
        if (chosen < 0) { chosen = best; low = 1; }
        const u64 c = dtile[(uint32_t)keys[chosen]];
        out->x = key_x(c);
        out->y = key_y(c);
        out->x_m = a.tile_m * (double)out->x;
        out->y_m = a.tile_m * (double)out->y;
        out->confidence = (double)circ[chosen] / (double)total;
        out->low_confidence = low;
        out->n_ranked = nr;
        out->total = total;
        out->_pad = 0;
    }
    for (uint32_t r = threadIdx.x; r < OL_MAX_TOP_C; r += blockDim.x) {
        ol_ranked_tile rt = {0, 0, 0, 0};
        if (r < nr) {
            const uint32_t d = (uint32_t)keys[r];
            const u64 c = dtile[d];
            rt.x = key_x(c);
            rt.y = key_y(c);
            rt.count = dcount[d];
            rt.circle = circ[r];
        }
        out->ranked[r] = rt;
    }
}

__global__ void __launch_bounds__(kAggThreads) aggregate_kernel(AggArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    aggregate_block(a, blockIdx.x, smem);
}

// ---------------------------------------------------------------- small problems (NK10)
// The whole launch sequence of a small world-1 query in ONE kernel (the latency configs:
// C1 = 2,000 rows x 1 frame ran 6 launches, ~5 us each).  Each (frame, subspace) job is one
// cluster of a.split CTAs (1, 2, 4 or 8; a single CTA read C1's 512 KB of rows at one SM's L2
// bandwidth, ~14 us): CTA g scores its contiguous share of the subspace's rows with the exact
// chain of R3 (k = 0..63 in order; the coarse plane for k < kc, the fine plane after -- the
// same values as one pass), keeps the keys (acc bits << 32 | frame) in shared memory and
// selects its min(N, rows) smallest (warp 0, rounds of a warp minimum above the previous one;
// keys are unique).  Cluster rank 0 reads the shares' lists over distributed shared memory
// and selects the N smallest of them -- the N smallest of the union, as every row is in
// exactly one share -- writes the candidate rows in SPEC order and, when its job is
// the last of its bundle (a counter per bundle; none for one-job bundles), runs Algorithm 2
// for the bundle.  Results are the plain definition's, bit for bit, like every other path.
//
// The c smallest keys above nothing of keys[0..n) (shared memory), ascending, into sel[0..c),
// by warp 0.
__device__ __forceinline__ void micro_select(const u64 *keys, uint32_t n, uint32_t c, u64 *sel, int lane) {
    u64 lo = 0;
    for (uint32_t r = 0; r < c; ++r) {
        u64 best = kPadKey;
        for (uint32_t t = lane; t < n; t += 32) {
            const u64 v = keys[t];
            if ((r == 0 || v > lo) && v < best) best = v;
        }
        for (int o = 16; o; o >>= 1) {
            const u64 w = __shfl_xor_sync(0xffffffffu, best, o);
            best = w < best ? w : best;
        }
        lo = best;
        if (lane == 0) sel[r] = best;
    }
}

__global__ void __launch_bounds__(kAggThreads) micro_kernel(MicroArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ __align__(16) float qs[kK];
    __shared__ u64 sel[OL_MAX_N];
    __shared__ u64 scratch[kAggThreads];
    __shared__ uint32_t is_last;
    const uint32_t split = a.split;
    const uint32_t job = blockIdx.x / split, g = blockIdx.x % split;
    const uint32_t q = job / a.n_sub, i = job % a.n_sub;
    const long long p0 = clock64();
    const SubInfo si = a.subs[i];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < kK) {
        const float v = a.queries[(size_t)q * kK + threadIdx.x];
        qs[threadIdx.x] = v;
        if (a.check_finite && g == 0 && !isfinite(v)) *a.flag_nonfinite = 1;
    }
    __syncthreads();
    u64 *keys = reinterpret_cast<u64 *>(smem);   // [share]
    const uint32_t n = (uint32_t)si.count;
    const uint32_t per = (n + split - 1) / split;          // this job's rows per share
    const uint32_t r_lo = min(n, g * per), cnt = min(n, r_lo + per) - r_lo;
    // one row per thread per pass, its 16 float4 loads in flight together (a small query is
    // latency-bound: one L2 round trip per pass), from the fine plane's full row
    const float4 *q4 = reinterpret_cast<const float4 *>(qs);
    for (uint32_t r = threadIdx.x; r < cnt; r += blockDim.x) {
        const uint64_t row = si.row_begin + r_lo + r;
        float4 f[kK / 4];
#pragma unroll
        for (int k4 = 0; k4 < kK / 4; ++k4) {
            f[k4] = __ldg(reinterpret_cast<const float4 *>(a.fine + fine_off(row, 4 * k4)));
        }
        float acc = 0.f;
#pragma unroll
        for (int k4 = 0; k4 < kK / 4; ++k4) {
            const float4 x = q4[k4];
            float d = __fsub_rn(x.x, f[k4].x); acc = __fmaf_rn(d, d, acc);
            d = __fsub_rn(x.y, f[k4].y); acc = __fmaf_rn(d, d, acc);
            d = __fsub_rn(x.z, f[k4].z); acc = __fmaf_rn(d, d, acc);
            d = __fsub_rn(x.w, f[k4].w); acc = __fmaf_rn(d, d, acc);
        }
        keys[r] = ((u64)__float_as_uint(acc) << 32) | (u64)(si.shard_begin + r_lo + r);
    }
    __syncthreads();
    const long long p1 = clock64();
    const uint32_t c = min(a.N, n);   // min(N, |n_i|) rows
    if (split == 1) {
        if (c <= 32) block_select32(keys, cnt, c, sel, scratch);
        else if (warp == 0) micro_select(keys, cnt, c, sel, lane);
    } else {
        // this share's min(N, cnt) smallest, padded to N; rank 0 gathers every share's list
        const uint32_t cl = min(a.N, cnt);
        if (cl <= 32) block_select32(keys, cnt, cl, sel, scratch);
        else if (warp == 0) micro_select(keys, cnt, cl, sel, lane);
        __syncthreads();
        for (uint32_t r = cl + threadIdx.x; r < a.N; r += blockDim.x) sel[r] = kPadKey;
        const long long pa = clock64();
        cluster_sync();   // (release / acquire: the lists are visible across the cluster)
        const long long pb = clock64();
        if (a.prof && threadIdx.x == 0 && g == 0) { atomicAdd(&a.prof[4], (unsigned long long)(pa - p1));
                                                    atomicAdd(&a.prof[5], (unsigned long long)(pb - pa)); }
        if (g == 0) {
            const uint32_t local = smem_u32(sel);
            for (uint32_t t = threadIdx.x; t < split * a.N; t += blockDim.x) {
                uint32_t ra;
                u64 v;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(local + 8u * (t % a.N)), "r"(t / a.N));
                asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
                keys[t] = v;
            }
        }
        cluster_sync();   // (the other shares may exit once rank 0 has read them)
        if (g != 0) return;
        const long long pc = clock64();
        __syncthreads();
        if (c <= 32) block_select32(keys, split * a.N, c, sel, scratch);
        else if (warp == 0) micro_select(keys, split * a.N, c, sel, lane);
        if (a.prof && threadIdx.x == 0) { atomicAdd(&a.prof[6], (unsigned long long)(pc - pb)); }
    }
    const long long pd = clock64();
    __syncthreads();
    // the candidate rows, all c in parallel (one coords round trip, not c)
    ol_candidate *co = a.cand + (uint64_t)q * a.sub_prefix[a.n_sub] + a.sub_prefix[i];
    for (uint32_t r = threadIdx.x; r < c; r += blockDim.x) {
        const u64 v = sel[r];
        const uint32_t frame = (uint32_t)v;
        const uint64_t row = si.row_begin + (frame - si.shard_begin);
        const float acc = __uint_as_float((uint32_t)(v >> 32));
        ol_candidate o;
        o.subspace = i; o.frame = frame; o.bundle = q / a.M; o.query_frame = q % a.M;
        o.dist2 = acc; o.dist = __fsqrt_rn(acc);
        const bool ok = OL_DCHECK(frame >= si.shard_begin && frame - si.shard_begin < si.count);
        o.x = ok ? a.coords[2 * row] : 0; o.y = ok ? a.coords[2 * row + 1] : 0;
        co[r] = o;
    }
    const long long p2 = clock64();
    if (a.prof && threadIdx.x == 0) { atomicAdd(&a.prof[7], (unsigned long long)(p2 - pd));
                                      atomicAdd(&a.prof[0], (unsigned long long)(p1 - p0));
                                      atomicAdd(&a.prof[1], (unsigned long long)(p2 - p1)); }
    if (!a.aggregate) return;
    const uint32_t b = q / a.M;
    if (a.M * a.n_sub > 1) {
        // Algorithm 2 once the bundle's last job has written its rows
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t done = atomicAdd(&a.bundle_count[b], 1u) + 1;
            is_last = done == a.M * a.n_sub;
            if (is_last) a.bundle_count[b] = 0;   // (ready for the next query)
        }
        __syncthreads();
        if (!is_last) return;
        __threadfence();
    } else {
        __syncthreads();   // (the bundle is this job: its rows were written by this CTA)
    }
    const long long p3 = clock64();
    aggregate_block(a.agg, b, smem);
    if (a.prof && threadIdx.x == 0) { atomicAdd(&a.prof[2], (unsigned long long)(p3 - p2));
                                      atomicAdd(&a.prof[3], (unsigned long long)(clock64() - p3)); }
}

// CTAs per job (the cluster size): a power of two <= 8, shares of >= ~256 rows, and no more
// CTAs in all than two per SM
uint32_t micro_split(uint64_t max_rows, uint64_t jobs) {
    const uint64_t want = (max_rows + 255) / 256, by_sm = 296 / (jobs ? jobs : 1);
    uint32_t g = 1;
    while (g < 8 && 2 * g <= want && 2 * g <= by_sm) g *= 2;
    return g;
}

size_t micro_smem_bytes(uint64_t max_rows, uint32_t split, uint32_t N, uint32_t agg_cap) {   // (split x N <= 1,024)
    const uint64_t share = (max_rows + split - 1) / split, merge = split > 1 ? (uint64_t)split * N : 0;
    const size_t rows = sizeof(u64) * (share > merge ? share : merge);
    const size_t agg = agg_cap ? sizeof(u64) * agg_cap * 2 + sizeof(uint32_t) * agg_cap : 0;
    return rows > agg ? rows : agg;
}

cudaError_t launch_micro(const MicroArgs &a, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(micro_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.nq * a.n_sub * a.split);
    cfg.blockDim = dim3(kAggThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = a.split; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, micro_kernel, a);
}

cudaError_t launch_aggregate(const AggArgs &a, cudaStream_t s) {
    // sized to the largest bundle: small bundles fit several CTAs per SM
    const size_t cap = a.cap ? a.cap : (size_t)kAggMax;
    const size_t smem = sizeof(u64) * cap * 2 + sizeof(uint32_t) * cap;
    const size_t max_smem = sizeof(u64) * kAggMax * 2 + sizeof(uint32_t) * kAggMax;
    cudaFuncSetAttribute(aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem);
    aggregate_kernel<<<a.n_bundles, kAggThreads, smem, s>>>(a);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_aggregate)

}  // namespace ol
