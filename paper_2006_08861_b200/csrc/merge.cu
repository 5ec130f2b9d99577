// merge.cu -- the top-N merges (NK4) and candidate assembly.
//
//  merge_chunks: the N smallest keys of every (query frame, subspace) over the
//    per-work-item lists the scan wrote; attaches the geo-referenced tile of
//    each winner ("mapped to their actual floor plan 2D coordinates by
//    checking the geo-referenced mapping table") -> this rank's payload.
//  merge_ranks: the N smallest of the W gathered payloads (cross-GPU merge).
//  candidates: records -> ol_candidate rows in (bundle, frame, subspace, rank)
//    order, dist = RN32(sqrt(acc)) (R3).  At world 1 merge_chunks writes
//    these rows itself (one launch fewer); candidates_kernel serves the W > 1 merge.
// Keys (acc bits << 32 | frame) are unique within a subspace apart from the
// all-ones pad, so "N rounds of extract-the-minimum" is the exact top-N.
#define OL_TU 2
#include "ol_internal.h"

namespace ol {

// record -> candidate row (R3: dist = RN32(sqrt(acc)))
__device__ __forceinline__ ol_candidate make_candidate(const uint4 rec, uint32_t i, uint32_t q, uint32_t M) {
    const float acc = __uint_as_float(rec.x);
    ol_candidate o;
    o.subspace = i;
    o.frame = rec.y;
    o.bundle = q / M;
    o.query_frame = q % M;
    o.dist2 = acc;
    o.dist = __fsqrt_rn(acc);
    o.x = (int32_t)rec.z;
    o.y = (int32_t)rec.w;
    return o;
}

__device__ __forceinline__ u64 warp_min_u64(u64 v) {
    for (int o = 16; o; o >>= 1) {
        u64 w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

constexpr int kMergeThreads = 256;     // (at most; fewer for subspaces of few work items)
constexpr uint32_t kMergeBuf = 2048;   // keys <= T gathered in shared memory (at most)

// the smallest value over the CTA (every thread passes v; all get the result)
__device__ __forceinline__ u64 block_min_u64(u64 v, u64 *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_min_u64(v);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    u64 m = kPadKey;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = red[w] < m ? red[w] : m;
    __syncthreads();
    return m;
}

// One CTA per (query, subspace): the N smallest keys over the subspace's work-item lists.
// Every list is ascending (the scans write sorted lists, pads last), so the global N-th best
// is <= T = min over lists of list[N-1] (that list holds N keys <= T).  Pass 1 computes T
// (one load per list), pass 2 gathers every key <= T -- a prefix of each list, usually
// empty -- into shared memory, and the N smallest of those are the answer.  (Round 1 ran N
// passes over all lists with one warp: 0.2-0.4 ms for small batches, where a frame's
// subspace has thousands of items.)  More than kMergeBuf keys <= T: N rounds of a CTA-wide
// "minimum above the last" over all keys instead.  Keys are unique apart from the all-ones
// pad, so either way the result is the exact top-N.  The buffer holds a.buf_cap keys (<=
// kMergeBuf; = lists x N when that is smaller, so the fallback never runs then) and the CTA
// is one warp when a subspace has at most 8 lists (C2: thousands of tiny jobs).
__global__ void __launch_bounds__(kMergeThreads) merge_chunks_kernel(MergeArgs a) {
    extern __shared__ __align__(16) unsigned char msm[];
    u64 *buf = reinterpret_cast<u64 *>(msm);                  // [buf_cap]
    u64 *sel = buf + a.buf_cap;                               // [N]
    u64 *scratch = sel + a.N;                                 // [blockDim]
    u64 *red = scratch + blockDim.x;                          // [blockDim / 32]
    __shared__ uint32_t nbuf;
    const uint32_t job = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t q = job / a.n_sub, i = job % a.n_sub;
    const SubInfo si = a.subs[i];
    // the subspace's work items exist; its candidate rows fit the candidate array
    if (!OL_DCHECK(si.chunk_begin <= si.chunk_end && si.chunk_end <= a.n_items &&
                   (!a.cand || (uint64_t)(q + 1) * a.sub_prefix[a.n_sub] <= a.n_cand)))
        return;   // (uniform over the CTA)
    const uint32_t N = a.N, nl = si.chunk_end - si.chunk_begin;
    const u64 *src = a.partial + ((size_t)q * a.n_items + si.chunk_begin) * N;
    if (threadIdx.x == 0) nbuf = 0;
    u64 t = kPadKey;
    for (uint32_t j = threadIdx.x; j < nl; j += blockDim.x) {
        const u64 v = src[(size_t)j * N + N - 1];
        t = v < t ? v : t;
    }
    const u64 T = block_min_u64(t, red);   // (its barriers also publish nbuf = 0)
    for (uint32_t j = threadIdx.x; j < nl; j += blockDim.x) {
        const u64 *L = src + (size_t)j * N;
        for (uint32_t r = 0; r < N; ++r) {
            const u64 v = L[r];
            if (v > T || v == kPadKey) break;
            (void)OL_DCHECK(r == 0 || L[r - 1] < v);   // (the lists are ascending)
            const uint32_t pos = atomicAdd(&nbuf, 1u);
            if (pos < a.buf_cap) buf[pos] = v;
        }
    }
    __syncthreads();
    const uint32_t nb = nbuf;
    if (nb <= a.buf_cap && !a.force_scan) {
        if (N <= 32) block_select32(buf, nb, N, sel, scratch);
        else if (warp == 0) {
            u64 lo = 0;
            for (uint32_t r = 0; r < N; ++r) {
                u64 best = kPadKey;
                for (uint32_t k = lane; k < nb; k += 32) {
                    const u64 v = buf[k];
                    if ((r == 0 || v > lo) && v < best) best = v;
                }
                best = warp_min_u64(best);
                lo = best;
                if (lane == 0) sel[r] = best;
            }
        }
    } else {
        const uint32_t nk = nl * N;
        u64 lo = 0;
        for (uint32_t r = 0; r < N; ++r) {
            u64 best = kPadKey;
            for (uint32_t k = threadIdx.x; k < nk; k += blockDim.x) {
                const u64 v = src[k];
                if ((r == 0 || v > lo) && v < best) best = v;
            }
            best = block_min_u64(best, red);
            lo = best;
            if (threadIdx.x == 0) sel[r] = best;
        }
    }
    __syncthreads();
    // records (and at world 1 the candidate rows: rank r < c of this (frame, subspace))
    uint4 *dst = a.records + ((size_t)q * a.n_sub + i) * N;
    const uint32_t c = a.cand ? a.sub_prefix[i + 1] - a.sub_prefix[i] : 0;
    ol_candidate *co = a.cand ? a.cand + (uint64_t)q * a.sub_prefix[a.n_sub] + a.sub_prefix[i] : nullptr;
    for (uint32_t r = threadIdx.x; r < N; r += blockDim.x) {
        const u64 best = sel[r];
        uint4 rec;
        if (best == kPadKey) {
            rec = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u);
        } else {
            const uint32_t frame = (uint32_t)best;
            const uint64_t row = si.row_begin + (frame - si.shard_begin);
            // a winner is a row of this rank's slice of this subspace
            const bool ok = OL_DCHECK(frame >= si.shard_begin && frame - si.shard_begin < si.count);
            rec = make_uint4((uint32_t)(best >> 32), frame, ok ? (uint32_t)a.coords[2 * row] : 0u,
                             ok ? (uint32_t)a.coords[2 * row + 1] : 0u);
        }
        dst[r] = rec;
        if (r < c) co[r] = make_candidate(rec, i, q, a.M);
    }
}

cudaError_t launch_merge_chunks(const MergeArgs &a_in, cudaStream_t s) {
    MergeArgs a = a_in;
    const uint64_t keys = (uint64_t)a.max_lists * a.N;
    a.buf_cap = a.force_scan ? 0u : (uint32_t)(keys < kMergeBuf ? (keys ? keys : 1) : kMergeBuf);
    const uint32_t threads = a.max_lists <= 8 ? 32u : a.max_lists <= 64 ? 128u : (uint32_t)kMergeThreads;
    const size_t smem = sizeof(u64) * ((size_t)a.buf_cap + a.N + threads + threads / 32);
    merge_chunks_kernel<<<(unsigned)((uint64_t)a.nq * a.n_sub), threads, smem, s>>>(a);
    return cudaGetLastError();
}

// One warp, one (query, subspace) gw: the N smallest of world sorted lists gathered
// back to back ([world][nq][n_sub][N] records).
__device__ void merge_rank_lists(RankMergeArgs a, uint32_t gw, int lane) {
    const size_t per_rank = (size_t)a.nq * a.n_sub * a.N;
    const size_t base = (size_t)gw * a.N;
    const uint32_t nk = a.world * a.N;
    u64 last = 0;
    bool have_last = false;
    for (uint32_t r = 0; r < a.N; ++r) {
        u64 best = kPadKey;
        uint32_t bt = 0xFFFFFFFFu;
        for (uint32_t t = lane; t < nk; t += 32) {
            const uint4 rec = __ldcg(&a.gathered[(t / a.N) * per_rank + base + (t % a.N)]);   // (L2: peers write it)
            const u64 v = ((u64)rec.x << 32) | rec.y;
            if ((!have_last || v > last) && v < best) { best = v; bt = t; }
        }
        const u64 wbest = warp_min_u64(best);
        // the lane that holds the winner writes it (carries x, y)
        const unsigned owner = __ballot_sync(0xffffffffu, best == wbest && bt != 0xFFFFFFFFu);
        if (wbest == kPadKey) {
            for (uint32_t rr = r + lane; rr < a.N; rr += 32)
                a.records[base + rr] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0u, 0u);
            break;
        }
        if (lane == __ffs(owner) - 1)
            a.records[base + r] = __ldcg(&a.gathered[(bt / a.N) * per_rank + base + (bt % a.N)]);
        last = wbest;
        have_last = true;
    }
}

__global__ void __launch_bounds__(kMergeThreads) merge_ranks_kernel(RankMergeArgs a) {
    const uint32_t gw = (blockIdx.x * kMergeThreads + threadIdx.x) / 32;
    if (gw >= a.nq * a.n_sub) return;
    merge_rank_lists(a, gw, threadIdx.x & 31);
}

// ---------------------------------------------------------------- peer-memory exchange
// The cross-GPU step as ONE kernel over NVLink/NVSwitch peer memory (§8e: all-gather of
// the per-rank top-N, then the N smallest of W·N): every block of rank r stores its
// slice of r's payload into slot r of every rank's mailbox (plain st.global to peer
// addresses opened by CUDA IPC), fences system-wide and adds 1 to the receiver's
// counter flag[r]; then waits until its own mailbox holds every rank's slices
// (flag[s] = epoch x blocks for all s, acquire loads) and merges its share of the
// (frame, subspace) lists straight out of the mailbox.  Mailbox data is double-
// buffered by epoch parity: a rank can only push epoch e + 1 after every rank has
// pushed e, i.e. after every rank finished merging e - 1.  Blocks wait on blocks of
// their own grid, so the launch is cooperative (co-resident).  Groups: with G > 1
// the grid emulates G ranks on one GPU (tests), group g acting as rank rank0 + g.
__global__ void __launch_bounds__(kMergeThreads) xchg_merge_kernel(XchgArgs a) {
    const uint32_t g = blockIdx.x / a.blocks, b = blockIdx.x % a.blocks;
    const uint32_t r = a.rank0 + g;
    const size_t P = (size_t)a.nq * a.n_sub * a.N;            // records per rank
    const size_t lo = P * b / a.blocks, hi = P * (b + 1) / a.blocks;
    const uint32_t par = a.epoch & 1u;
    const uint4 *src = a.payload[g];
    for (uint32_t p = 0; p < a.world; ++p) {
        uint4 *dst = a.mbox[p] + ((size_t)par * a.world + r) * P;
        for (size_t t = lo + threadIdx.x; t < hi; t += blockDim.x) dst[t] = src[t];
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x < a.world) {
        unsigned int *f = a.flag[threadIdx.x] + r;
        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(f) : "memory");
    }
    const unsigned int target = a.epoch * a.blocks;
    if (threadIdx.x < a.world) {
        const unsigned int *f = a.flag[r] + threadIdx.x;
        unsigned int v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
            if ((int)(v - target) >= 0) break;
            __nanosleep(64);
        }
    }
    __syncthreads();
    RankMergeArgs m;
    m.gathered = a.mbox[r] + (size_t)par * a.world * P;
    m.records = a.records[g];
    m.nq = a.nq; m.n_sub = a.n_sub; m.N = a.N; m.world = a.world;
    const uint32_t warps = a.blocks * (kMergeThreads / 32);
    for (uint32_t gw = b * (kMergeThreads / 32) + threadIdx.x / 32; gw < a.nq * a.n_sub; gw += warps)
        merge_rank_lists(m, gw, threadIdx.x & 31);
}

cudaError_t launch_xchg_merge(const XchgArgs &a, uint32_t groups, cudaStream_t s) {
    XchgArgs x = a;
    void *args[] = {&x};
    return cudaLaunchCooperativeKernel((const void *)xchg_merge_kernel, dim3(groups * a.blocks), dim3(kMergeThreads),
                                       args, 0, s);
}

cudaError_t launch_merge_ranks(const RankMergeArgs &a, cudaStream_t s) {
    uint64_t warps = (uint64_t)a.nq * a.n_sub;
    uint64_t blocks = (warps * 32 + kMergeThreads - 1) / kMergeThreads;
    merge_ranks_kernel<<<(unsigned)blocks, kMergeThreads, 0, s>>>(a);
    return cudaGetLastError();
}

__global__ void candidates_kernel(CandArgs a) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t total = (uint64_t)a.nq * a.n_sub * a.N;
    if (t >= total) return;
    const uint32_t r = (uint32_t)(t % a.N);
    const uint32_t i = (uint32_t)((t / a.N) % a.n_sub);
    const uint32_t q = (uint32_t)(t / ((uint64_t)a.N * a.n_sub));
    const uint32_t c = a.sub_prefix[i + 1] - a.sub_prefix[i];
    if (r >= c) return;
    if (OL_DCHECK((uint64_t)q * a.sub_prefix[a.n_sub] + a.sub_prefix[i] + r < a.n_cand))
        a.out[(uint64_t)q * a.sub_prefix[a.n_sub] + a.sub_prefix[i] + r] = make_candidate(a.records[t], i, q, a.M);
}

cudaError_t launch_candidates(const CandArgs &a, cudaStream_t s) {
    uint64_t total = (uint64_t)a.nq * a.n_sub * a.N;
    candidates_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_merge)

}  // namespace ol
