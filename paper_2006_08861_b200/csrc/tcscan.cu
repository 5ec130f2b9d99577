// tcscan.cu -- tensor-core certified filter for the scan (NEXT-2 in SURVEY §8f,
// kernel NK8), used when a tile holds many query frames.
//
// The exact answer is still the fp32 chain of R3 (P:157 calculateDistance,
// P:202 "smallest Euclidean distance"); tensor cores only decide which pairs
// cannot possibly be in the top-N.  For fp32 vectors q, f with real squared
// distance A = ||q||^2 + ||f||^2 - 2 q.f and their fp16 roundings q^, f^:
//   q.f = q^.f^ + (q - q^).f + q^.(f - f^) <= q^.f^ + e_q Nf + Nq e_f,
// e = RU||x - x^||, Nq >= ||q^||, Nf >= ||f|| (batch / database maxima).  The tensor
// core computes P = q^.f^ (64 exact fp16 products, fp32 accumulation: error
// <= 2^-14 sum|products| <= 2^-14 Nq Nf).  With g_r = RD||f||^2 / 2 - Nq e_f,
//   A >= alpha_q + 2 g_r - 2 P - 2^-13 Nq Nf,   alpha_q = RD||q||^2 - 2 e_q Nf.
// The fp32 chain satisfies acc >= A (1 - 66 u) >= A / (1 + 2^-17).  Hence
//   acc > tau_q  is guaranteed when  P - g_r < h_q = (alpha'_q - tau_q (1 + 2^-17)) / 2,
//   alpha'_q = alpha_q - 2^-13 Nq Nf - sigma,  sigma = 2^-18 (Nq + Nf)^2
// (sigma absorbs the fp32 roundings of computing h).  For a 32-row block B with
// g_B <= min_{r in B} g_r (rounded down from per-block minima of RD||f||^2 / 2 and
// maxima of e_f), P < thr = RD(h_q + g_B) implies P - g_r < h_q for every row of
// the block, so the epilogue tests max_{r in B} P >= thr: FMNMX3 only.  Pairs of a
// passing block that pass the per-element test ("survivors", ~1e-5 of pairs on
// paper-shaped data) are re-scored with the exact fp32 chain on CUDA cores and
// enter the top-N; everything else is provably outside it, so results are
// bit-identical to the one-pass scan (tests: test_gpu_tc, test_gpu_parity,
// test_gpu_fullsize).
//
// Prefix filter (a.kf < 64): every quantity above taken over the first kf coordinates
// only bounds the prefix distance, itself <= A, so pruning stays exact;
// kf = 32 halves the MMA work, and the fp16 plane then holds just those 32 columns
// (a.pw = 32: 64-B rows, 64-byte swizzle).
//
// CTA = one work item (rows of one subspace) x <= 128 query frames (one M-tile); CTA
// pairs (kPair, cluster of 2) share each row tile: M = 256 frames, each CTA loads half.
// Warp roles: 0 TMA producer (256-row tiles of fp16 rows, 128-B or 64-B swizzle, a
// mbarrier ring of n_stages); 1 TMEM allocator + single-thread tcgen05.mma issuer (the
// pair's leader): per tile, M = 128 / 256 frames x N = 256 rows x K = kf (kf / 16 K16
// MMAs) into a double-buffered fp32 TMEM accumulator (2 x 256 columns); 2..17 epilogue
// in two groups of 8 warps on alternate tiles (thread = one frame x 128 of the tile's
// rows: tcgen05.ld, release the buffer, per-block max, survivor events); 18..19 exact
// re-scoring + top-N insertion.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#define OL_TU 4
#include "ol_internal.h"
#include "tc_ptx.cuh"

namespace ol {

using namespace tc;

constexpr int kTileRows = 256;          // MMA N (rows per tile)
constexpr int kTBufs = 2;               // TMEM accumulator buffers (2 x 256 columns)
constexpr int kQB = 128;                // frames per CTA: one M-tile
constexpr int kMaxStages = 8;
constexpr int kEpiWarps = 16;           // two groups of 8 (alternate tiles)
constexpr int kExactWarps = 2;
constexpr int kTcThreads = 32 * (2 + kEpiWarps + kExactWarps);
constexpr int kEv = 8;                  // survivor event ring entries per exact warp: a short ring
                                        // back-pressures the epilogue so thresholds stay fresh
                                        // (measured with the 32-dim filter, 1,024 frames, ring
                                        // 32 / 16 / 8 / 4: 100M rows 10.05 / 9.93 / 9.95 / 9.96 ms,
                                        // 20M 2.82 / 2.70 / 2.66 / 2.67, 1M 0.68 / - / 0.58 / 0.57)
constexpr int kTrackMax = 16;           // largest N of the bound pre-pass (register list)
constexpr int kBndRing = 16;            // >= kMaxStages + kTBufs: see TcSmem::bnd
constexpr uint32_t kTlTiles = 120;      // profiling timeline (tc_debug 32 | 2048): tiles of CTA 0 recorded
constexpr float kTauInflate = 1.0f + 1.0f / 131072.0f;   // 1 + 2^-17

struct TcSmem {
    alignas(1024) __half qm[kQB * kK];      // frames, main K (SW128), resident
    uint64_t full[kMaxStages], empty[kMaxStages], tfull[kTBufs], tempty[kTBufs], qbar;
    // the row-term bounds of tile t's 8 32-row blocks, in slot t % kBndRing, brought
    // by the producer's bulk copy next to the rows (subspaces start on 256-row tiles, so a
    // tile's 64 bytes of bounds are 64-byte aligned): the epilogue reads them from shared
    // memory -- a global load in its per-tile path stalls the tcgen05.wait::ld after it.  The
    // producer runs at most n_stages tiles ahead of the MMA and the MMA at most kTBufs ahead
    // of the epilogue, so a slot is never rewritten while it is read.
    alignas(16) float2 bnd[kBndRing][kTileRows / 32];
    long long tma_t0[kMaxStages];   // profiling (prof): when the stage's TMA was issued
    uint64_t bfull[kBndRing];
    uint32_t tmem_base;
    float alpha[kQB];
    uint32_t tau[kQB];
    int lock[kQB];
    // survivor events, one MPSC ring per exact warp (frames ql % kExactWarps == w):
    // event = (first row of a 128-row block << 8 | ql, 4 x 32-row pass masks); slot i
    // is free for position p when seq == p, filled when seq == p + 1 (Vyukov)
    uint4 ev_mask[kExactWarps][kEv];
    uint32_t ev_head[kExactWarps][kEv];
    uint32_t seq[kExactWarps][kEv];
    unsigned int prod[kExactWarps], closed_at[kExactWarps];
    int closed;
    // dynamic, 1024-aligned: n_stages x rows [256][pw] fp16 (SW128 / SW64), then the
    // top-N lists u64 [qb][N]
};

static __host__ __device__ constexpr size_t tc_fixed_bytes() { return (sizeof(TcSmem) + 1023) / 1024 * 1024; }

size_t tc_smem_bytes(uint32_t qb, uint32_t N, uint32_t stages, uint32_t pw) {
    return 1024 + tc_fixed_bytes() + (size_t)stages * (kTileRows * pw * 2) + sizeof(u64) * qb * N;
}

__device__ __forceinline__ float chain_step_tc(float acc, float q, float f) {
    float d = __fsub_rn(q, f);
    return __fmaf_rn(d, d, acc);
}

__device__ __forceinline__ uint32_t lds_u32(const void *p) {
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
__device__ __forceinline__ uint64_t lds_u64(const void *p) {
    return *reinterpret_cast<const volatile uint64_t *>(p);
}
__device__ __forceinline__ void sts_u32(void *p, uint32_t v) { *reinterpret_cast<volatile uint32_t *>(p) = v; }

__device__ __forceinline__ float max3f(float a, float b, float c) {  // FMNMX3
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Publish one survivor event (the passing rows of one frame's 128-row block) on
// the ring of the exact warp that owns the frame, waiting while it is full.
__device__ __noinline__ void tc_enqueue_event(TcSmem &s, uint32_t mk0, uint32_t mk1, uint32_t mk2, uint32_t mk3,
                                              uint32_t rb, uint32_t ql, unsigned long long *prof) {
    const uint32_t w = ql % kExactWarps;
    const unsigned pos = atomicAdd(&s.prod[w], 1u);
    uint32_t *sq = &s.seq[w][pos % kEv];
    if (lds_u32(sq) != pos) {
        const long long r0 = clock64();
        while (lds_u32(sq) != pos) __nanosleep(64);
        if (prof) atomicAdd(&prof[10], (unsigned long long)(clock64() - r0));
    }
    s.ev_mask[w][pos % kEv] = make_uint4(mk0, mk1, mk2, mk3);
    s.ev_head[w][pos % kEv] = (rb << 8) | ql;
    __threadfence_block();
    sts_u32(sq, pos + 1);
}

// Merge one key per lane (kPadKey = none) into the ascending list L[0..N) held in
// shared memory, keeping the N smallest.  List element a goes to a + #(keys < L[a]);
// key j to #(L < key_j) + #(keys < key_j).  Ranks of distinct keys are distinct, so
// the scatter writes each slot < N exactly once.
__device__ __noinline__ void tc_warp_merge(u64 *L, uint32_t N, u64 key, int lane) {
    constexpr int kPer = (OL_MAX_N + 31) / 32;
    u64 lv[kPer];
    uint32_t rk[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const uint32_t a = lane + 32 * i;
        lv[i] = a < N ? L[a] : kPadKey;
        rk[i] = a;
    }
    // my key's rank among the list: lower bound by binary search
    uint32_t lo = 0, hi = N;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (L[mid] < key) lo = mid + 1; else hi = mid;
    }
    uint32_t kr = lo;
    for (int j = 0; j < 32; ++j) {
        const u64 kj = __shfl_sync(0xffffffffu, key, j);
        kr += kj < key;
#pragma unroll
        for (int i = 0; i < kPer; ++i) rk[i] += kj < lv[i];
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kPer; ++i)
        if (lane + 32 * i < N && rk[i] < N) L[rk[i]] = lv[i];
    if (key != kPadKey && kr < N) L[kr] = key;
    __syncwarp();
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Inline exact re-scoring (a.inline_rescore, short work items): one epilogue warp re-scores
// its own survivors.  Lane l contributes the passing rows of its frame (masks mk0..3 over the
// warp's 128 rows from rb); the warp re-scores them 32 at a time, one lane per (frame, row),
// with the exact fp32 chain (R3; the second half of a row only while the chain is within the
// frame's threshold), merges each frame's keys into its list under the frame's lock (the 4
// epilogue warps of a frame share its list) and publishes the tightened threshold.  With
// short items (C2: 16 tiles per CTA, 3 % of pairs surviving) the two exact warps were the
// bottleneck; on long items the round trips on the epilogue's path cost more than they save.
__device__ __noinline__ void tc_rescore_warp(const TcScanArgs &a, TcSmem &s, u64 *lists, const WorkItem &it,
                                             uint32_t q0, uint32_t qbase, uint32_t mk0, uint32_t mk1, uint32_t mk2,
                                             uint32_t mk3, uint32_t rb) {
    constexpr uint32_t kAll = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const uint32_t N = a.N;
    const uint32_t cnt = __popc(mk0) + __popc(mk1) + __popc(mk2) + __popc(mk3);
    uint32_t incl = cnt;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kAll, incl, o);
        if (lane >= o) incl += v;
    }
    const uint32_t total = __shfl_sync(kAll, incl, 31);
    for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t sidx = base + lane;
        uint32_t e = 0;   // owner lane: the first with incl > sidx
        for (int j = 0; j < 32; ++j) e += __shfl_sync(kAll, incl, j) <= sidx;
        const uint32_t es = min(e, 31u);
        const uint32_t e_incl = __shfl_sync(kAll, incl, es), e_cnt = __shfl_sync(kAll, cnt, es);
        const uint32_t w0 = __shfl_sync(kAll, mk0, es), w1 = __shfl_sync(kAll, mk1, es);
        const uint32_t w2 = __shfl_sync(kAll, mk2, es), w3 = __shfl_sync(kAll, mk3, es);
        const uint32_t col = qbase + es;   // frame within the CTA
        u64 key = kPadKey;
        if (sidx < total) {
            uint32_t k = sidx - (e_incl - e_cnt), wsel = 0, w = w0;
            if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w1; wsel = 1;
                if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w2; wsel = 2;
                    if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w3; wsel = 3; } } }
            const uint32_t bit = __fns(w, 0, (int)k + 1);
            const uint32_t rl = rb + 32 * wsel + bit;
            const uint64_t row = it.row_begin + rl;
            if (OL_DCHECK(rl < it.count && col < kQB && q0 + col < a.nq)) {
                const float4 *qv = reinterpret_cast<const float4 *>(a.queries + (size_t)(q0 + col) * kK);
                const float tcur = __uint_as_float(lds_u32(&s.tau[col]));
                float acc = 0.f;
                float4 f[kK / 8];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (h == 1 && acc > tcur) break;
#pragma unroll
                    for (int kk = 0; kk < kK / 8; ++kk)
                        f[kk] = __ldg(reinterpret_cast<const float4 *>(a.fine + fine_off(row, 4 * (h * (kK / 8) + kk))));
#pragma unroll
                    for (int kk = 0; kk < kK / 8; ++kk) {
                        const float4 x = __ldg(qv + h * (kK / 8) + kk);
                        acc = chain_step_tc(acc, x.x, f[kk].x); acc = chain_step_tc(acc, x.y, f[kk].y);
                        acc = chain_step_tc(acc, x.z, f[kk].z); acc = chain_step_tc(acc, x.w, f[kk].w);
                    }
                }
                key = ((u64)__float_as_uint(acc) << 32) | (u64)(it.frame_begin + rl);
                if (acc > tcur || !(key < lists[(size_t)col * N + N - 1])) key = kPadKey;   // cannot enter the top-N
            }
        }
        // (bit e: some lane holds a key of owner e's frame) one warp-wide merge per frame, locked
        const uint32_t frames = __reduce_or_sync(kAll, key != kPadKey ? (1u << es) : 0u);
        for (uint32_t fb = frames; fb; fb &= fb - 1) {
            const uint32_t eo = (uint32_t)(__ffs(fb) - 1), f = qbase + eo;
            if (lane == 0) {
                while (atomicCAS(&s.lock[f], 0, 1) != 0) __nanosleep(32);
                __threadfence_block();
            }
            __syncwarp();
            u64 *L = lists + (size_t)f * N;
            tc_warp_merge(L, N, es == eo ? key : kPadKey, lane);
            if (lane == 0) {
                const u64 last = L[N - 1];
                __threadfence_block();
                atomicExch(&s.lock[f], 0);
                if (last != kPadKey) {   // publish this frame's tightened threshold
                    const uint32_t tb = (uint32_t)(last >> 32);
                    atomicMin(&s.tau[f], tb);
                    const size_t ti = (size_t)(q0 + f) * a.n_sub + it.sub;
                    atomicMin(&a.g_tau[ti], tb);
                    for (uint32_t pr = 0; pr < a.n_peer; ++pr) atomicMin(&a.peer_tau[pr][ti], tb);   // (RED over NVLink)
                }
            }
            __syncwarp();
        }
    }
    if (lane == 0 && a.stat_survivors) atomicAdd(a.stat_survivors, (unsigned long long)total);
}


// max over 32 accumulator columns into two running maxima
__device__ __forceinline__ void max32(const uint32_t (&v)[32], float &m0, float &m1) {
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        m0 = max3f(m0, __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
        m1 = max3f(m1, __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
    }
}
// bit mask of the columns >= h, invalid columns (>= nvalid) excluded
__device__ __forceinline__ uint32_t mask32(const uint32_t (&v)[32], float h, int base, uint32_t nvalid) {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) m |= (uint32_t)(__uint_as_float(v[j]) >= h && (uint32_t)(base + j) < nvalid) << j;
    return m;
}

template <bool kProf, bool kBound, bool kPair, bool kInline = false>
__global__ void __launch_bounds__(kTcThreads, 1)
tcscan_kernel(const __grid_constant__ CUtensorMap map_rows, const __grid_constant__ CUtensorMap map_q, TcScanArgs a) {
    extern __shared__ __align__(1024) unsigned char raw[];
    // (offsetting raw keeps the shared address space visible to the compiler: LDS/STS)
    unsigned char *base = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
    TcSmem &s = *reinterpret_cast<TcSmem *>(base);
    unsigned char *stage0 = base + tc_fixed_bytes();
    const uint32_t n_stages = a.stages;
    const uint32_t stage_bytes = kTileRows * a.pw * 2;
    u64 *lists = reinterpret_cast<u64 *>(stage0 + (size_t)n_stages * stage_bytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t item_id = blockIdx.x / a.n_qblocks;
    const uint32_t qblk = blockIdx.x % a.n_qblocks;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qblk * a.qb;
    const uint32_t qn = q0 < a.nq ? min(a.qb, a.nq - q0) : 0u;   // 0: a pair's padding CTA
    // CTA pairs (kPair): the two query blocks of a cluster share every row tile; rank 0
    // issues M = 256 MMAs over both CTAs' frames, each CTA loads half of each row tile
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;
    const uint32_t N = a.N;
    const uint32_t n_tiles = (it.count + kTileRows - 1) / kTileRows;
    constexpr bool prof = kProf;
    // a work item's rows lie inside the planes (the pre-pass: inside its strided view), its
    // subspace and query block exist, the lists fit the frames
    if (!OL_DCHECK(item_id < a.n_items && qblk < a.n_qblocks && it.sub < a.n_sub && a.qb <= (uint32_t)kQB &&
                   (kBound || it.row_begin + it.count <= (uint64_t)a.n_blk * 32)))
        return;   // (uniform over the CTA / cluster: before any barrier)   // profiling counters (tc_debug & 32): a separate instantiation
    const long long t_start = clock64();

    // ---------------------------------------------------------------- setup
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < n_stages; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        for (int i = 0; i < kTBufs; ++i) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], (kPair ? 2 : 1) * kEpiWarps / 2); }
        for (int i = 0; i < kBndRing; ++i) mbar_init(&s.bfull[i], 1);
        mbar_init(&s.qbar, 1);
        fence_mbar_init();
        for (int w = 0; w < kExactWarps; ++w) s.prod[w] = s.closed_at[w] = 0;
        s.closed = 0;
        tma_prefetch(&map_rows);
    }
    if (warp == 1) { if (kPair) tmem_alloc2<512>(&s.tmem_base); else tmem_alloc<512>(&s.tmem_base); }
    const float nqm = __uint_as_float(a.bounds[2]), nfm = a.nf_max;
    // a frame outside the fp16 range, or an unbounded batch: every pair is re-scored
    const bool force_all = a.bounds[3] != 0 || !(nqm < 300.f);
    const float sigma = 3.814697265625e-06f * (nqm + nfm) * (nqm + nfm);      // 2^-18 (Nq + Nf)^2
    const float c0 = 1.220703125e-04f * nqm * nfm;                            // 2^-13 Nq Nf
    for (uint32_t q = threadIdx.x; q < kQB; q += blockDim.x) {
        if (q < qn) {
            const float4 m = a.qmeta[q0 + q];  // (RD ||q||^2, RU e_q, RU ||q||^2)
            s.alpha[q] = force_all ? -INFINITY : m.x - 2.f * m.y * nfm - c0 - sigma;
            s.tau[q] = a.g_tau[(size_t)(q0 + q) * a.n_sub + it.sub];
        } else {
            s.alpha[q] = INFINITY;  // padded frame: h = +inf, never passes
            s.tau[q] = 0;
        }
        s.lock[q] = 0;
    }
    for (uint32_t i = threadIdx.x; i < kExactWarps * kEv; i += blockDim.x) s.seq[i / kEv][i % kEv] = i % kEv;
    for (uint32_t i = threadIdx.x; i < a.qb * N; i += blockDim.x) lists[i] = kPadKey;
    tc_fence_before();
    if (kPair) cluster_sync(); else __syncthreads();   // (pair: the leader's barriers exist before any remote use)
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            if (kPair) {
                // each CTA loads its own frames and its half of each row tile; the bytes of
                // both complete on the leader's barriers
                if (rank == 0) mbar_expect_tx(&s.qbar, 2 * a.qb * a.pw * (uint32_t)sizeof(__half));
                tma_load_2d_pair(s.qm, &map_q, &s.qbar, 0, (int)q0);
            } else {
                mbar_expect_tx(&s.qbar, a.qb * a.pw * (uint32_t)sizeof(__half));
                tma_load_2d(s.qm, &map_q, &s.qbar, 0, (int)q0);
            }
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % n_stages;
                if (t >= n_stages) mbar_wait_sleep(&s.empty[st], ((t / n_stages) - 1) & 1);
                unsigned char *sb = stage0 + (size_t)st * stage_bytes;
                const int r0 = (int)(it.row_begin + (uint64_t)t * kTileRows);
                if (!kBound) {   // this tile's block bounds (64 B, aligned: items start on 256-row tiles;
                                 // pairs: each CTA its own copy)
                    const uint32_t sl = t % kBndRing;
                    mbar_expect_tx(&s.bfull[sl], (kTileRows / 32) * sizeof(float2));
                    bulk_load(&s.bnd[sl][0], &a.blk[(size_t)r0 >> 5], (kTileRows / 32) * sizeof(float2), &s.bfull[sl]);
                }
                if (kPair) {
                    if (rank == 0) mbar_expect_tx(&s.full[st], stage_bytes);   // both halves
                    tma_load_2d_pair(sb, &map_rows, &s.full[st], 0, r0 + (int)rank * (kTileRows / 2));
                    continue;
                }
                if ((a.dbg & 128) && t >= n_stages) { mbar_arrive(&s.full[st]); continue; }   // profiling: stale rows
                if (kProf) s.tma_t0[st] = clock64();
                mbar_expect_tx(&s.full[st], stage_bytes);
                tma_load_2d(sb, &map_rows, &s.full[st], 0, r0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // The whole warp runs the loop and the waits (so stage / buffer / descriptor values are
        // warp-uniform and live in uniform registers); one elected lane issues the MMAs and
        // commits.  Round 2: with lane 0 alone in a divergent branch every operand went through
        // R2UR first -- 291 cycles to issue the tile's two MMAs and 149 for its two commits.
        if (rank == 0) {
            // M = 128 frames (pair: 256, both CTAs' frames), N = 256 rows
            const uint32_t idesc = idesc_f16_f32(kPair ? 256 : 128, kTileRows);
            long long pw_full = 0, pw_tempty = 0, pw_issue = 0, pw_lat = 0, pw_commit = 0;   // (profiling: prof[0], [1], [16..18])
            mbar_wait(&s.qbar, 0);
            const uint32_t qm = smem_u32(s.qm);
            const bool leader = elect_one();
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % n_stages, buf = t % kTBufs;
                long long c0 = clock64();
                mbar_wait_sleep(&s.full[st], (t / n_stages) & 1);
                long long c1 = clock64();
                if (t >= kTBufs) mbar_wait_sleep(&s.tempty[buf], ((t / kTBufs) - 1) & 1);
                long long c2 = prof ? clock64() : 0;
                if (prof) { pw_full += c1 - c0; pw_tempty += c2 - c1; pw_lat += c1 - *(volatile long long *)&s.tma_t0[st]; }
                const bool tl = prof && (a.dbg & 2048) && blockIdx.x == 0 && t < kTlTiles && leader;   // (timeline)
                if (tl) a.prof[64 + t * 8 + 0] = (unsigned long long)c2;
                tc_fence_after();
                const uint32_t rm = smem_u32(stage0 + (size_t)st * stage_bytes);
                const uint32_t d = tmem + buf * kTileRows;
                if (!(a.dbg & 2)) {
#pragma unroll
                    for (int k = 0; k < kK / 16; ++k) {
                        if (k * 16 >= (int)a.kf) break;
                        // (K-step k: +32 B along the rows, inside the swizzle atom)
                        const uint64_t da = a.pw == 64 ? desc_sw128_kmajor(qm + k * 32) : desc_sw64_kmajor(qm + k * 32);
                        const uint64_t db = a.pw == 64 ? desc_sw128_kmajor(rm + k * 32) : desc_sw64_kmajor(rm + k * 32);
                        if (leader) {
                            if (kPair) mma_f16_pair(d, da, db, idesc, k > 0 ? 1u : 0u);
                            else mma_f16(d, da, db, idesc, k > 0 ? 1u : 0u);
                        }
                    }
                }
                long long c3 = prof ? clock64() : 0;
                if (leader) {
                    if (kPair) { mma_commit_pair(&s.empty[st], 3); mma_commit_pair(&s.tfull[buf], 3); }
                    else { mma_commit(&s.empty[st]); mma_commit(&s.tfull[buf]); }
                }
                __syncwarp();
                if (prof) { pw_issue += c3 - c2; pw_commit += clock64() - c3; }
                if (tl) a.prof[64 + t * 8 + 1] = (unsigned long long)clock64();
            }
            if (prof && leader) {
                atomicAdd(&a.prof[0], (unsigned long long)pw_full); atomicAdd(&a.prof[1], (unsigned long long)pw_tempty);
                atomicAdd(&a.prof[16], (unsigned long long)pw_issue); atomicAdd(&a.prof[17], (unsigned long long)pw_lat);
                atomicAdd(&a.prof[18], (unsigned long long)pw_commit);
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // ------------------------------------------------------------ epilogue
        // two groups of 8 warps take alternate tiles (group g: tiles g, g + 2, ...), so one
        // group's tcgen05.ld overlaps the other's compares.  Thread = one frame (TMEM lane)
        // x 128 of the tile's 256 rows, read as two 64-column chunks (register budget).
        const int ew = warp - 2;                  // 0..15
        const uint32_t quarter = warp & 3;        // TMEM lanes 32*quarter ..
        const uint32_t half = (ew >> 2) & 1;      // row columns half*128 .. +128
        const uint32_t grp = ew >> 3;             // tile parity
        const uint32_t ql = quarter * 32 + lane;  // frame within the CTA
        const bool refresher = half == 0 && grp == 0 && !(a.dbg & 256);   // one warp per frame refreshes tau (dbg 256: none, profiling)
        const float alpha = s.alpha[ql];
        // lanes 0..3: the row-term bound g_B of this warp's 4 blocks
        auto load_g = [&](uint32_t t) -> float2 {
            if (!kBound) return make_float2(0.f, 0.f);   // (bounds staged in shared memory)
            if (a.dbg & 4096) return make_float2(0.f, 0.f);   // (profiling: no bound loads)
            const uint32_t b = min((uint32_t)((it.row_begin + t * kTileRows + half * 128) >> 5) + (lane & 3), a.n_blk - 1);
            return __ldg(&a.blk[b]);
        };
        uint32_t gt = 0xFFFFFFFFu;                // shared running threshold, loaded at the start of each tile
        long long ew_tfull = 0, ew_ld = 0, ew_math = 0, ew_tile = 0;
        // bound pre-pass (kBound): the thread keeps, in registers, the N largest
        // y = RD(max_S P - G) over disjoint 16-row sets S of its sampled rows (the two running
        // maxima of each 32-row block), G >= RU||f||^2/2 + Nq e_f for every row.  With
        // gamma_q = RU(RU||q||^2 + 2 e_q Nf + 2^-13 Nq Nf):
        //   acc <= A (1 + 2^-17) <= (gamma_q + 2 (G - P)) (1 + 2^-17)
        // for the row attaining each maximum -- N distinct real rows -- so
        // RU((gamma_q - 2 y_N)(1 + 2^-17)) bounds the N-th best acc of the subspace.
        // The list is descending; the first kTrackMax - N slots hold +inf.
        float tl[kBound ? kTrackMax : 1];
        if constexpr (kBound) {
#pragma unroll
            for (int e = 0; e < kTrackMax; ++e) tl[e] = e < kTrackMax - (int)N ? INFINITY : -INFINITY;
        }
        const float Gg = kBound ? __fadd_ru(__uint_as_float(a.bounds[4]), __fmul_ru(nqm, __uint_as_float(a.bounds[5]))) : 0.f;
        auto track = [&](float y) {
            if constexpr (kBound) {
                if (y > tl[kTrackMax - 1]) {
#pragma unroll
                    for (int e = 0; e < kTrackMax; ++e) {
                        const float z = fmaxf(tl[e], y);
                        y = fminf(tl[e], y);
                        tl[e] = z;
                    }
                }
            }
        };
        // (register values loaded from global memory are only read tiles later and never
        // copied in between: a copy would stall on the load)
        auto tile = [&](uint32_t t, const float2 gb) {
            const long long ts = prof ? clock64() : 0;
            const uint32_t buf = t % kTBufs;
            if (refresher && ql < qn) gt = __ldcg(&a.g_tau[(size_t)(q0 + ql) * a.n_sub + it.sub]);
            const long long w0 = prof ? clock64() : 0;
            mbar_wait_sleep(&s.tfull[buf], (t / kTBufs) & 1);
            const long long w1 = prof ? clock64() : 0;
            if (prof && lane == 0) ew_tfull += w1 - w0;
            const bool tl = prof && (a.dbg & 2048) && blockIdx.x == 0 && t < kTlTiles && lane == 0;   // (timeline)
            if (tl) atomicMax(&a.prof[64 + t * 8 + 2], (unsigned long long)w1);
            tc_fence_after();
            if (quarter * 32 >= qn) {   // no frame in this warp's TMEM lanes (few frames, a pair's padding CTA)
                tc_fence_before();
                __syncwarp();
                if (lane == 0) { if (kPair) mbar_arrive_leader(&s.tempty[buf]); else mbar_arrive(&s.tempty[buf]); }
                return;
            }
            const uint32_t taddr = tmem + ((quarter * 32) << 16) + buf * kTileRows + half * 128;
            const float h = 0.5f * (alpha - __uint_as_float(s.tau[ql]) * kTauInflate);
            float th0, th1, th2, th3;
            if (!kBound) {   // this half's 4 blocks from the staged bounds (broadcast loads)
                const uint32_t sl = t % kBndRing;
                mbar_wait(&s.bfull[sl], (t / kBndRing) & 1);   // (long complete: loaded with the rows)
                const float4 *bp = reinterpret_cast<const float4 *>(&s.bnd[sl][half * 4]);
                const float4 b01 = bp[0], b23 = bp[1];   // (g, e) of blocks 0, 1 | 2, 3
                if (tl) atomicMax(&a.prof[64 + t * 8 + 6], (unsigned long long)clock64());
                th0 = __fadd_rd(h, __fsub_rd(b01.x, __fmul_ru(nqm, b01.y)));
                th1 = __fadd_rd(h, __fsub_rd(b01.z, __fmul_ru(nqm, b01.w)));
                th2 = __fadd_rd(h, __fsub_rd(b23.x, __fmul_ru(nqm, b23.y)));
                th3 = __fadd_rd(h, __fsub_rd(b23.z, __fmul_ru(nqm, b23.w)));
            } else {
                // lanes 0..3 (block c = lane): gB <= g_r on the block
                const float gB = __fsub_rd(gb.x, __fmul_ru(nqm, gb.y));
                th0 = __fadd_rd(h, __shfl_sync(0xffffffffu, gB, 0));
                th1 = __fadd_rd(h, __shfl_sync(0xffffffffu, gB, 1));
                th2 = __fadd_rd(h, __shfl_sync(0xffffffffu, gB, 2));
                th3 = __fadd_rd(h, __shfl_sync(0xffffffffu, gB, 3));
            }
            const uint32_t rb = t * kTileRows + half * 128;   // first row (within the item) of my columns
            const uint32_t nvalid = rb < it.count ? min(128u, it.count - rb) : 0u;
            const bool live = ql < qn && !(a.dbg & 4);
            uint32_t mk0 = 0u, mk1 = 0u, mk2 = 0u, mk3 = 0u;
            bool any = false;
            uint32_t v0[32], v1[32];
            // chunk 0: columns 0..63
            tmem_ld32(taddr, v0);
            tmem_ld32(taddr + 32, v1);
            tmem_ld_wait_regs(v0);   // orders every use of v0, v1 after the wait
            reg_fence(v1);
            if (tl) atomicMax(&a.prof[64 + t * 8 + 7], (unsigned long long)clock64());
            if (kBound) {
                float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
                max32(v0, m0, m1);
                max32(v1, m2, m3);
                if (nvalid >= 32) { track(__fsub_rd(m0, Gg)); track(__fsub_rd(m1, Gg)); }
                if (nvalid >= 64) { track(__fsub_rd(m2, Gg)); track(__fsub_rd(m3, Gg)); }
            } else if (!(a.dbg & 1)) {
                float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
                max32(v0, m0, m1);
                max32(v1, m2, m3);
                if ((fmaxf(m0, m1) >= th0 || fmaxf(m2, m3) >= th1) && live) {   // cold: the exact masks
                    mk0 = mask32(v0, th0, 0, nvalid);
                    mk1 = mask32(v1, th1, 32, nvalid);
                    any = true;
                }
            }
            // chunk 1: columns 64..127, then the buffer is free
            tmem_ld32(taddr + 64, v0);
            tmem_ld32(taddr + 96, v1);
            tmem_ld_wait_regs(v0);
            reg_fence(v1);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) { if (kPair) mbar_arrive_leader(&s.tempty[buf]); else mbar_arrive(&s.tempty[buf]); }
            const long long w2 = prof ? clock64() : 0;
            if (prof && lane == 0) ew_ld += w2 - w1;
            if (tl) atomicMax(&a.prof[64 + t * 8 + 3], (unsigned long long)w2);
            if (kBound) {
                float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
                max32(v0, m0, m1);
                max32(v1, m2, m3);
                if (nvalid >= 96) { track(__fsub_rd(m0, Gg)); track(__fsub_rd(m1, Gg)); }
                if (nvalid >= 128) { track(__fsub_rd(m2, Gg)); track(__fsub_rd(m3, Gg)); }
            } else if (!(a.dbg & 1)) {
                float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
                max32(v0, m0, m1);
                max32(v1, m2, m3);
                if ((fmaxf(m0, m1) >= th2 || fmaxf(m2, m3) >= th3) && live) {
                    mk2 = mask32(v0, th2, 64, nvalid);
                    mk3 = mask32(v1, th3, 96, nvalid);
                    any = true;
                }
                if (prof && lane == 0) ew_math += clock64() - w2;
                // cold path (rare): enqueue exactly the passing columns; columns past the
                // item's last row (last tile only) are excluded by the masks
                if constexpr (kInline) {   // (a separate instantiation: the call's ABI costs the others registers)
                    if (__any_sync(0xffffffffu, any)) {
                        if (a.stat_flagged && any) atomicAdd(a.stat_flagged, 1ull);
                        tc_rescore_warp(a, s, lists, it, q0, quarter * 32, mk0, mk1, mk2, mk3, rb);
                    }
                } else if (any) {
                    const long long e0 = clock64();
                    const uint32_t cnt = __popc(mk0) + __popc(mk1) + __popc(mk2) + __popc(mk3);
                    if (cnt) tc_enqueue_event(s, mk0, mk1, mk2, mk3, rb, ql, prof ? a.prof : nullptr);
                    if (prof && (a.dbg & 2048) && blockIdx.x == 0 && t < kTlTiles) atomicAdd(&a.prof[64 + t * 8 + 5], 1ull);
                    if (a.stat_flagged) atomicAdd(a.stat_flagged, 1ull);
                    if (prof) {
                        const unsigned long long d = clock64() - e0;
                        atomicAdd(&a.prof[2], d); atomicMax(&a.prof[3], d); atomicAdd(&a.prof[4], (unsigned long long)cnt);
                        atomicMax(&a.prof[5], (unsigned long long)cnt);
                    }
                }
            }
            // the shared threshold loaded at the start of this tile (its latency hidden by the tile):
            // tighten this frame's if another CTA did better.  Every tile: with the 32-dim filter
            // and 8-entry rings, refreshing every 4 / 2 / 1 own tiles measured C4 10.14 / 10.10 /
            // 10.08 ms (box-normalised), 20M rows 2.72 / 2.69 / 2.69, 1M 0.583 / 0.554 / 0.543
            if (refresher && ql < qn && gt < s.tau[ql]) atomicMin(&s.tau[ql], gt);
            if (prof && lane == 0) ew_tile += clock64() - ts;
            if (tl) atomicMax(&a.prof[64 + t * 8 + 4], (unsigned long long)clock64());
        };
        float2 gA = load_g(grp), gC = load_g(grp + 2);
        const long long l0 = clock64();
        for (uint32_t t = grp; t < n_tiles; t += 4) {
            tile(t, gA);
            if (t + 4 < n_tiles) gA = load_g(t + 4);
            if (t + 2 >= n_tiles) break;
            tile(t + 2, gC);
            if (t + 6 < n_tiles) gC = load_g(t + 6);
        }
        if constexpr (kBound) {
            if (ql < qn && !force_all && tl[kTrackMax - 1] > -INFINITY) {
                const float4 m = a.qmeta[q0 + ql];
                const float gam = __fadd_ru(__fadd_ru(m.z, __fmul_ru(2.f * m.y, nfm)), __fmul_ru(nqm, nfm) * 1.220703125e-04f);
                const float tu = fmaxf(__fmul_ru(__fsub_ru(gam, 2.f * tl[kTrackMax - 1]), kTauInflate), 0.f);
                atomicMin(&a.g_tau[(size_t)(q0 + ql) * a.n_sub + it.sub], __float_as_uint(tu));
            }
        }
        if (prof && lane == 0) {
            atomicAdd(&a.prof[6], (unsigned long long)ew_tfull);
            atomicAdd(&a.prof[12], (unsigned long long)ew_ld);
            atomicAdd(&a.prof[13], (unsigned long long)ew_math);
            atomicAdd(&a.prof[14], (unsigned long long)(clock64() - l0));
            atomicAdd(&a.prof[11], (unsigned long long)ew_tile);
            atomicAdd(&a.prof[15], (unsigned long long)(l0 - t_start));
        }
        named_bar(1, 32 * kEpiWarps);
        if (warp == 2 && lane == 0) {
            __threadfence_block();
            for (int w = 0; w < kExactWarps; ++w) sts_u32(&s.closed_at[w], lds_u32(&s.prod[w]));
            __threadfence_block();
            sts_u32(&s.closed, 1u);
        }
    } else {
        // ------------------------------------------------------------ exact re-scoring
        // The warp drains every published event of its ring at once (up to 32), flattens
        // their survivors and re-scores them 32 at a time, one lane per (frame, row), with
        // the exact fp32 chain (R3); then merges each frame's keys into its list.  The
        // warp owns its frames' lists (ql % kExactWarps), so no locks.  While idle, lanes
        // import the thresholds other CTAs published (any value ever held is a valid
        // bound, so races only loosen the test).
        const uint32_t xw = warp - (2 + kEpiWarps);
        for (unsigned p = 0; !kBound;) {
            bool got = false;
            uint32_t idle = 0, nap = 32;
            while (true) {
                if (lds_u32(&s.seq[xw][p % kEv]) == p + 1) { got = true; break; }
                if (lds_u32(&s.closed) && p >= lds_u32(&s.closed_at[xw])) break;
                const uint32_t qi = ((idle++ * 32 + lane) * kExactWarps + xw) % kQB;
                if (qi < qn) {
                    const uint32_t g = __ldcg(&a.g_tau[(size_t)(q0 + qi) * a.n_sub + it.sub]);
                    if (g < lds_u32(&s.tau[qi])) atomicMin(&s.tau[qi], g);
                }
                __nanosleep(nap);
                if (nap < 1024) nap <<= 1;
            }
            if (!__any_sync(0xffffffffu, got)) break;
            const long long x0 = prof ? clock64() : 0;
            // the run of published events p, p+1, ... (lane i: event p + i)
            const unsigned mp = p + lane;
            const bool rdy = lds_u32(&s.seq[xw][mp % kEv]) == mp + 1;
            const uint32_t rbits = __ballot_sync(0xffffffffu, rdy);
            const uint32_t ne = rbits == 0xFFFFFFFFu ? 32u : (uint32_t)(__ffs(~rbits) - 1);
            __threadfence_block();
            uint4 mv = make_uint4(0u, 0u, 0u, 0u);
            uint32_t head = 0;
            if (lane < ne) { mv = s.ev_mask[xw][mp % kEv]; head = s.ev_head[xw][mp % kEv]; }
            __syncwarp();
            __threadfence_block();
            if (lane < ne) sts_u32(&s.seq[xw][mp % kEv], mp + kEv);
            p += ne;
            if (a.dbg & 8) continue;   // profiling: drop survivors unscored (wrong results)
            // survivors per event and their inclusive prefix over the events
            const uint32_t cnt = __popc(mv.x) + __popc(mv.y) + __popc(mv.z) + __popc(mv.w);
            uint32_t incl = cnt;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            for (uint32_t base = 0; base < total; base += 32) {
                const uint32_t sidx = base + lane;
                // my survivor: event e (first with incl > sidx), its k-th passing row
                uint32_t e = 0;
                for (uint32_t j = 0; j < ne; ++j) e += __shfl_sync(0xffffffffu, incl, j) <= sidx;
                const uint32_t es = min(e, 31u);
                const uint32_t e_incl = __shfl_sync(0xffffffffu, incl, es), e_cnt = __shfl_sync(0xffffffffu, cnt, es);
                const uint32_t eh = __shfl_sync(0xffffffffu, head, es);
                const uint32_t w0 = __shfl_sync(0xffffffffu, mv.x, es), w1 = __shfl_sync(0xffffffffu, mv.y, es);
                const uint32_t w2 = __shfl_sync(0xffffffffu, mv.z, es), w3 = __shfl_sync(0xffffffffu, mv.w, es);
                const bool act = sidx < total;
                uint32_t col = 0xFFFFFFFFu;
                u64 key = kPadKey;
                if (act) {
                    uint32_t k = sidx - (e_incl - e_cnt), wsel = 0, w = w0;
                    if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w1; wsel = 1;
                        if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w2; wsel = 2;
                            if (k >= (uint32_t)__popc(w)) { k -= __popc(w); w = w3; wsel = 3; } } }
                    const uint32_t bit = __fns(w, 0, (int)k + 1);
                    col = eh & 0xFF;
                    const uint32_t rl = (eh >> 8) + 32 * wsel + bit;
                    const uint64_t row = it.row_begin + rl;
                    if (OL_DCHECK(rl < it.count && col < qn && q0 + col < a.nq)) {
                        const float4 *qv = reinterpret_cast<const float4 *>(a.queries + (size_t)(q0 + col) * kK);
                        // The chain is monotone (each step adds a square, RN is monotone), so once
                        // its first 32 steps exceed the frame's threshold the pair cannot reach the
                        // top-N: the second half of the row is read only for the rest (~1/3 of the
                        // survivors; this halves their random DRAM reads, which crowd the row
                        // stream's TMA loads during every CTA's start-up burst)
                        const float tcur = __uint_as_float(lds_u32(&s.tau[col]));
                        float acc = 0.f;
                        float4 f[kK / 8];
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            if (h == 1 && acc > tcur) break;
#pragma unroll
                            for (int k = 0; k < kK / 8; ++k) {
                                const int k4 = h * (kK / 8) + k;
                                f[k] = __ldg(reinterpret_cast<const float4 *>(a.fine + fine_off(row, 4 * k4)));
                            }
#pragma unroll
                            for (int k = 0; k < kK / 8; ++k) {
                                const float4 x = __ldg(qv + h * (kK / 8) + k);
                                acc = chain_step_tc(acc, x.x, f[k].x); acc = chain_step_tc(acc, x.y, f[k].y);
                                acc = chain_step_tc(acc, x.z, f[k].z); acc = chain_step_tc(acc, x.w, f[k].w);
                            }
                        }
                        key = ((u64)__float_as_uint(acc) << 32) | (u64)(it.frame_begin + rl);
                        // beyond the frame's threshold (a bound on the N-th best over all CTAs), or
                        // not below this CTA's N-th: cannot enter the top-N
                        if (acc > tcur || !(key < lists[(size_t)col * N + N - 1])) key = kPadKey;
                    } else col = 0xFFFFFFFFu;
                }
                // insert the keys into their frames' sorted lists: lanes of distinct frames in
                // parallel, lanes sharing a frame one after another (match groups)
                const bool has = key != kPadKey;
                const uint32_t peers = __match_any_sync(0xffffffffu, has ? col : 0xFFFFFFFFu);
                const uint32_t rank = __popc(peers & ((1u << lane) - 1));
                const uint32_t maxrank = __reduce_max_sync(0xffffffffu, has ? rank : 0u);
                const uint32_t heads = __ballot_sync(0xffffffffu, has && rank == 0);   // one lane per frame
                // few frames with many keys each: one warp-wide merge per frame; otherwise
                // lane-parallel insertion, maxrank + 1 rounds
                if (__popc(heads) <= 2 && maxrank >= 2) {
                    for (uint32_t hb = heads; hb; hb &= hb - 1) {
                        const uint32_t f = __shfl_sync(0xffffffffu, col, __ffs(hb) - 1);
                        tc_warp_merge(lists + (size_t)f * N, N, has && col == f ? key : kPadKey, lane);
                    }
                } else for (uint32_t r = 0; r <= maxrank; ++r) {
                    if (has && rank == r) {
                        u64 *L = lists + (size_t)col * N;
                        if (OL_DCHECK(col < qn) && key < L[N - 1]) {
                            int pidx = (int)N - 1;
                            while (pidx > 0 && L[pidx - 1] > key) { L[pidx] = L[pidx - 1]; --pidx; }
                            L[pidx] = key;
                        }
                    }
                    __syncwarp();
                }
                if (has && rank == 0) {   // one lane per frame: publish its tightened threshold
                    const u64 last = lists[(size_t)col * N + N - 1];
                    if (last != kPadKey) {
                        const uint32_t tb = (uint32_t)(last >> 32);
                        atomicMin(&s.tau[col], tb);
                        const size_t ti = (size_t)(q0 + col) * a.n_sub + it.sub;
                        atomicMin(&a.g_tau[ti], tb);
                        for (uint32_t pr = 0; pr < a.n_peer; ++pr) atomicMin(&a.peer_tau[pr][ti], tb);   // (RED over NVLink)
                    }
                }
                __syncwarp();
            }
            if (lane == 0) {
                if (a.stat_survivors) atomicAdd(a.stat_survivors, (unsigned long long)total);
                if (prof) atomicAdd(&a.prof[7], (unsigned long long)(clock64() - x0));
            }
            __syncwarp();
        }
    }

    // ---------------------------------------------------------------- teardown
    tc_fence_before();
    if (kPair) cluster_sync(); else __syncthreads();
    if (warp == 1) { if (kPair) tmem_dealloc2<512>(tmem); else tmem_dealloc<512>(tmem); }
    if (prof && threadIdx.x == 0) { atomicAdd(&a.prof[8], (unsigned long long)(clock64() - t_start)); atomicAdd(&a.prof[9], (unsigned long long)n_tiles); }
    for (uint32_t i = threadIdx.x; !kBound && i < qn * N; i += blockDim.x) {
        const uint32_t q = i / N, r = i % N;
        if (OL_DCHECK(q0 + q < a.nq))
            a.partial[((size_t)(q0 + q) * a.n_items + item_id) * N + r] = lists[(size_t)q * N + r];
    }
}

}  // namespace ol

namespace ol {

// ------------------------------------------------------------------ preparation kernels
// Per database row: the fp16 operand (RN) [rows][64]; per 32-row block (one warp's
// rows) the row-term bounds blk = (min_r RD||f_r||^2 / 2, max_r RU||f_r - f^_r||);
// the row norm bound max(||f||, ||f^||) folded into a database maximum (atomicMax on
// the bits of a non-negative float); the largest |f| (fp16 range check).  rows is a
// multiple of 32 (tile-padded), so every warp owns whole blocks.
__global__ void tc_prep_rows_kernel(const float *coarse, const float *fine, int kc, uint64_t rows,
                                    __half *plane, float2 *blk, uint32_t *stat, int kf, int pw) {
    uint32_t lmax = 0, lnorm = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        double n2 = 0, e2 = 0, h2 = 0;
        float amax = 0.f;
        __half2 *dst = reinterpret_cast<__half2 *>(plane + r * pw);
        for (int k = 0; k < kK; k += 2) {
            const float f0 = fine[fine_off(r, k)];
            const float f1 = fine[fine_off(r, k + 1)];
            const __half h0 = __float2half_rn(f0), h1 = __float2half_rn(f1);
            if (k < pw) dst[k / 2] = __halves2half2(h0, h1);
            amax = fmaxf(amax, fmaxf(fabsf(f0), fabsf(f1)));
            if (k >= kf) continue;   // the filter's terms cover dimensions < kf only
            const double d0 = (double)f0 - (double)__half2float(h0), d1 = (double)f1 - (double)__half2float(h1);
            n2 += (double)f0 * f0 + (double)f1 * f1;
            e2 += d0 * d0 + d1 * d1;
            h2 += (double)__half2float(h0) * __half2float(h0) + (double)__half2float(h1) * __half2float(h1);
        }
        // the double sums carry relative error < 2^-45; the (1 -+ 2^-20) factors cover it
        float x = 0.5f * __double2float_rd(n2 * (1.0 - 1.0 / 1048576.0));   // halving is exact
        float ef = __double2float_ru(sqrt(e2) * (1.0 + 1.0 / 1048576.0));
        // database maxima of RU||f||^2 / 2 and of e_f (the bound pre-pass's G); bits of
        // non-negative floats order like the floats
        atomicMax(&stat[4], __float_as_uint(0.5f * __double2float_ru(n2 * (1.0 + 1.0 / 1048576.0))));
        atomicMax(&stat[5], __float_as_uint(ef));
        for (int o = 16; o; o >>= 1) {
            x = fminf(x, __shfl_xor_sync(0xffffffffu, x, o));
            ef = fmaxf(ef, __shfl_xor_sync(0xffffffffu, ef, o));
        }
        if ((threadIdx.x & 31) == 0) blk[r >> 5] = make_float2(x, ef);
        const float nb = __double2float_ru(sqrt(fmax(n2, h2)) * (1.0 + 1.0 / 1048576.0));
        lnorm = max(lnorm, __float_as_uint(nb));
        lmax = max(lmax, __float_as_uint(amax));
    }
    for (int o = 16; o; o >>= 1) {
        lnorm = max(lnorm, __shfl_xor_sync(0xffffffffu, lnorm, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if ((threadIdx.x & 31) == 0) { atomicMax(&stat[0], lnorm); atomicMax(&stat[1], lmax); }
}

cudaError_t launch_tc_prep_rows(const float *coarse, const float *fine, int kc, uint64_t rows, void *plane,
                                float2 *blk, uint32_t *stat, uint32_t kf, uint32_t pw, cudaStream_t s) {
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    tc_prep_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(coarse, fine, kc, rows, (__half *)plane, blk, stat, (int)kf, (int)pw);
    return cudaGetLastError();
}

// Per query frame: fp16 operand rows [nq_pad][64] (zeros past nq), (RD ||q||^2,
// RU e_q), and the batch norm bound in *nq_max (+inf if a value leaves the fp16
// range: see force_all).  One warp per frame.
__global__ void tc_prep_queries_kernel(const float *q, uint32_t nq, uint32_t nq_pad, __half *q16,
                                       float4 *qmeta, uint32_t *nq_max, uint32_t *force_all, uint32_t kf, uint32_t pw) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nq_pad) return;
    __half2 *dst = reinterpret_cast<__half2 *>(q16 + (size_t)w * pw);
    const __half2 zero = __halves2half2(__float2half(0.f), __float2half(0.f));
    const bool wr = 2 * lane < pw;   // lanes holding a plane column
    if (w >= nq) { if (wr) dst[lane] = zero; return; }
    const float f0 = q[(size_t)w * kK + 2 * lane], f1 = q[(size_t)w * kK + 2 * lane + 1];
    // a value outside the fp16 range (or non-finite): this batch is scored exactly
    // for every pair (force_all); the frame's fp16 operand is zeroed to stay finite
    const bool bad = __any_sync(0xffffffffu, !(fabsf(f0) < 65000.f && fabsf(f1) < 65000.f));
    if (bad) {
        if (wr) dst[lane] = zero;
        if (lane == 0) { qmeta[w] = make_float4(0.f, 0.f, 0.f, 0.f); atomicOr(force_all, 1u); }
        return;
    }
    const __half h0 = __float2half_rn(f0), h1 = __float2half_rn(f1);
    if (wr) dst[lane] = __halves2half2(h0, h1);
    const double d0 = (double)f0 - (double)__half2float(h0), d1 = (double)f1 - (double)__half2float(h1);
    const bool in = 2 * lane < kf;   // the filter's terms cover dimensions < kf only
    double n2 = in ? (double)f0 * f0 + (double)f1 * f1 : 0.0, e2 = in ? d0 * d0 + d1 * d1 : 0.0;
    double h2 = in ? (double)__half2float(h0) * __half2float(h0) + (double)__half2float(h1) * __half2float(h1) : 0.0;
    for (int o = 16; o; o >>= 1) {
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    if (lane == 0) {
        qmeta[w] = make_float4(__double2float_rd(n2 * (1.0 - 1.0 / 1048576.0)),
                               __double2float_ru(sqrt(e2) * (1.0 + 1.0 / 1048576.0)),
                               __double2float_ru(n2 * (1.0 + 1.0 / 1048576.0)), 0.f);
        const float nb = __double2float_ru(sqrt(fmax(n2, h2)) * (1.0 + 1.0 / 1048576.0));
        atomicMax(nq_max, __float_as_uint(nb));
    }
}

cudaError_t launch_tc_prep_queries(const float *q, uint32_t nq, uint32_t nq_pad, void *q16, float4 *qmeta,
                                   uint32_t *bounds, uint32_t kf, uint32_t pw, cudaStream_t s) {
    const uint32_t threads = 256, blocks = (nq_pad * 32 + threads - 1) / threads;
    tc_prep_queries_kernel<<<blocks, threads, 0, s>>>(q, nq, nq_pad, (__half *)q16, qmeta, bounds + 2, bounds + 3, kf, pw);
    return cudaGetLastError();
}

__global__ void fill_u32_kernel(uint32_t *p, uint64_t n, uint32_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

cudaError_t launch_fill_u32(uint32_t *p, uint64_t n, uint32_t v, cudaStream_t s) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    if (blocks == 0) blocks = 1;
    fill_u32_kernel<<<(unsigned)blocks, 256, 0, s>>>(p, n, v);
    return cudaGetLastError();
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// 2-D map over an fp16 [rows][width] array (every row_stride-th row: a strided view) (width 64 -> 128-byte swizzle, width 16 ->
// 32-byte swizzle: the UMMA K-major canonical layouts), box {width, box_rows}.
bool make_tc_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint32_t box_rows, uint32_t width,
                 uint32_t row_stride) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)(rows / row_stride)};
    cuuint64_t strides[1] = {(cuuint64_t)width * sizeof(__half) * row_stride};
    cuuint32_t box[2] = {width, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE,
              width == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : width == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_tcscan(const CUtensorMap &map_rows, const CUtensorMap &map_q, const TcScanArgs &a, int grid,
                          cudaStream_t s) {
    const size_t smem = tc_smem_bytes(a.qb, a.N, a.stages, a.pw);
    const bool prof = (a.dbg & 32) != 0;
    const bool pair = a.pair && !a.bound;
    auto kern = a.bound ? (prof ? tcscan_kernel<true, true, false> : tcscan_kernel<false, true, false>)
              : pair    ? (prof ? tcscan_kernel<true, false, true> : tcscan_kernel<false, false, true>)
              : a.inline_rescore ? (prof ? tcscan_kernel<true, false, false, true> : tcscan_kernel<false, false, false, true>)
                        : (prof ? tcscan_kernel<true, false, false> : tcscan_kernel<false, false, false>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    // thread-block clusters over the query blocks of one work item (consecutive blockIdx):
    // co-scheduled on one GPC, so the CTAs streaming the same rows share a die's L2
    uint32_t cs = pair ? 2u : a.cluster ? a.cluster : 1;
    if (pair && (a.n_qblocks % 2 || grid % 2)) return cudaErrorInvalidValue;   // the runtime pads to pairs
    while (!pair && cs > 1 && (a.n_qblocks % cs || grid % cs)) cs >>= 1;
    if (cs <= 1) {
        kern<<<grid, kTcThreads, smem, s>>>(map_rows, map_q, a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, map_rows, map_q, a);
}

// Frames per CTA (128 or 256) and pipeline depth for top-N lists of N: the lists
// share the 227 KB of shared memory with the resident frames and the row stages.
bool tc_shape(uint32_t N, uint32_t nq, uint32_t pw, uint32_t *qb, uint32_t *stages) {
    (void)nq;
    const size_t budget = 227 * 1024, sb = kTileRows * pw * 2;
    const size_t fixed = 1024 + tc_fixed_bytes() + sizeof(u64) * kQB * N;
    if (fixed + 2 * sb > budget) return false;
    const uint32_t st = (uint32_t)((budget - fixed) / sb);
    *qb = kQB;
    *stages = st > (uint32_t)kMaxStages ? (uint32_t)kMaxStages : st;
    return true;
}

OL_CHECK_EXPORT(check_tcscan)

}  // namespace ol
