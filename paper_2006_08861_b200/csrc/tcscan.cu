// tcscan.cu -- tensor-core certified filter for the scan (NEXT-2 in SURVEY §8f,
// kernel NK8), used when a tile holds many query frames.
//
// The exact answer is still the fp32 chain of R3 (P:157 calculateDistance,
// P:202 "smallest Euclidean distance"); tensor cores only decide which pairs
// cannot possibly be in the top-N.  For fp32 vectors q, f with real squared
// distance A = ||q||^2 + ||f||^2 - 2 q.f and their fp16 roundings q^, f^:
//   q.f <= q^.f^ + ||q - q^|| ||f|| + ||q^|| ||f - f^||.
// With Nq, Nf upper bounds of the norms (batch / database maxima):
//   A >= alpha_q + beta_r - 2 q^.f^,
//   alpha_q = RD||q||^2 - 2 e_q Nf,   beta_r = RD||f||^2 - 2 Nq e_f,
// e = RU||x - x^||.  The tensor core computes, per (frame q, row r), the 80-term
// fp16 product sum  D' = q^.f^ + [-1, -1, Nq16] . [hi_r, lo_r, ef16_r]  with
// hi_r + lo_r <= beta_r's RD||f||^2 / 2 and Nq16 ef16_r >= Nq e_f (fp16, rounded
// the safe way), i.e. D' >= q^.f^ - beta_r / 2 up to the fp32 accumulation error
// of 80 exact products, <= 2^-14 sum|products| <= 2^-14 S (S bounded per batch).
// The fp32 chain satisfies acc >= A (1 - 66 u) >= A / (1 + 2^-17).  Hence
//   acc > tau_q  is guaranteed when  D' < h_q = (alpha'_q - tau_q (1 + 2^-17)) / 2,
//   alpha'_q = alpha_q - 2^-13 S - sigma,  sigma = 2^-18 (Nq + Nf)^2
// (sigma absorbs every fp32 rounding of the test).  Per (frame, row tile) the
// epilogue only needs max_r D' >= h_q: one FMNMX3 per two accumulators.  Pairs
// that pass ("survivors", ~1e-5 of pairs on paper-shaped data) are re-scored with
// the exact fp32 chain on CUDA cores and enter the top-N; everything else is
// provably outside it, so results are bit-identical to the one-pass scan
// (tests: test_gpu_tc, test_gpu_parity, test_gpu_fullsize).
//
// CTA = one work item (rows of one subspace) x <= 128 query frames (one M-tile).
// Warp roles: 0 TMA producer (128-row tiles: fp16 rows, 128-B swizzle; their
// 16-wide extra K block, 32-B swizzle; a mbarrier ring of n_stages);
// 1 TMEM allocator + single-thread tcgen05.mma issuer: per 256-row tile,
// M=128 frames x N=256 rows x K=80 (4 K16 blocks SW128 + 1 SW32) into a
// double-buffered fp32 TMEM accumulator (2 x 256 columns); 2..9 epilogue
// (thread = one frame x 128 of the tile's rows: tcgen05.ld, release the buffer,
// max, survivor enqueue); 10 exact re-scoring + top-N insertion.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "ol_internal.h"
#include "tc_ptx.cuh"

namespace ol {

using namespace tc;

constexpr int kTileRows = 256;          // MMA N (rows per tile)
constexpr int kQB = 128;                // frames per CTA: one M-tile
constexpr int kKx = 16;                 // extra K block (fp16): [-1, -1, Nq16] . [hi, lo, ef16]
constexpr int kMaxStages = 8;
constexpr int kEpiWarps = 8;
constexpr int kExactWarps = 2;
constexpr int kTcThreads = 32 * (2 + kEpiWarps + kExactWarps);
constexpr int kEv = 128;                // survivor event ring entries per exact warp
constexpr float kTauInflate = 1.0f + 1.0f / 131072.0f;   // 1 + 2^-17
constexpr uint32_t kStageBytes = kTileRows * (kK + kKx) * 2;   // 20 KB

struct TcSmem {
    alignas(1024) __half qm[kQB * kK];      // frames, main K (SW128), resident
    alignas(1024) __half qx[kQB * kKx];     // frames, extra K block (SW32), resident
    uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2], qbar;
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
    alignas(16) float qexact[kExactWarps][kK];   // the event's frame (fp32), per exact warp
    unsigned int prod[kExactWarps], closed_at[kExactWarps];
    int closed;
    // dynamic, 1024-aligned: n_stages x {rows main [128][64] SW128, rows extra [128][16] SW32},
    // then the top-N lists u64 [qb][N]
};

static __host__ __device__ constexpr size_t tc_fixed_bytes() { return (sizeof(TcSmem) + 1023) / 1024 * 1024; }

size_t tc_smem_bytes(uint32_t qb, uint32_t N, uint32_t stages) {
    return 1024 + tc_fixed_bytes() + (size_t)stages * kStageBytes + sizeof(u64) * qb * N;
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
__device__ __noinline__ void tc_enqueue_event(TcSmem &s, const uint32_t (&mk)[4], uint32_t rb, uint32_t ql,
                                              unsigned long long *prof) {
    const uint32_t w = ql % kExactWarps;
    const unsigned pos = atomicAdd(&s.prod[w], 1u);
    uint32_t *sq = &s.seq[w][pos % kEv];
    if (lds_u32(sq) != pos) {
        const long long r0 = clock64();
        while (lds_u32(sq) != pos) __nanosleep(64);
        if (prof) atomicAdd(&prof[10], (unsigned long long)(clock64() - r0));
    }
    s.ev_mask[w][pos % kEv] = make_uint4(mk[0], mk[1], mk[2], mk[3]);
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

__global__ void __launch_bounds__(kTcThreads, 1)
tcscan_kernel(const __grid_constant__ CUtensorMap map_rows, const __grid_constant__ CUtensorMap map_rowsx,
              const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_qx, TcScanArgs a) {
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char *base = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    TcSmem &s = *reinterpret_cast<TcSmem *>(base);
    unsigned char *stage0 = base + tc_fixed_bytes();
    const uint32_t n_stages = a.stages;
    u64 *lists = reinterpret_cast<u64 *>(stage0 + (size_t)n_stages * kStageBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t item_id = blockIdx.x / a.n_qblocks;
    const uint32_t qblk = blockIdx.x % a.n_qblocks;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qblk * a.qb;
    const uint32_t qn = min(a.qb, a.nq - q0);
    const uint32_t N = a.N;
    const uint32_t n_tiles = (it.count + kTileRows - 1) / kTileRows;
    const bool prof = (a.dbg & 32) != 0;
    const long long t_start = clock64();

    // ---------------------------------------------------------------- setup
    if (threadIdx.x == 0) {
        for (uint32_t i = 0; i < n_stages; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], kEpiWarps); }
        mbar_init(&s.qbar, 1);
        fence_mbar_init();
        for (int w = 0; w < kExactWarps; ++w) s.prod[w] = s.closed_at[w] = 0;
        s.closed = 0;
        tma_prefetch(&map_rows);
        tma_prefetch(&map_rowsx);
    }
    if (warp == 1) tmem_alloc<512>(&s.tmem_base);
    const float nqm = __uint_as_float(a.bounds[2]), nfm = a.nf_max;
    const bool force_all = a.bounds[3] != 0;
    const float sigma = 3.814697265625e-06f * (nqm + nfm) * (nqm + nfm);      // 2^-18 (Nq + Nf)^2
    // 2^-13 x a bound of sum |products| over the 80 terms: Nq Nf + Nf^2 / 2 + Nq16 (2^-11 Nf + 2^-22)
    const float S = nqm * nfm + 0.5f * nfm * nfm + 1.001f * nqm * (4.8828125e-04f * nfm + 2.384185791e-07f);
    const float c0 = 1.220703125e-04f * S;
    for (uint32_t q = threadIdx.x; q < kQB; q += blockDim.x) {
        if (q < qn) {
            const float2 m = a.qmeta[q0 + q];  // (RD ||q||^2, RU e_q)
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
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            mbar_expect_tx(&s.qbar, a.qb * (kK + kKx) * (uint32_t)sizeof(__half));
            tma_load_2d(s.qm, &map_q, &s.qbar, 0, (int)q0);
            tma_load_2d(s.qx, &map_qx, &s.qbar, 0, (int)q0);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % n_stages;
                if (t >= n_stages) mbar_wait_sleep(&s.empty[st], ((t / n_stages) - 1) & 1);
                unsigned char *sb = stage0 + (size_t)st * kStageBytes;
                const int r0 = (int)(it.row_begin + (uint64_t)t * kTileRows);
                if ((a.dbg & 128) && t >= n_stages) { mbar_arrive(&s.full[st]); continue; }   // profiling: stale rows
                mbar_expect_tx(&s.full[st], kStageBytes);
                tma_load_2d(sb, &map_rows, &s.full[st], 0, r0);
                tma_load_2d(sb + kTileRows * kK * 2, &map_rowsx, &s.full[st], 0, r0);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_f16_f32(128, kTileRows);   // M = 128 frames, N = 256 rows
            long long pw_full = 0, pw_tempty = 0;
            mbar_wait(&s.qbar, 0);
            const uint32_t qm = smem_u32(s.qm), qx = smem_u32(s.qx);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % n_stages, buf = t & 1;
                long long c0 = clock64();
                mbar_wait_sleep(&s.full[st], (t / n_stages) & 1);
                long long c1 = clock64();
                if (t >= 2) mbar_wait_sleep(&s.tempty[buf], ((t >> 1) - 1) & 1);
                if (prof) { pw_full += c1 - c0; pw_tempty += clock64() - c1; }
                tc_fence_after();
                const uint32_t rm = smem_u32(stage0 + (size_t)st * kStageBytes), rx = rm + kTileRows * kK * 2;
                const uint32_t d = tmem + buf * kTileRows;
                if (!(a.dbg & 2)) {
#pragma unroll
                    for (int k = 0; k < kK / 16; ++k)
                        mma_f16(d, desc_sw128_kmajor(qm + k * 32), desc_sw128_kmajor(rm + k * 32), idesc, k > 0 ? 1u : 0u);
                    mma_f16(d, desc_sw32_kmajor(qx), desc_sw32_kmajor(rx), idesc, 1u);
                }
                mma_commit(&s.empty[st]);
                mma_commit(&s.tfull[buf]);
            }
            if (prof) { atomicAdd(&a.prof[0], (unsigned long long)pw_full); atomicAdd(&a.prof[1], (unsigned long long)pw_tempty); }
        }
    } else if (warp < 2 + kEpiWarps) {
        // ------------------------------------------------------------ epilogue
        // thread = one frame (TMEM lane) of one M-tile; its 128 row columns per tile
        const int ew = warp - 2;                  // 0..7
        const uint32_t quarter = warp & 3;        // TMEM lanes 32*quarter ..
        const uint32_t half = ew >> 2;            // row columns half*128 .. +128
        const uint32_t ql = quarter * 32 + lane;  // frame within the CTA
        const bool refresher = half == 0;         // one of the two warps per frame refreshes tau
        const float alpha = s.alpha[ql];
        uint32_t gt = 0xFFFFFFFFu;                // shared running threshold, loaded 8 tiles ahead
        long long ew_tfull = 0;
        for (uint32_t t = 0; t < n_tiles; ++t) {
            const uint32_t buf = t & 1;
            const uint32_t gt_prev = gt;
            if (refresher && (t & 7) == 0 && ql < qn) gt = __ldcg(&a.g_tau[(size_t)(q0 + ql) * a.n_sub + it.sub]);
            const long long w0 = prof ? clock64() : 0;
            mbar_wait_sleep(&s.tfull[buf], (t >> 1) & 1);
            if (prof && lane == 0) ew_tfull += clock64() - w0;
            tc_fence_after();
            uint32_t v0[32], v1[32], v2[32], v3[32];
            const uint32_t taddr = tmem + ((quarter * 32) << 16) + buf * kTileRows + half * 128;
            tmem_ld32(taddr, v0);
            tmem_ld32(taddr + 32, v1);
            tmem_ld32(taddr + 64, v2);
            tmem_ld32(taddr + 96, v3);
            tmem_ld_wait_regs(v0);   // orders every use of v0..v3 after the wait
            reg_fence(v1);
            reg_fence(v2);
            reg_fence(v3);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.tempty[buf]);
            if (!(a.dbg & 1)) {
                const float h = 0.5f * (alpha - __uint_as_float(lds_u32(&s.tau[ql])) * kTauInflate);
                const uint32_t rb = t * kTileRows + half * 128;   // first row (within the item) of my columns
                const uint32_t nvalid = rb < it.count ? min(128u, it.count - rb) : 0u;
                float m0 = -INFINITY, m1 = -INFINITY;
                max32(v0, m0, m1);
                max32(v1, m0, m1);
                max32(v2, m0, m1);
                max32(v3, m0, m1);
                // cold path (rare): enqueue exactly the passing columns; columns past the
                // item's last row (last tile only) are excluded by the mask
                if (fmaxf(m0, m1) >= h && ql < qn && !(a.dbg & 4)) {
                    const long long e0 = clock64();
                    uint32_t mk[4] = {mask32(v0, h, 0, nvalid), mask32(v1, h, 32, nvalid),
                                      mask32(v2, h, 64, nvalid), mask32(v3, h, 96, nvalid)};
                    const uint32_t cnt = __popc(mk[0]) + __popc(mk[1]) + __popc(mk[2]) + __popc(mk[3]);
                    if (cnt) tc_enqueue_event(s, mk, rb, ql, prof ? a.prof : nullptr);
                    if (a.stat_flagged) atomicAdd(a.stat_flagged, 1ull);
                    if (prof) {
                        const unsigned long long d = clock64() - e0;
                        atomicAdd(&a.prof[2], d); atomicMax(&a.prof[3], d); atomicAdd(&a.prof[4], (unsigned long long)cnt);
                        atomicMax(&a.prof[5], (unsigned long long)cnt);
                    }
                }
            }
            // the shared threshold loaded 8 tiles ago: tighten this frame's if another CTA did better
            if (refresher && (t & 7) == 7 && ql < qn && gt_prev < lds_u32(&s.tau[ql])) atomicMin(&s.tau[ql], gt_prev);
        }
        if (prof && lane == 0) atomicAdd(&a.prof[6], (unsigned long long)ew_tfull);
        named_bar(1, 32 * kEpiWarps);
        if (warp == 2 && lane == 0) {
            __threadfence_block();
            for (int w = 0; w < kExactWarps; ++w) sts_u32(&s.closed_at[w], lds_u32(&s.prod[w]));
            __threadfence_block();
            sts_u32(&s.closed, 1u);
        }
    } else {
        // ------------------------------------------------------------ exact re-scoring
        // one warp per event: lane j re-scores row rb + 32 c + j of each pass mask c with
        // the exact fp32 chain (R3); the warp owns its frames' lists, so insertion needs
        // no lock.  Idle lanes import the thresholds other CTAs published (any value ever
        // held is a valid bound, so races only loosen the test).
        const uint32_t xw = warp - (2 + kEpiWarps);
        float *qe = s.qexact[xw];
        for (unsigned p = 0;; ++p) {
            uint32_t *sq = &s.seq[xw][p % kEv];
            bool got = false;
            uint32_t idle = 0, nap = 32;
            while (true) {
                if (lds_u32(sq) == p + 1) { got = true; break; }
                if (lds_u32(&s.closed) && p >= lds_u32(&s.closed_at[xw])) break;
                const uint32_t qi = ((idle++ * 32 + lane) * kExactWarps + xw) % kQB;
                if (qi < qn) {
                    const uint32_t g = __ldcg(&a.g_tau[(size_t)(q0 + qi) * a.n_sub + it.sub]);
                    if (g < lds_u32(&s.tau[qi])) atomicMin(&s.tau[qi], g);
                }
                __nanosleep(nap);
                if (nap < 1024) nap <<= 1;
            }
            if (!got) break;
            const long long x0 = prof ? clock64() : 0;
            __threadfence_block();
            const uint4 mv = s.ev_mask[xw][p % kEv];
            const uint32_t head = s.ev_head[xw][p % kEv];
            __syncwarp();
            __threadfence_block();
            if (lane == 0) sts_u32(sq, p + kEv);
            if (a.dbg & 8) continue;   // profiling: drop survivors unscored (wrong results)
            const uint32_t col = head & 0xFF, rb = head >> 8;
            if (lane < kK / 4)
                reinterpret_cast<float4 *>(qe)[lane] = __ldg(reinterpret_cast<const float4 *>(a.queries + (size_t)(q0 + col) * kK) + lane);
            __syncwarp();
            u64 *L = lists + (size_t)col * N;
            const uint32_t mks[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                if (!mks[c]) continue;
                const bool act = (mks[c] >> lane) & 1u;
                u64 key = kPadKey;
                if (act) {
                    const uint32_t rl = rb + 32 * c + lane;
                    const uint64_t row = it.row_begin + rl;
                    float4 f[kK / 4];
#pragma unroll
                    for (int k4 = 0; k4 < kK / 4; ++k4)
                        f[k4] = 4 * k4 < (int)a.kc
                                    ? __ldg(reinterpret_cast<const float4 *>(a.coarse + coarse_off(row, 4 * k4, a.kc)))
                                    : __ldg(reinterpret_cast<const float4 *>(a.fine + row * (kK - a.kc) + (4 * k4 - a.kc)));
                    float acc = 0.f;
#pragma unroll
                    for (int k4 = 0; k4 < kK / 4; ++k4) {
                        const float4 x = reinterpret_cast<const float4 *>(qe)[k4];
                        acc = chain_step_tc(acc, x.x, f[k4].x); acc = chain_step_tc(acc, x.y, f[k4].y);
                        acc = chain_step_tc(acc, x.z, f[k4].z); acc = chain_step_tc(acc, x.w, f[k4].w);
                    }
                    key = ((u64)__float_as_uint(acc) << 32) | (u64)(it.frame_begin + rl);
                }
                // merge the warp's keys into the sorted list: every key's rank in the union
                // (keys are distinct: one per (frame, row); pads rank last) is its new slot
                if (__any_sync(0xffffffffu, key < lds_u64(&L[N - 1]))) tc_warp_merge(L, N, key, lane);
            }
            if (lane == 0) {
                const u64 last = L[N - 1];
                if (last != kPadKey) {
                    const uint32_t tb = (uint32_t)(last >> 32);
                    atomicMin(&s.tau[col], tb);
                    atomicMin(&a.g_tau[(size_t)(q0 + col) * a.n_sub + it.sub], tb);
                }
                if (a.stat_survivors) atomicAdd(a.stat_survivors, (unsigned long long)(__popc(mv.x) + __popc(mv.y) + __popc(mv.z) + __popc(mv.w)));
                if (prof) atomicAdd(&a.prof[7], (unsigned long long)(clock64() - x0));
            }
            __syncwarp();
        }
    }

    // ---------------------------------------------------------------- teardown
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<512>(tmem);
    if (prof && threadIdx.x == 0) { atomicAdd(&a.prof[8], (unsigned long long)(clock64() - t_start)); atomicAdd(&a.prof[9], (unsigned long long)n_tiles); }
    for (uint32_t i = threadIdx.x; i < qn * N; i += blockDim.x) {
        const uint32_t q = i / N, r = i % N;
        a.partial[((size_t)(q0 + q) * a.n_items + item_id) * N + r] = lists[(size_t)q * N + r];
    }
}

}  // namespace ol

namespace ol {

// ------------------------------------------------------------------ preparation kernels
// Per database row: the fp16 operand (RN), RD(||f||^2), RU(||f - f^||), and the
// row norm bound max(||f||, ||f^||) folded into a database maximum (atomicMax on
// the bits of a non-negative float).  Also the largest |f| (fp16 range check).
// Per database row: the fp16 operand (RN) [rows][64]; its extra K block [rows][16]
// = (hi, lo, ef16, 0...) with hi = RN16(x), lo = RD16(x - hi) for x = RD||f||^2 / 2
// (so hi + lo <= x) and ef16 = RU16(RU||f - f^||); the row norm bound
// max(||f||, ||f^||) folded into a database maximum (atomicMax on the bits of a
// non-negative float); the largest |f| (fp16 range check).
__global__ void tc_prep_rows_kernel(const float *coarse, const float *fine, int kc, uint64_t rows,
                                    __half *plane, __half *ext, uint32_t *nf_max, uint32_t *maxabs) {
    uint32_t lmax = 0, lnorm = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows;
         r += (uint64_t)gridDim.x * blockDim.x) {
        double n2 = 0, e2 = 0, h2 = 0;
        float amax = 0.f;
        __half2 *dst = reinterpret_cast<__half2 *>(plane + r * kK);
        for (int k = 0; k < kK; k += 2) {
            const float f0 = k < kc ? coarse[coarse_off(r, k, kc)] : fine[r * (kK - kc) + (k - kc)];
            const float f1 = k + 1 < kc ? coarse[coarse_off(r, k + 1, kc)] : fine[r * (kK - kc) + (k + 1 - kc)];
            const __half h0 = __float2half_rn(f0), h1 = __float2half_rn(f1);
            dst[k / 2] = __halves2half2(h0, h1);
            const double d0 = (double)f0 - (double)__half2float(h0), d1 = (double)f1 - (double)__half2float(h1);
            n2 += (double)f0 * f0 + (double)f1 * f1;
            e2 += d0 * d0 + d1 * d1;
            h2 += (double)__half2float(h0) * __half2float(h0) + (double)__half2float(h1) * __half2float(h1);
            amax = fmaxf(amax, fmaxf(fabsf(f0), fabsf(f1)));
        }
        const float fn_lo = __double2float_rd(n2 * (1.0 - 1.0 / 1048576.0));
        const float ef = __double2float_ru(sqrt(e2) * (1.0 + 1.0 / 1048576.0));
        const float x = 0.5f * fn_lo;   // exact
        const __half hi = __float2half_rn(x);
        const __half lo = __float2half_rd(x - __half2float(hi));   // x - hi is exact in fp32
        __half *xr = ext + r * 16;
        xr[0] = hi; xr[1] = lo; xr[2] = __float2half_ru(ef);
        for (int k = 3; k < 16; ++k) xr[k] = __float2half(0.f);
        const float nb = __double2float_ru(sqrt(fmax(n2, h2)) * (1.0 + 1.0 / 1048576.0));
        lnorm = max(lnorm, __float_as_uint(nb));
        lmax = max(lmax, __float_as_uint(amax));
    }
    for (int o = 16; o; o >>= 1) {
        lnorm = max(lnorm, __shfl_xor_sync(0xffffffffu, lnorm, o));
        lmax = max(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    }
    if ((threadIdx.x & 31) == 0) { atomicMax(nf_max, lnorm); atomicMax(maxabs, lmax); }
}

cudaError_t launch_tc_prep_rows(const float *coarse, const float *fine, int kc, uint64_t rows, void *plane,
                                void *ext, uint32_t *nf_max, uint32_t *maxabs, cudaStream_t s) {
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    tc_prep_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(coarse, fine, kc, rows, (__half *)plane, (__half *)ext,
                                                         nf_max, maxabs);
    return cudaGetLastError();
}

// Per query frame: fp16 operand rows [nq_pad][64] (zeros past nq), (RD ||q||^2,
// RU e_q), and the batch norm bound in *nq_max (+inf if a value leaves the fp16
// range: see force_all).  One warp per frame.
__global__ void tc_prep_queries_kernel(const float *q, uint32_t nq, uint32_t nq_pad, __half *q16,
                                       float2 *qmeta, uint32_t *nq_max, uint32_t *force_all) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= nq_pad) return;
    __half2 *dst = reinterpret_cast<__half2 *>(q16 + (size_t)w * kK);
    const __half2 zero = __halves2half2(__float2half(0.f), __float2half(0.f));
    if (w >= nq) { dst[lane] = zero; return; }
    const float f0 = q[(size_t)w * kK + 2 * lane], f1 = q[(size_t)w * kK + 2 * lane + 1];
    // a value outside the fp16 range (or non-finite): this batch is scored exactly
    // for every pair (force_all); the frame's fp16 operand is zeroed to stay finite
    const bool bad = __any_sync(0xffffffffu, !(fabsf(f0) < 65000.f && fabsf(f1) < 65000.f));
    if (bad) {
        dst[lane] = zero;
        if (lane == 0) { qmeta[w] = make_float2(0.f, 0.f); atomicOr(force_all, 1u); }
        return;
    }
    const __half h0 = __float2half_rn(f0), h1 = __float2half_rn(f1);
    dst[lane] = __halves2half2(h0, h1);
    const double d0 = (double)f0 - (double)__half2float(h0), d1 = (double)f1 - (double)__half2float(h1);
    double n2 = (double)f0 * f0 + (double)f1 * f1, e2 = d0 * d0 + d1 * d1;
    double h2 = (double)__half2float(h0) * __half2float(h0) + (double)__half2float(h1) * __half2float(h1);
    for (int o = 16; o; o >>= 1) {
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
        h2 += __shfl_xor_sync(0xffffffffu, h2, o);
    }
    if (lane == 0) {
        qmeta[w] = make_float2(__double2float_rd(n2 * (1.0 - 1.0 / 1048576.0)),
                               __double2float_ru(sqrt(e2) * (1.0 + 1.0 / 1048576.0)));
        const float nb = __double2float_ru(sqrt(fmax(n2, h2)) * (1.0 + 1.0 / 1048576.0));
        atomicMax(nq_max, __float_as_uint(nb));
    }
}

// The frames' extra K block [nq_pad][16] = (-1, -1, RU16(Nq), 0...) once the batch
// norm bound is known; zeros for padded / out-of-range frames.  A bound too large
// for the fp16 products (Nq >= 300) sends the whole batch to exact re-scoring.
__global__ void tc_prep_qext_kernel(uint32_t nq, uint32_t nq_pad, const float2 *qmeta, uint32_t *bounds,
                                    __half *qx) {
    const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= nq_pad) return;
    const float nq_max = __uint_as_float(bounds[2]);
    if (w == 0 && !(nq_max < 300.f)) atomicOr(&bounds[3], 1u);
    __half *x = qx + (size_t)w * 16;
    const bool live = w < nq && nq_max < 300.f;
    x[0] = __float2half(live ? -1.f : 0.f);
    x[1] = __float2half(live ? -1.f : 0.f);
    x[2] = live ? __float2half_ru(nq_max) : __float2half(0.f);
    for (int k = 3; k < 16; ++k) x[k] = __float2half(0.f);
}

cudaError_t launch_tc_prep_queries(const float *q, uint32_t nq, uint32_t nq_pad, void *q16, void *qx, float2 *qmeta,
                                   uint32_t *bounds, cudaStream_t s) {
    const uint32_t threads = 256, blocks = (nq_pad * 32 + threads - 1) / threads;
    tc_prep_queries_kernel<<<blocks, threads, 0, s>>>(q, nq, nq_pad, (__half *)q16, qmeta, bounds + 2, bounds + 3);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    tc_prep_qext_kernel<<<(nq_pad + 255) / 256, 256, 0, s>>>(nq, nq_pad, qmeta, bounds, (__half *)qx);
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

// 2-D map over an fp16 [rows][width] array (width 64 -> 128-byte swizzle, width 16 ->
// 32-byte swizzle: the UMMA K-major canonical layouts), box {width, box_rows}.
bool make_tc_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint32_t box_rows, uint32_t width) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)width * sizeof(__half)};
    cuuint32_t box[2] = {width, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, width == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_32B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_tcscan(const CUtensorMap &map_rows, const CUtensorMap &map_rowsx, const CUtensorMap &map_q,
                          const CUtensorMap &map_qx, const TcScanArgs &a, int grid, cudaStream_t s) {
    const size_t smem = tc_smem_bytes(a.qb, a.N, a.stages);
    cudaError_t e = cudaFuncSetAttribute(tcscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tcscan_kernel<<<grid, kTcThreads, smem, s>>>(map_rows, map_rowsx, map_q, map_qx, a);
    return cudaGetLastError();
}

// Frames per CTA (128 or 256) and pipeline depth for top-N lists of N: the lists
// share the 227 KB of shared memory with the resident frames and the row stages.
bool tc_shape(uint32_t N, uint32_t nq, uint32_t *qb, uint32_t *stages) {
    (void)nq;
    const size_t budget = 227 * 1024;
    const size_t fixed = 1024 + tc_fixed_bytes() + sizeof(u64) * kQB * N;
    if (fixed + 2 * kStageBytes > budget) return false;
    const uint32_t st = (uint32_t)((budget - fixed) / kStageBytes);
    *qb = kQB;
    *stages = st > (uint32_t)kMaxStages ? (uint32_t)kMaxStages : st;
    return true;
}

}  // namespace ol
