// tcscan.cu -- tensor-core certified filter for the scan (NEXT-2 in SURVEY §8f,
// kernel NK8), used when a batch has many query frames.
//
// The exact answer is still the fp32 chain of R3 (P:157 calculateDistance,
// P:202 "smallest Euclidean distance"); tensor cores only decide which pairs
// cannot possibly be in the top-N.  For fp32 vectors q, f with real squared
// distance A = ||q||^2 + ||f||^2 - 2 q.f, and their fp16 roundings q^, f^:
//   q.f <= D + 2^-14 |q^||f^| + ||q - q^|| ||f|| + ||q^|| ||f - f^||
// where D is the tensor core's fp32-accumulated fp16 dot product (products of
// fp16 are exact; 2^-14 over-covers any accumulation order of 64 terms).  With
// Nq, Nf upper bounds of the norms (batch / database maxima):
//   A >= alpha_q + beta_r - 2 D,
//   alpha_q = RD(||q||^2) - 2 e_q Nf - 2^-13 Nq Nf - sigma,   e_q = RU||q - q^||,
//   beta_r  = RD(||f||^2) - 2 Nq e_f,                          e_f = RU||f - f^||,
// sigma = 2^-18 (Nq + Nf)^2 absorbing every fp32 rounding of this test.  The
// fp32 chain satisfies acc >= A (1 - 66 u) >= A / (1 + 2^-17), so
//   acc > tau  is guaranteed when  D < h_q + g_r,  h_q = (alpha_q - tau(1+2^-17))/2,
//   g_r = beta_r / 2.
// Pairs failing that test ("survivors", ~1e-4 of pairs on paper-shaped data)
// are re-scored with the exact fp32 chain on CUDA cores and enter the top-N;
// everything else is provably outside it.  Results are therefore bit-identical
// to the one-pass scan (tests: test_gpu_parity, test_gpu_tc).
//
// CTA = one work item (rows of one subspace) x one block of <= 256 query frames.
// Warp roles: 0 TMA producer of 128-row fp16 tiles (SW128, 4-stage mbarrier
// ring); 1 TMEM allocator + single-thread tcgen05.mma issuer (M=128 rows,
// N=query block, K=64 as 4 x K16) into a double-buffered TMEM accumulator
// (2 x 256 columns); 2..17 epilogue (tcgen05.ld, threshold test, survivor
// push; 4 warps per TMEM lane quarter, 64 columns each); 18..19 exact
// re-scoring + top-N insertion.
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "ol_internal.h"
#include "tc_ptx.cuh"

namespace ol {

using namespace tc;

constexpr int kTileRows = 128;
constexpr int kStages = 8;
constexpr int kQB = 256;                 // max query frames per CTA (MMA N)
constexpr int kEpiWarps = 16;
constexpr int kExactWarps = 1;
constexpr int kTcThreads = 32 * (2 + kEpiWarps + kExactWarps);
constexpr int kRing = 1024;              // survivor ring entries (r_local << 8 | q_local)
constexpr float kTauInflate = 1.0f + 1.0f / 131072.0f;   // 1 + 2^-17

struct TcSmem {
    alignas(1024) __half b[kQB * kK];                // query block (resident)
    alignas(1024) __half a[kStages][kTileRows * kK];  // row tiles
    alignas(16) float2 rm[kStages][kTileRows + 2];   // the tiles' (RD ||f||^2, RU e_f), from an
                                                     // even row (16-B aligned bulk copy)
    uint64_t full[kStages], empty[kStages], tfull[2], tempty[2], qbar;
    uint32_t tmem_base;
    alignas(16) float alpha[kQB];
    alignas(16) float h[kQB];   // h_q = (alpha_q - tau_q (1 + 2^-17)) / 2
    uint32_t tau[kQB];
    int lock[kQB];
    // survivor queue: bounded MPMC ring with per-slot sequence numbers (Vyukov):
    // slot i is free for position p when seq == p, filled when seq == p + 1
    uint32_t seq[kRing], val[kRing];
    unsigned int prod, cons_res, closed_at;
    int closed;
    // top-N lists follow (dynamic): u64 [qb][N]
};

size_t tc_smem_bytes(uint32_t qb, uint32_t N) { return sizeof(TcSmem) + 1024 + sizeof(u64) * qb * N; }

__device__ __forceinline__ float chain_step_tc(float acc, float q, float f) {
    float d = __fsub_rn(q, f);
    return __fmaf_rn(d, d, acc);
}

__device__ __forceinline__ uint32_t lds_u32(const void *p) {  // volatile shared-memory load
    return *reinterpret_cast<const volatile uint32_t *>(p);
}
__device__ __forceinline__ uint64_t lds_u64(const void *p) {
    return *reinterpret_cast<const volatile uint64_t *>(p);
}
__device__ __forceinline__ void sts_u32(void *p, uint32_t v) {  // volatile shared-memory store
    *reinterpret_cast<volatile uint32_t *>(p) = v;
}

__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) { return ((uint64_t)hi << 32) | lo; }
__device__ __forceinline__ uint64_t sub2(uint64_t a, uint64_t b) {  // FADD2: two RN fp32 subtractions
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ float h_of(float alpha, uint32_t tau_bits) {
    return 0.5f * (alpha - __uint_as_float(tau_bits) * kTauInflate);
}

__device__ __forceinline__ float max3f(float a, float b, float c) {  // FMNMX3
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Threshold test of 32 accumulator columns of one row: x = (D - g) - h per
// column (two FADD2 per column pair); sets bit `chunk` of flags if any x >= 0.
__device__ __forceinline__ void tc_test32(const uint32_t (&v)[32], uint64_t gg, const uint64_t *h2,
                                          uint32_t &flags, int chunk) {
    uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu;
#pragma unroll
    for (int j = 0; j < 16; j += 2) {
        const uint64_t x0 = sub2(sub2(pack2(v[2 * j], v[2 * j + 1]), gg), h2[j]);
        const uint64_t x1 = sub2(sub2(pack2(v[2 * j + 2], v[2 * j + 3]), gg), h2[j + 1]);
        const uint32_t m = (uint32_t)x0 & (uint32_t)(x0 >> 32) & (uint32_t)x1 & (uint32_t)(x1 >> 32);
        if (j & 2) a1 &= m; else a0 &= m;
    }
    flags |= ((~(a0 & a1)) >> 31) << chunk;
}
// Bit mask of the passing columns among 32 (same arithmetic as tc_test32).
__device__ __forceinline__ uint32_t tc_mask32(const uint32_t (&v)[32], uint64_t gg, const uint64_t *h2) {
    uint32_t mask = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const uint64_t x = sub2(sub2(pack2(v[2 * j], v[2 * j + 1]), gg), h2[j]);
        mask |= ((~(uint32_t)x >> 31) << (2 * j)) | ((~(uint32_t)(x >> 32) >> 31) << (2 * j + 1));
    }
    return mask;
}

// Enqueue a survivor (r_local << 8 | column) on the MPMC ring, waiting while
// the ring is full.
__device__ __forceinline__ void tc_enqueue(TcSmem &s, uint32_t e) {
    const unsigned pos = atomicAdd(&s.prod, 1u);
    uint32_t *sq = &s.seq[pos % kRing];
    while (lds_u32(sq) != pos) __nanosleep(64);
    s.val[pos % kRing] = e;
    __threadfence_block();
    sts_u32(sq, pos + 1);
}

// Cold path of the epilogue: the row passed for some of its 64 columns; find them
// (same arithmetic as the hot test) and enqueue them.  Kept out of line so the
// hot loop's register allocation does not carry it.
__device__ __noinline__ void tc_cold(TcSmem &s, const uint32_t *v, float g, uint32_t cb, uint32_t qn,
                                     uint32_t rl, unsigned long long *stat_flagged) {
    for (uint32_t j = 0; j < 64; ++j)
        if (cb + j < qn && __fsub_rn(__uint_as_float(v[j]), s.h[cb + j]) >= g) tc_enqueue(s, (rl << 8) | (cb + j));
    if (stat_flagged) atomicAdd(stat_flagged, 1ull);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(kTcThreads, 1)
tcscan_kernel(const __grid_constant__ CUtensorMap map_rows, const __grid_constant__ CUtensorMap map_q,
              TcScanArgs a) {
    extern __shared__ __align__(1024) unsigned char raw[];
    TcSmem &s = *reinterpret_cast<TcSmem *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    u64 *lists = reinterpret_cast<u64 *>(&s + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t item_id = blockIdx.x / a.n_qblocks;
    const uint32_t qblk = blockIdx.x % a.n_qblocks;
    const WorkItem it = a.items[item_id];
    const uint32_t q0 = qblk * a.qb;
    const uint32_t qn = min(a.qb, a.nq - q0);
    const uint32_t N = a.N;
    const uint32_t n_tiles = (it.count + kTileRows - 1) / kTileRows;

    // ---------------------------------------------------------------- setup
    if (threadIdx.x == 0) {
        // a stage is free once the MMA consumed its rows AND every epilogue warp read
        // its bound terms (rm)
        for (int i = 0; i < kStages; ++i) { mbar_init(&s.full[i], 1); mbar_init(&s.empty[i], 1 + kEpiWarps); }
        for (int i = 0; i < 2; ++i) { mbar_init(&s.tfull[i], 1); mbar_init(&s.tempty[i], kEpiWarps); }
        mbar_init(&s.qbar, 1);
        fence_mbar_init();
        s.prod = s.cons_res = s.closed_at = 0;
        s.closed = 0;
        tma_prefetch(&map_rows);
        tma_prefetch(&map_q);
    }
    if (warp == 1) tmem_alloc<512>(&s.tmem_base);
    const float nqm = __uint_as_float(*a.nq_max);
    const bool force_all = *a.force_all != 0;
    const float nfm = a.nf_max;
    const float sigma = 3.814697265625e-06f * (nqm + nfm) * (nqm + nfm);  // 2^-18 (Nq + Nf)^2
    const float c0 = 1.220703125e-04f * nqm * nfm;                        // 2^-13 Nq Nf
    for (uint32_t q = threadIdx.x; q < kQB; q += blockDim.x) {
        if (q < qn) {
            const float2 m = a.qmeta[q0 + q];  // (RD ||q||^2, RU e_q)
            s.alpha[q] = force_all ? -INFINITY : m.x - 2.f * m.y * nfm - c0 - sigma;
            s.tau[q] = a.g_tau[(size_t)(q0 + q) * a.n_sub + it.sub];
            s.h[q] = h_of(s.alpha[q], s.tau[q]);
        } else {
            s.alpha[q] = INFINITY;  // padded query column: h = +inf, never passes
            s.tau[q] = 0;
            s.h[q] = INFINITY;
        }
        s.lock[q] = 0;
    }
    for (uint32_t i = threadIdx.x; i < kRing; i += blockDim.x) s.seq[i] = i;
    for (uint32_t i = threadIdx.x; i < a.qb * N; i += blockDim.x) lists[i] = kPadKey;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s.tmem_base;

    if (warp == 0) {
        if (lane == 0) {
            // query block (resident B operand): 256 rows x 128 B, one box
            mbar_expect_tx(&s.qbar, a.qb * kK * (uint32_t)sizeof(__half));
            tma_load_2d(s.b, &map_q, &s.qbar, 0, (int)q0);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % kStages;
                if (t >= kStages) mbar_wait_sleep(&s.empty[st], ((t / kStages) - 1) & 1);
                const uint64_t r0 = it.row_begin + (uint64_t)t * kTileRows;
                mbar_expect_tx(&s.full[st], sizeof(s.a[0]) + sizeof(s.rm[0]));
                tma_load_2d(s.a[st], &map_rows, &s.full[st], 0, (int)r0);
                bulk_load(s.rm[st], a.rmeta + (r0 & ~1ull), sizeof(s.rm[0]), &s.full[st]);  // rmeta padded
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = idesc_f16_f32(kTileRows, (int)a.qb_mma);
            mbar_wait(&s.qbar, 0);
            const uint32_t b_base = smem_u32(s.b);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t st = t % kStages, buf = t & 1;
                mbar_wait_sleep(&s.full[st], (t / kStages) & 1);
                if (t >= 2) mbar_wait_sleep(&s.tempty[buf], ((t >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t a_base = smem_u32(s.a[st]);
#pragma unroll
                for (int k = 0; k < ((a.dbg & 2) ? 0 : kK / 16); ++k)
                    mma_f16(tmem + buf * kQB, desc_sw128_kmajor(a_base + k * 32),
                            desc_sw128_kmajor(b_base + k * 32), idesc, k > 0 ? 1u : 0u);
                mma_commit(&s.empty[st]);
                mma_commit(&s.tfull[buf]);
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // ------------------------------------------------------------ epilogue
        // 16 warps: warp -> (TMEM lane quarter, 64 query columns); thread = one row.
        // Per tile: read the 64 accumulator columns, hand the TMEM buffer back at once,
        // then on registers: y_c = RN(D_c - h_c) (FADD2) and max over c (FMNMX3); the
        // row survives for some column iff max_c y_c >= g (cold path, rare).
        const int ew = warp - 2;                  // 0..15
        const uint32_t quarter = warp & 3;        // TMEM lanes 32*quarter ..
        const uint32_t part = ew >> 2;            // columns part*64 .. +64
        const uint32_t ncol = part * 64 < a.qb_mma ? min(64u, a.qb_mma - part * 64) : 0u;
        const uint32_t r_in_tile = quarter * 32 + lane;
        const uint32_t rc = ew * 32 + lane;       // threshold column refreshed by this thread
        uint32_t gt = 0xFFFFFFFFu;                // shared running threshold, loaded one tile ahead
        for (uint32_t t = 0; t < n_tiles; ++t) {
            const uint32_t buf = t & 1, st = t % kStages;
            const uint32_t rl = t * kTileRows + r_in_tile;   // row within the item
            const bool valid = rl < it.count;
            const uint32_t gt_prev = gt;   // loaded 8 tiles ago (latency hidden)
            if ((t & 7) == 0 && rc < qn) gt = __ldcg(&a.g_tau[(size_t)(q0 + rc) * a.n_sub + it.sub]);
            mbar_wait_sleep(&s.tfull[buf], (t >> 1) & 1);    // MMA t done (its stage landed)
            tc_fence_after();
            const float2 m = s.rm[st][r_in_tile + (it.row_begin & 1)];   // (RD ||f||^2, RU e_f)
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.empty[st]);
            const float g = valid ? 0.5f * (m.x - 2.f * nqm * m.y) : INFINITY;
            const uint32_t taddr = tmem + ((quarter * 32) << 16) + buf * kQB + part * 64;
            uint32_t va[32], vb[32];
            if (ncol) {
                tmem_ld32(taddr, va);
                tmem_ld32(taddr + 32, vb);
                tmem_ld_wait_regs(va);   // orders every use of va and vb after the wait
                reg_fence(vb);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s.tempty[buf]);
            if (ncol && !(a.dbg & 1)) {
                const float4 *H4 = reinterpret_cast<const float4 *>(s.h + part * 64);
                float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 h = H4[j];
                    const uint64_t y0 = sub2(pack2(va[4 * j], va[4 * j + 1]), pack2(__float_as_uint(h.x), __float_as_uint(h.y)));
                    const uint64_t y1 = sub2(pack2(va[4 * j + 2], va[4 * j + 3]), pack2(__float_as_uint(h.z), __float_as_uint(h.w)));
                    mx0 = max3f(mx0, __uint_as_float((uint32_t)y0), __uint_as_float((uint32_t)(y0 >> 32)));
                    mx1 = max3f(mx1, __uint_as_float((uint32_t)y1), __uint_as_float((uint32_t)(y1 >> 32)));
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 h = H4[8 + j];
                    const uint64_t y0 = sub2(pack2(vb[4 * j], vb[4 * j + 1]), pack2(__float_as_uint(h.x), __float_as_uint(h.y)));
                    const uint64_t y1 = sub2(pack2(vb[4 * j + 2], vb[4 * j + 3]), pack2(__float_as_uint(h.z), __float_as_uint(h.w)));
                    mx0 = max3f(mx0, __uint_as_float((uint32_t)y0), __uint_as_float((uint32_t)(y0 >> 32)));
                    mx1 = max3f(mx1, __uint_as_float((uint32_t)y1), __uint_as_float((uint32_t)(y1 >> 32)));
                }
                // cold path (rare): enqueue exactly the passing columns
                if (!(a.dbg & 4) && valid && fmaxf(mx0, mx1) >= g) {   // (rows past the item
                    // end have g = +inf, which still passes while h = -inf: hence `valid`)
                    uint32_t spill[64];   // cold path (rare): out of line, via local memory
#pragma unroll
                    for (int j = 0; j < 32; ++j) { spill[j] = va[j]; spill[32 + j] = vb[j]; }
                    tc_cold(s, spill, g, part * 64, qn, rl, a.stat_flagged);
                }
            }
            // the threshold loaded a tile ago: tighten this column if another CTA did better
            if ((t & 7) == 7 && rc < qn && gt_prev < lds_u32(&s.tau[rc])) {
                atomicMin(&s.tau[rc], gt_prev);
                s.h[rc] = h_of(s.alpha[rc], lds_u32(&s.tau[rc]));
            }
        }
        named_bar(1, 32 * kEpiWarps);
        if (warp == 2 && lane == 0) {
            __threadfence_block();
            sts_u32(&s.closed_at, lds_u32(&s.prod));
            __threadfence_block();
            sts_u32(&s.closed, 1u);
        }
    } else {
        // ------------------------------------------------------------ exact re-scoring
        while (true) {
            const unsigned p = atomicAdd(&s.cons_res, 1u);
            uint32_t *sq = &s.seq[p % kRing];
            bool got = false;
            uint32_t idle = 0, nap = 64;
            while (true) {
                if (lds_u32(sq) == p + 1) { got = true; break; }
                if (lds_u32(&s.closed) && p >= lds_u32(&s.closed_at)) break;
                // idle: now and then import the running thresholds other CTAs
                // published (any value ever held is a valid bound, so races only loosen h)
                {
                    const uint32_t qi = (idle++ * (32 * kExactWarps) + (threadIdx.x - 32 * (2 + kEpiWarps))) % kQB;
                    if (qi < qn) {
                        const uint32_t gt = __ldcg(&a.g_tau[(size_t)(q0 + qi) * a.n_sub + it.sub]);
                        if (gt < lds_u32(&s.tau[qi])) {
                            atomicMin(&s.tau[qi], gt);
                            s.h[qi] = h_of(s.alpha[qi], lds_u32(&s.tau[qi]));
                        }
                    }
                }
                __nanosleep(nap);
                if (nap < 2048) nap <<= 1;
            }
            if (!got) break;
            __threadfence_block();
            const uint32_t e = s.val[p % kRing];
            __threadfence_block();
            sts_u32(sq, p + kRing);
            const uint32_t rl = e >> 8, col = e & 0xFF;
            const uint64_t row = it.row_begin + rl;
            const float4 *qv = reinterpret_cast<const float4 *>(a.queries + (size_t)(q0 + col) * kK);
            float acc = 0.f;
            for (uint32_t k4 = 0; k4 < a.kc / 4; ++k4) {
                const float4 x = __ldg(qv + k4);
                const float4 f = __ldg(reinterpret_cast<const float4 *>(a.coarse + coarse_off(row, 4 * k4, a.kc)));
                acc = chain_step_tc(acc, x.x, f.x); acc = chain_step_tc(acc, x.y, f.y);
                acc = chain_step_tc(acc, x.z, f.z); acc = chain_step_tc(acc, x.w, f.w);
            }
            if (a.kc < (uint32_t)kK) {
                const float4 *fr = reinterpret_cast<const float4 *>(a.fine + row * (kK - a.kc));
                for (uint32_t k4 = a.kc / 4; k4 < (uint32_t)kK / 4; ++k4) {
                    const float4 x = __ldg(qv + k4), f = __ldg(fr + k4 - a.kc / 4);
                    acc = chain_step_tc(acc, x.x, f.x); acc = chain_step_tc(acc, x.y, f.y);
                    acc = chain_step_tc(acc, x.z, f.z); acc = chain_step_tc(acc, x.w, f.w);
                }
            }
            const u64 key = ((u64)__float_as_uint(acc) << 32) | (u64)(it.frame_begin + rl);
            u64 *L = lists + (size_t)col * N;
            if (key < lds_u64(&L[N - 1])) {
                while (atomicCAS(&s.lock[col], 0, 1) != 0) __nanosleep(16);
                __threadfence_block();
                if (key < L[N - 1]) {
                    int pidx = (int)N - 1;
                    while (pidx > 0 && L[pidx - 1] > key) { L[pidx] = L[pidx - 1]; --pidx; }
                    L[pidx] = key;
                    if (L[N - 1] != kPadKey) {
                        const uint32_t tb = (uint32_t)(L[N - 1] >> 32);
                        atomicMin(&s.tau[col], tb);
                        s.h[col] = h_of(s.alpha[col], lds_u32(&s.tau[col]));
                        atomicMin(&a.g_tau[(size_t)(q0 + col) * a.n_sub + it.sub], tb);
                    }
                }
                __threadfence_block();
                atomicExch(&s.lock[col], 0);
            }
            if (a.stat_survivors) atomicAdd(a.stat_survivors, 1ull);
        }
    }

    // ---------------------------------------------------------------- teardown
    tc_fence_before();
    __syncthreads();
    if ((a.dbg & 16) && blockIdx.x == 0)
        for (uint32_t q = threadIdx.x; q < kQB; q += blockDim.x) {
            a.prof[16 + q] = __float_as_uint(s.h[q]);
            a.prof[16 + 256 + q] = s.tau[q];
            a.prof[16 + 512 + q] = __float_as_uint(s.alpha[q]);
        }
    if (warp == 1) tmem_dealloc<512>(tmem);
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
__global__ void tc_prep_rows_kernel(const float *coarse, const float *fine, int kc, uint64_t rows,
                                    __half *plane, float2 *rmeta, uint32_t *nf_max, uint32_t *maxabs) {
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
        rmeta[r] = make_float2(fn_lo, ef);
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
                                float2 *rmeta, uint32_t *nf_max, uint32_t *maxabs, cudaStream_t s) {
    uint64_t blocks = (rows + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    tc_prep_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(coarse, fine, kc, rows, (__half *)plane, rmeta, nf_max,
                                                         maxabs);
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

cudaError_t launch_tc_prep_queries(const float *q, uint32_t nq, uint32_t nq_pad, void *q16, float2 *qmeta,
                                   uint32_t *nq_max, uint32_t *force_all, cudaStream_t s) {
    const uint32_t threads = 256, blocks = (nq_pad * 32 + threads - 1) / threads;
    tc_prep_queries_kernel<<<blocks, threads, 0, s>>>(q, nq, nq_pad, (__half *)q16, qmeta, nq_max, force_all);
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

// 2-D map over an fp16 [rows][64] array, box {64, box_rows}, 128-byte swizzle
// (the UMMA K-major SW128 canonical layout).
bool make_tc_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint32_t box_rows) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)kK, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)kK * sizeof(__half)};
    cuuint32_t box[2] = {(cuuint32_t)kK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void *>(ptr), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_tcscan(const CUtensorMap &map_rows, const CUtensorMap &map_q, const TcScanArgs &a, int grid,
                          cudaStream_t s) {
    const size_t smem = tc_smem_bytes(a.qb, a.N);
    cudaError_t e = cudaFuncSetAttribute(tcscan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    tcscan_kernel<<<grid, kTcThreads, smem, s>>>(map_rows, map_q, a);
    return cudaGetLastError();
}

uint32_t tc_max_qb(uint32_t N) {
    const size_t budget = 227 * 1024 - sizeof(TcSmem) - 1024;   // what the top-N lists may use
    uint32_t qb = (uint32_t)(budget / (N * sizeof(u64)));
    qb = qb / 16 * 16;
    if (qb > (uint32_t)kQB) qb = kQB;
    if (qb < 16) qb = 16;
    return qb;
}

}  // namespace ol
