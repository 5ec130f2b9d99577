// shift.cu -- NEXT-1 (kernel NK7): shift-resolved re-scoring of the
// final candidates.  For candidate (query frame q, database row p) the minimum
// over circular shifts s of the fp32 chain sum_w (q[(w+s) mod W] - p[w])^2
// (w in order, RN subtract + fused multiply-add, as the descriptor distance,
// DESIGN R3/R21) and its smallest argmin: the camera heading difference.  The
// descriptor (FFT magnitude) is rotation invariant; this step recovers the
// rotation it discards.  One warp per candidate: the two profiles in shared
// memory, lane l scores shifts l, l+32, ...; a warp min over (acc bits, s) keys.
#define OL_TU 5
#include "ol_internal.h"

namespace ol {

constexpr int kShiftWarps = 8;

__global__ void __launch_bounds__(32 * kShiftWarps) shift_kernel(ShiftArgs a) {
    extern __shared__ float sh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t c = (uint64_t)blockIdx.x * kShiftWarps + warp;
    if (c >= a.n_cand) return;
    const uint32_t W = a.W;
    float *q = sh + (size_t)warp * 2 * W, *p = q + W;
    const ol_candidate cd = a.cand[c];
    const float *ps;
    if (a.cprof) {   // the caller supplied every candidate's database profile, in candidate order
        ps = a.cprof + c * W;
    } else {
        const SubInfo si = a.subs[cd.subspace];
        if (cd.frame < si.shard_begin || cd.frame >= si.shard_begin + si.count) {
            if (lane == 0) a.keys[c] = kShiftPad;   // another rank owns this frame
            return;
        }
        ps = a.prof + (si.row_begin + (cd.frame - si.shard_begin)) * W;
    }
    if (!OL_DCHECK((uint64_t)cd.bundle * a.M + cd.query_frame < a.nq && cd.query_frame < a.M)) return;
    const float *qs = a.qprof + ((uint64_t)cd.bundle * a.M + cd.query_frame) * W;
    for (uint32_t w = lane; w < W; w += 32) { q[w] = qs[w]; p[w] = ps[w]; }
    __syncwarp();
    u64 best = ~0ull;
    for (uint32_t s = lane; s < W; s += 32) {
        float acc = 0.f;
        uint32_t i = s;
        for (uint32_t w = 0; w < W; ++w) {
            const float d = __fsub_rn(q[i], p[w]);
            acc = __fmaf_rn(d, d, acc);
            if (++i == W) i = 0;
        }
        const u64 key = ((u64)__float_as_uint(acc) << 32) | s;
        best = key < best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if (lane == 0) a.keys[c] = best;
}

// W = 32 * SPL (SPL shifts per lane, lane l owns shifts SPL l .. SPL l + SPL - 1): the query
// profile duplicated in shared memory (q2 = q ++ q, no index wrap), and per 4 columns each lane
// loads the 4 + SPL - 1 query values its SPL chains need with 128-bit loads and the 4 database
// values (broadcast), then advances SPL chains by 4 steps: ~2.1 instructions per chain step
// instead of ~7.  Same chains in the same order as shift_kernel, so the same keys.
template <int SPL>
__global__ void __launch_bounds__(32 * kShiftWarps) shift_fast_kernel(ShiftArgs a) {
    constexpr uint32_t W = 32u * SPL;
    __shared__ __align__(16) float sq[kShiftWarps][2 * W + 16];
    __shared__ __align__(16) float sp[kShiftWarps][W];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t c = (uint64_t)blockIdx.x * kShiftWarps + warp;
    if (c >= a.n_cand) return;
    const ol_candidate cd = a.cand[c];
    const float *ps;
    if (a.cprof) {
        ps = a.cprof + c * W;
    } else {
        const SubInfo si = a.subs[cd.subspace];
        if (cd.frame < si.shard_begin || cd.frame >= si.shard_begin + si.count) {
            if (lane == 0) a.keys[c] = kShiftPad;   // another rank owns this frame
            return;
        }
        ps = a.prof + (si.row_begin + (cd.frame - si.shard_begin)) * W;
    }
    if (!OL_DCHECK((uint64_t)cd.bundle * a.M + cd.query_frame < a.nq && cd.query_frame < a.M)) return;
    const float *qs = a.qprof + ((uint64_t)cd.bundle * a.M + cd.query_frame) * W;
    float *q2 = sq[warp], *p = sp[warp];
    for (uint32_t w = lane; w < W; w += 32) { const float v = qs[w]; q2[w] = v; q2[w + W] = v; p[w] = ps[w]; }
    if (lane < 16) q2[2 * W + lane] = 0.f;
    __syncwarp();
    float acc[SPL];
#pragma unroll
    for (int j = 0; j < SPL; ++j) acc[j] = 0.f;
    const uint32_t s0 = (uint32_t)lane * SPL;
    for (uint32_t w = 0; w < W; w += 4) {
        // q2[w + s0 + j + t] for j < SPL, t < 4: SPL + 3 values from a 16-byte aligned start
        float qv[SPL + 4];
        const float4 *src = reinterpret_cast<const float4 *>(q2 + w + s0);
#pragma unroll
        for (int v = 0; v < (SPL + 4) / 4; ++v) {
            const float4 x = src[v];
            qv[4 * v] = x.x; qv[4 * v + 1] = x.y; qv[4 * v + 2] = x.z; qv[4 * v + 3] = x.w;
        }
        const float4 pv = *reinterpret_cast<const float4 *>(p + w);
        const float pw[4] = {pv.x, pv.y, pv.z, pv.w};
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int j = 0; j < SPL; ++j) {
                const float d = __fsub_rn(qv[j + t], pw[t]);
                acc[j] = __fmaf_rn(d, d, acc[j]);
            }
    }
    u64 best = ~0ull;
#pragma unroll
    for (int j = 0; j < SPL; ++j) {
        const u64 key = ((u64)__float_as_uint(acc[j]) << 32) | (s0 + j);
        best = key < best ? key : best;
    }
    for (int o = 16; o; o >>= 1) {
        const u64 other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if (lane == 0) a.keys[c] = best;
}

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
    if (a.W == 256) {   // the paper-shaped profile width: the register-blocked kernel
        const uint64_t blocks = (a.n_cand + kShiftWarps - 1) / kShiftWarps;
        shift_fast_kernel<8><<<(unsigned)(blocks ? blocks : 1), 32 * kShiftWarps, 0, s>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = sizeof(float) * 2 * a.W * kShiftWarps;
    cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t blocks = (a.n_cand + kShiftWarps - 1) / kShiftWarps;
    shift_kernel<<<(unsigned)(blocks ? blocks : 1), 32 * kShiftWarps, smem, s>>>(a);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_shift)

}  // namespace ol
