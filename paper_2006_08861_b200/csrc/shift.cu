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

cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s) {
    const size_t smem = sizeof(float) * 2 * a.W * kShiftWarps;
    cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const uint64_t blocks = (a.n_cand + kShiftWarps - 1) / kShiftWarps;
    shift_kernel<<<(unsigned)(blocks ? blocks : 1), 32 * kShiftWarps, smem, s>>>(a);
    return cudaGetLastError();
}

OL_CHECK_EXPORT(check_shift)

}  // namespace ol
