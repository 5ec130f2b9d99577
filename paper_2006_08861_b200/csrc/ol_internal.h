// ol_internal.h -- shared declarations of the omniloc runtime and its kernels.
// Product code only (no oracle, no generator).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../include/omniloc.h"

namespace ol {

typedef unsigned long long u64;

// ---- checked build (-DOL_CHECKED: libomniloc_checked.so, _build.py) ------------------
// compute-sanitizer is closed on this GPU pool, so every kernel states the index
// invariants its global / shared accesses rely on with OL_DCHECK(cond).  In the checked
// library a failed check records (translation unit << 24 | line) of the first failure in
// a device word that ol_get_stat("check") reads back (and the guarded access is skipped);
// in the product library OL_DCHECK is the constant true and generates no code.
#ifndef OL_TU
#define OL_TU 0
#endif
#ifdef OL_CHECKED
static __device__ unsigned int g_ol_check;
__device__ __forceinline__ bool ol_check(bool ok, unsigned line) {
    if (!ok) atomicCAS(&g_ol_check, 0u, ((unsigned)OL_TU << 24) | line);
    return ok;
}
#define OL_DCHECK(cond) ::ol::ol_check((cond), __LINE__)
#define OL_CHECK_EXPORT(fn)                                                        \
    uint32_t fn(bool reset) {                                                      \
        unsigned v = 0, z = 0;                                                     \
        cudaMemcpyFromSymbol(&v, g_ol_check, sizeof(v));                           \
        if (reset) cudaMemcpyToSymbol(g_ol_check, &z, sizeof(z));                  \
        return v;                                                                  \
    }
#else
#define OL_DCHECK(cond) true
#define OL_CHECK_EXPORT(fn) \
    uint32_t fn(bool) { return 0; }
#endif
// first failed check of each translation unit (0 = none); reset clears it
uint32_t check_scan(bool reset);
uint32_t check_merge(bool reset);
uint32_t check_aggregate(bool reset);
uint32_t check_tcscan(bool reset);
uint32_t check_shift(bool reset);
uint32_t check_extract(bool reset);

constexpr int kK = OL_K;
constexpr int kScanThreads = 256;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kMaxQT = 64;            // query frames per scan CTA
constexpr int kAggMax = 8192;         // candidates per bundle in the aggregation kernel
constexpr u64 kPadKey = ~0ull;
// every subspace starts on a 256-row tile of the device planes (padding rows repeat its last
// row): a tensor-core row tile's 32-row block bounds are then one aligned 64-byte copy
constexpr uint64_t kPadRows = 256;
constexpr uint32_t kInfBits = 0x7F800000u;  // +inf: "no threshold yet"

// Coarse plane layout: tiles of 32 rows; inside a tile, 16-byte columns of 4
// coefficients, each column 32 rows x 16 B contiguous.  A warp whose lane i owns
// row (32 t + i) loads 512 contiguous bytes per LDG.128.  Every subspace starts
// on a tile boundary (rows padded to a multiple of 32).
// The fine plane holds every row in full, row-major [rows][64] (round 2: the exact re-scoring
// reads a survivor's first 32 coefficients as one 128-B line, the rest as a second; round 1
// stored only coefficients kc..63 there); the scans' fine passes start at column kc.
__host__ __device__ __forceinline__ uint64_t fine_off(uint64_t row, uint32_t k) { return row * 64ull + k; }
__host__ __device__ __forceinline__ uint64_t coarse_off(uint64_t row, uint32_t k, uint32_t kc) {
    return (((row >> 5) * (kc >> 2) + (k >> 2)) << 7) + ((row & 31) << 2) + (k & 3);
}

// One scan work item: a contiguous run of rows of one subspace.
struct WorkItem {
    uint32_t sub;          // subspace
    uint32_t count;        // rows in this chunk
    uint64_t row_begin;    // first row in the device planes
    uint32_t frame_begin;  // global frame index (within the subspace) of that row
    uint32_t _pad;
};

struct SubInfo {
    uint64_t row_begin;    // first local row of the subspace in the device planes
    uint64_t count;        // local rows (this rank's shard)
    uint32_t shard_begin;  // global frame index of the first local row
    uint32_t global_size;  // |n_i|
    uint32_t chunk_begin;  // first work item of the subspace
    uint32_t chunk_end;
};

struct ScanArgs {
    const float *coarse;         // [rows][kc]
    const float *fine;           // [rows][K] full rows (fine_off)
    const float *queries;        // [nq][K]
    const WorkItem *items;
    uint32_t *tau0;              // [nq][n_sub] acc bits (seeded; shared running minimum), or null
    u64 *partial;                // [nq][n_items][N]
    unsigned long long *stat_survivors;  // may be null
    uint32_t nq, n_items, n_qtiles, qt, n_sub, N;
    uint64_t rows_pad;           // device rows (bounds checks)
};

struct SeedArgs {
    const float *coarse, *fine, *queries;
    const SubInfo *subs;
    uint32_t *tau0;              // [nq][n_sub]
    uint32_t nq, n_sub, N, samples, kc, splits;   // splits: independent samples per (frame, sub)
    uint32_t *scratch;           // [nq][n_sub][splits][samples] acc bits (seed_acc -> seed_select)
    uint64_t rows_pad;           // device rows (bounds checks)
    uint32_t select_old = 0;     // 1: the CTA / radix selects even where the warp gather applies (tests, A/B)
};

struct MergeArgs {
    const u64 *partial;          // [nq][n_items][N]
    const SubInfo *subs;
    const int32_t *coords;       // [rows][2]
    uint4 *records;              // [nq][n_sub][N]
    uint32_t nq, n_items, n_sub, N;
    // world 1: also write the candidate rows (candidates_kernel's output) when non-null
    ol_candidate *cand;
    const uint32_t *sub_prefix;  // [n_sub+1] prefix of min(N, |n_i|)
    uint32_t M;
    uint64_t n_cand;             // candidate rows (bounds checks)
    uint32_t max_lists;          // the most work items of one subspace (launch shape)
    uint32_t buf_cap;            // (set by launch_merge_chunks)
    uint32_t force_scan;         // tests: always the N-round scan over all keys (the fallback)
};

struct RankMergeArgs {
    const uint4 *gathered;       // [world][nq][n_sub][N]
    uint4 *records;              // [nq][n_sub][N]
    uint32_t nq, n_sub, N, world;
};

constexpr int kXchgMax = 8;   // ranks of the peer-memory exchange (one NVSwitch node)
static_assert(kXchgMax - 1 <= 7, "TcScanArgs::peer_tau");
constexpr uint32_t kXchgBlocks = 16;   // blocks per rank of xchg_merge_kernel (fixed: the arrival counters count them)

struct XchgArgs {
    uint4 *mbox[kXchgMax];        // rank p's mailbox records: [2 (epoch parity)][world][nq][n_sub][N]
    unsigned int *flag[kXchgMax]; // rank p's arrival counters [world] (monotonic: epoch x blocks)
    const uint4 *payload[kXchgMax];   // group g's own payload [nq][n_sub][N]
    uint4 *records[kXchgMax];     // group g's merged output [nq][n_sub][N]
    uint32_t rank0, world, blocks, epoch;
    uint32_t nq, n_sub, N;
};

struct CandArgs {
    const uint4 *records;        // [nq][n_sub][N]
    const uint32_t *sub_prefix;  // [n_sub+1] prefix of min(N, |n_i|)
    ol_candidate *out;
    uint32_t nq, n_sub, N, M;
    uint64_t n_cand;             // candidate rows (bounds checks)
};

struct AggArgs {
    const ol_candidate *cand;    // if non-null: bundle b = cand[b*per .. (b+1)*per)
    uint32_t per_bundle;
    const uint32_t *offsets;     // else: xy pairs with offsets
    const int32_t *xy;
    ol_estimate *out;            // device
    int *err_empty;              // device flag
    uint32_t n_bundles, top_c;
    double toler_per, r2, tile_m;
    uint32_t cap;                // power of two >= every bundle's size (<= kAggMax); 0 = kAggMax
    uint32_t block_only = 0;     // 1: the CTA-wide version for small bundles too (tests: both agree)
};

// NK10: one kernel for a whole small world-1 query (aggregate.cu)
struct MicroArgs {
    const float *coarse, *fine, *queries;   // planes, frames [nq][K]
    const SubInfo *subs;
    const int32_t *coords;
    const uint32_t *sub_prefix;             // [n_sub+1] prefix of min(N, |n_i|)
    ol_candidate *cand;
    uint32_t *bundle_count;                 // [n_bundles] zeroed; each last job resets its own
    uint32_t split;                         // CTAs per (frame, subspace) job: the cluster size, 1..8
    int *flag_nonfinite;
    uint32_t nq, n_sub, N, M, kc;
    int check_finite, aggregate;
    AggArgs agg;                            // cand / per_bundle / out / params of Algorithm 2
    unsigned long long *prof;               // profiling only (tc_debug & 32): phase cycles, or null
};
// tensor-core scan: inline re-scoring when the subspaces average at most this many rows -- many
// small subspaces (per-subspace top-N) leave 0.5-3 % of pairs to the exact path, which the two
// exact warps cannot absorb (C2, 4,000 rows: 1.61 -> 1.00 ms; C3 split 50 ways, 20,000: 3.07 ->
// 2.51 ms); with 200,000 (C3 in 5) or more rows per subspace the queue wins (0.82 vs 1.33 ms)
constexpr uint64_t kInlineMaxRowsPerSub = 65536;
constexpr uint64_t kMicroMaxRows = 8192;    // per subspace (64 KB of keys in shared memory)
constexpr uint64_t kMicroMaxPairs = 1u << 16;   // frames x rows of the whole query
size_t micro_smem_bytes(uint64_t max_rows, uint32_t split, uint32_t N, uint32_t agg_cap);
uint32_t micro_split(uint64_t max_rows, uint64_t jobs);
cudaError_t launch_micro(const MicroArgs &a, size_t smem, cudaStream_t s);

struct TcScanArgs {
    const WorkItem *items;
    const float2 *blk;            // [rows_pad / 32] per 32-row block: (min RD||f||^2/2, max RU e_f)
    const float4 *qmeta;          // [nq] (RD ||q||^2, RU ||q - fp16(q)||, RU ||q||^2, 0)
    const uint32_t *bounds;       // [2] batch norm bound bits, [3] force_all (a frame left the fp16 range),
                                  // [4] max RU||f||^2/2 bits, [5] max RU e_f bits (bound pre-pass)
    float nf_max;                 // database norm bound
    uint32_t *g_tau;              // [nq][n_sub] acc bits: seeded, then shared running minimum
    const float *queries;         // fp32 [nq][K]
    const float *coarse, *fine;   // fp32 planes (exact re-scoring)
    u64 *partial;                 // [nq][n_items][N] (unused by the bound pre-pass)
    uint32_t bound;               // 1: bound pre-pass over a strided row view (items index that view)
    uint32_t cluster;             // CTAs per thread-block cluster (query blocks of one item); 0/1 = none
    uint32_t pair;                // 1: CTA pairs (cta_group::2, M = 256) over query-block pairs; n_qblocks even
    unsigned long long *stat_survivors;
    unsigned long long *stat_flagged;   // (frame, row tile) pairs that took the cold path
    uint32_t nq, n_items, n_qblocks, qb, n_sub, N, kc, stages;
    uint32_t inline_rescore;      // 1: the epilogue warps re-score their own survivors (short items: C2-like)
    uint32_t dbg;                 // profiling only: 1 skip epilogue math, 2 skip MMA, 4 skip cold path, 8 drop
                                  // survivors, 16 / 32 counters, 64 keep the last thresholds, 128 stale rows,
                                  // 256 no threshold refresh
    uint32_t n_blk;               // rows_pad / 32
    uint32_t kf;                  // filter on the first kf of K dimensions (16..64, multiple of 16)
    uint32_t pw;                  // fp16 plane / frame row width in halves: 64 (128-B rows, SW128) or 32 (kf = 32: 64-B rows, SW64)
    unsigned long long *prof;     // [16] per-role cycle counters when dbg & 32 (profiling only)
    // other ranks' threshold arrays (same [nq][n_sub] layout, peer memory over NVLink): every
    // threshold this CTA publishes is also MIN-ed into them (each is a valid bound for every
    // rank: the N-th best of N real rows of the subspace), so small shards converge like the
    // whole database would
    uint32_t *peer_tau[7];
    uint32_t n_peer;
};

constexpr u64 kShiftPad = 0x7FFFFFFFFFFFFFFFull;   // "not scored on this rank" (MIN-reducible)

struct ShiftArgs {
    const ol_candidate *cand;
    const SubInfo *subs;
    const float *prof;            // [rows][W] database profiles (tile-padded row index)
    const float *cprof;           // or, when non-null: [n_cand][W] profiles in candidate order
    const float *qprof;           // [nq][W] query profiles
    u64 *keys;                    // [n_cand]
    uint64_t n_cand;
    uint32_t W, M;
    uint32_t nq;                  // query frames (bounds checks)
};

// launchers (return cudaGetLastError())
cudaError_t launch_shift(const ShiftArgs &a, cudaStream_t s);
cudaError_t launch_tc_prep_rows(const float *coarse, const float *fine, int kc, uint64_t rows, void *plane,
                                float2 *blk, uint32_t *stat, uint32_t kf, uint32_t pw, cudaStream_t s);
cudaError_t launch_tc_prep_queries(const float *q, uint32_t nq, uint32_t nq_pad, void *q16, float4 *qmeta,
                                   uint32_t *bounds, uint32_t kf, uint32_t pw, cudaStream_t s);
cudaError_t launch_fill_u32(uint32_t *p, uint64_t n, uint32_t v, cudaStream_t s);
size_t extract_smem_bytes(uint32_t W);
cudaError_t launch_extract(const double *prof, uint64_t n, uint32_t W, float *out32, double *out64,
                           uint8_t *degenerate, float *prof_out, cudaStream_t s);
cudaError_t launch_pad_rows(const SubInfo *subs, uint32_t n_sub, int kc, float *coarse, float *fine, cudaStream_t s);
bool make_tc_map(CUtensorMap *m, const void *ptr, uint64_t rows, uint32_t box_rows, uint32_t width,
                 uint32_t row_stride = 1);
cudaError_t launch_tcscan(const CUtensorMap &map_rows, const CUtensorMap &map_q, const TcScanArgs &a, int grid,
                          cudaStream_t s);
size_t tc_smem_bytes(uint32_t qb, uint32_t N, uint32_t stages, uint32_t pw);
bool tc_shape(uint32_t N, uint32_t nq, uint32_t pw, uint32_t *qb, uint32_t *stages);
cudaError_t launch_tau_seed(const SeedArgs &a, cudaStream_t s);
cudaError_t launch_scan(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s);
size_t scan_smem_bytes(uint32_t qt, uint32_t N);
cudaError_t launch_scan2(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s);
size_t scan2_smem_bytes(uint32_t qt, uint32_t N, int kc);
cudaError_t launch_scan3(int kc, const ScanArgs &a, size_t smem, int grid, cudaStream_t s);
size_t scan3_smem_bytes(uint32_t qt, uint32_t N, int kc);
cudaError_t launch_merge_chunks(const MergeArgs &a, cudaStream_t s);
cudaError_t launch_merge_ranks(const RankMergeArgs &a, cudaStream_t s);
cudaError_t launch_xchg_merge(const XchgArgs &a, uint32_t groups, cudaStream_t s);
cudaError_t launch_candidates(const CandArgs &a, cudaStream_t s);
cudaError_t launch_aggregate(const AggArgs &a, cudaStream_t s);
cudaError_t launch_check_finite(const float *p, uint64_t n, int *flag, cudaStream_t s);
cudaError_t launch_relayout(const float *src, uint64_t rows, uint64_t dst_row0, int kc, float *coarse,
                            float *fine, cudaStream_t s);
// flag = 1 if any (x, y) lies outside [x0, x1) x [y0, y1)
cudaError_t launch_check_coords(const int32_t *xy, uint64_t rows, int32_t x0, int32_t x1, int32_t y0,
                                int32_t y1, int *flag, cudaStream_t s);

// ---- warp / block selection of the smallest unique u64 keys (NK4 merges, NK10)
// one key per lane -> the warp's 32 keys ascending across the lanes (bitonic network)
__device__ __forceinline__ u64 warp_sort32(u64 k, int lane) {
#pragma unroll
    for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
            const u64 o = __shfl_xor_sync(0xffffffffu, k, j);
            const bool keep_min = ((lane & j) == 0) == ((lane & kk) == 0);
            k = keep_min ? (o < k ? o : k) : (o > k ? o : k);
        }
    }
    return k;
}
// two ascending 32-key warp lists -> the 32 smallest of both, ascending: min(a_i, b_{31-i})
// is the lower half of the bitonic merge of a with b reversed, then 5 half-cleaner steps
__device__ __forceinline__ u64 warp_merge32(u64 a, u64 b, int lane) {
    const u64 br = __shfl_sync(0xffffffffu, b, 31 - lane);
    u64 v = a < br ? a : br;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const u64 o = __shfl_xor_sync(0xffffffffu, v, j);
        v = (lane & j) == 0 ? (o < v ? o : v) : (o > v ? o : v);
    }
    return v;
}

// The c <= 32 smallest of keys[0..n) (shared memory), ascending, into sel[0..c), by the whole
// CTA: every warp folds its 32-key chunks into a running sorted 32-list (sort, merge), then
// the warps' lists are merged pairwise in log2(warps) rounds (scratch: 32 per warp).  Keys
// are unique, so this is the same set and order as c rounds of "the minimum above the last".
__device__ inline void block_select32(const u64 *keys, uint32_t n, uint32_t c, u64 *sel, u64 *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    u64 run = kPadKey;
    for (uint32_t base = 32u * warp; base < n; base += 32u * nw) {
        const u64 v = base + lane < n ? keys[base + lane] : kPadKey;
        run = warp_merge32(run, warp_sort32(v, lane), lane);
    }
    for (int st = 1; st < nw; st <<= 1) {
        scratch[warp * 32 + lane] = run;
        __syncthreads();
        if (warp % (2 * st) == 0 && warp + st < nw) run = warp_merge32(run, scratch[(warp + st) * 32 + lane], lane);
        __syncthreads();
    }
    if (warp == 0 && (uint32_t)lane < c) sel[lane] = run;
}

}  // namespace ol
