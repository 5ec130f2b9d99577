/*
 * omniloc.h -- C-ABI of the B200-native hot path of arXiv 2006.08861
 * ("GPU-accelerated Hierarchical Panoramic Image Feature Retrieval for Indoor
 * Localization", Hu, Zhu, Zhang, ICMR'16).
 *
 * The library retrieves, for every query frame and every database subspace,
 * the N database descriptors nearest in Euclidean distance (P:139, P:157,
 * P:162; Algorithm 1) and fuses each M-frame bundle's candidates into
 * one floor-plan tile with the 2-D multi-frame aggregation (
 * Algorithm 2).  Everything runs in hand-written sm_100a kernels; there is no
 * CPU fallback.  The database may be sharded over ranks (one process per GPU);
 * ranks then exchange their per-rank top-N (see ol_payload / ol_finalize).
 *
 * Citation key: P:n = PAPER.md line n; S:n = SPEC.md line n; R<k> = DESIGN.md
 * reading k.
 *
 * Conventions for every entry point:
 *   - returns ol_status: OL_OK (0) or a negative OL_ERR_* code; no exception
 *     ever crosses the ABI.  ol_last_error(ctx) gives a one-line message.
 *   - "device" pointers are CUDA global-memory pointers on the context's
 *     device; "host" pointers are ordinary (pageable or pinned) memory.
 *   - all device work is ordered on the context's stream (borrowed from the
 *     caller); calls are not thread-safe per context.
 *
 * Numeric contract (R3): descriptors and queries are fp32.  For a query q and
 * a database row f the library computes acc = squared distance by the fixed
 * chain  acc = +0;  for k = 0..K-1: d = RN32(q_k - f_k); acc = fma32(d, d, acc),
 * reports dist = RN32(sqrt(acc)), and ranks by (acc, frame index).  Results are
 * bit-identical to a sequential scan for any launch shape, shard count or
 * pruning threshold (the coarse/fine hierarchy, R2, is exact).
 */
#ifndef OMNILOC_H
#define OMNILOC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define OL_API __attribute__((visibility("default")))
#else
#define OL_API
#endif

typedef int32_t ol_status;

#define OL_OK                       0
#define OL_ERR_INVALID_ARGUMENT    (-1)  /* a parameter outside its documented range   */
#define OL_ERR_DIMENSION_MISMATCH  (-2)  /* K != 64                              */
#define OL_ERR_NONFINITE           (-3)  /* NaN/Inf in features or frames        */
#define OL_ERR_OUT_OF_RANGE        (-4)  /* tile outside the grid, m>=n  */
#define OL_ERR_OOM                 (-5)  /* cudaMalloc failed                           */
#define OL_ERR_CUDA                (-6)  /* any other CUDA runtime error                */
#define OL_ERR_NOT_READY           (-7)  /* query before upload / get before query      */
#define OL_ERR_EMPTY               (-8)  /* a bundle with no candidates, or no
                                            estimates because aggregation was off      */
#define OL_ERR_NCCL                (-9)  /* NCCL missing, or a communicator error       */

#define OL_NCCL_ID_BYTES 128  /* ncclUniqueId */

#define OL_K 64           /* descriptor length: |DFT| bins 1..64       */
#define OL_MAX_N 128      /* largest supported top-N per (frame, subspace)          */
#define OL_MAX_TOP_C 64   /* largest supported TopC (P:197 uses 10)                 */
#define OL_MAX_M 64       /* largest bundle                                 */

typedef struct ol_ctx ol_ctx;

/* Context configuration (ol_create). */
typedef struct {
    int32_t device;        /* CUDA device ordinal                                   */
    int32_t rank, world;   /* this process's shard index and the shard count (>=1)  */
    void *cuda_stream;     /* cudaStream_t to borrow (e.g. torch's current stream);
                              NULL = the CUDA legacy default stream.  The library
                              never creates or destroys streams.               */
    uint32_t K;            /* must be OL_K                                           */
    uint32_t coarse_k;     /* prefix length of the coarse pass (R2): 0 or 64 = one
                              pass over full rows; 8, 16 or 32 = exact coarse/fine  */
    const void *nccl_unique_id;  /* OL_NCCL_ID_BYTES from ol_nccl_unique_id() on one rank,
                              broadcast to all (e.g. torch.distributed); NULL = no
                              communicator.  With an id, ol_create is collective over
                              `world` ranks and the context owns a NCCL communicator:
                              ol_query then exchanges and merges the per-rank top-N
                              itself.  Allowed at world 1 (a 1-rank
                              communicator: the same code path).                  */
} ol_config;

/* Database to upload (ol_upload_db).  The database is n_subspaces independent
 * subspaces ("each floor data is counted as one subspace"; "the n_i
 * subspace has |n_i| modeled frames").  This rank holds, for every subspace i,
 * the contiguous slice of frames [shard_begin[i], shard_begin[i]+shard_count[i])
 * of its global_sizes[i] frames; features/coords hold those slices back to back
 * in subspace order.  Frame indices in results are global within a subspace. */
typedef struct {
    uint32_t n_subspaces;
    const uint64_t *global_sizes;  /* [n_subspaces] |n_i| >= 1 (host)               */
    const uint64_t *shard_begin;   /* [n_subspaces] (host); NULL together with
                                      shard_count -> the library takes the equal
                                      contiguous slice r of world (ol_shard_range) */
    const uint64_t *shard_count;   /* [n_subspaces] (host) or NULL                  */
    const float *features;         /* [sum shard_count][K] fp32 row-major           */
    const int32_t *coords;         /* [sum shard_count][2] (x, y) 30 cm tiles*/
    int32_t grid_w, grid_h;        /* tile grid; every coord must satisfy
                                      0 <= x < grid_w, 0 <= y < grid_h     */
    int32_t on_device;             /* 1: features/coords are device pointers         */
} ol_db_desc;

/* Retrieval + aggregation parameters. */
typedef struct {
    uint32_t N;          /* top-N per (query frame, subspace), 1..OL_MAX_N (15) */
    uint32_t top_c;      /* TopC tiles scanned, 1..OL_MAX_TOP_C (10)             */
    double toler_per;    /* acceptance fraction in (0, 1] (0.2)                  */
    double radius_m;     /* tolerance-circle radius in metres, > 0 (3)           */
    double tile_m;       /* tile edge in metres, > 0 (0.30)                      */
} ol_params;

/* One retrieval hit. 32 bytes. */
typedef struct {
    uint32_t subspace;     /* subspace index i (0-based)                             */
    uint32_t frame;        /* global frame index t within subspace i (0-based)      */
    uint32_t bundle;       /* bundle index                                           */
    uint32_t query_frame;  /* frame index within the bundle, 0..M-1                 */
    float dist2;           /* acc, the fp32 squared distance (R3)                    */
    float dist;            /* RN32(sqrt(acc))                                        */
    int32_t x, y;          /* the frame's floor tile (geo-referenced table)  */
} ol_candidate;

typedef struct {
    int32_t x, y;
    uint32_t count;        /* candidates binned in this tile (Alg. 2 step 2)         */
    uint32_t circle;       /* candidates within the tolerance circle         */
} ol_ranked_tile;

/* Aggregated location of one bundle (Algorithm 2). */
typedef struct {
    int32_t x, y;              /* FinalPosition tile                                  */
    double x_m, y_m;           /* tile_m * (x, y): tile centre in metres      */
    double confidence;         /* circle / total (binary64 division)                  */
    uint32_t low_confidence;   /* 1 if no ranked tile passed (fallback) */
    uint32_t n_ranked;         /* min(top_c, distinct tiles)                          */
    uint32_t total;            /* candidates in the bundle                            */
    uint32_t _pad;
    ol_ranked_tile ranked[OL_MAX_TOP_C];
} ol_estimate;

/* ---- lifetime ------------------------------------------------------------ */

/* Create a context on cfg->device.  Errors: INVALID_ARGUMENT (world < 1, rank
 * outside [0, world), coarse_k not in {0, 8, 16, 32, 64}), DIMENSION_MISMATCH
 * (K != 64), CUDA, NCCL (cfg->nccl_unique_id set and NCCL cannot be loaded or
 * ncclCommInitRank fails).  On error *out is NULL and ol_last_error(NULL)
 * explains. */
OL_API ol_status ol_create(const ol_config *cfg, ol_ctx **out);

/* A fresh NCCL unique id (OL_NCCL_ID_BYTES bytes written to out) for
 * ol_config.nccl_unique_id: one rank creates it and sends it to the others by any
 * means.  Pure host function; loads NCCL on first use ("libnccl.so.2", or the path
 * in $OL_NCCL_LIB).  Errors: INVALID_ARGUMENT (NULL), NCCL. */
OL_API ol_status ol_nccl_unique_id(void *out);

/* Free all device/host resources of the context, the NCCL communicator included
 * (aborted if it is in an error state).  NULL is a no-op. */
OL_API void ol_destroy(ol_ctx *ctx);

/* Replace the stream all later calls are ordered on (borrowed; NULL = the
 * legacy default stream). */
OL_API ol_status ol_set_stream(ol_ctx *ctx, void *cuda_stream);

/* Last error message of ctx (or of the calling thread if ctx is NULL). Never NULL. */
OL_API const char *ol_last_error(const ol_ctx *ctx);

/* The contiguous slice [begin, begin+count) of a subspace of `global_size`
 * frames owned by `rank` of `world`: begin = floor(rank*size/world).  Pure host
 * function.  Errors: INVALID_ARGUMENT (world < 1 or rank >= world). */
OL_API ol_status ol_shard_range(uint64_t global_size, int32_t rank, int32_t world, uint64_t *begin,
                         uint64_t *count);

/* ---- database ------------------------------------------------------------ */

/* Copy (and re-lay out) the database into device memory owned by the context;
 * replaces any previous database.  Synchronous.  Errors: INVALID_ARGUMENT
 * (n_subspaces = 0, a size 0, shard outside its subspace, grid <= 0),
 * NONFINITE, OUT_OF_RANGE (coord outside the grid), OOM, CUDA. */
OL_API ol_status ol_upload_db(ol_ctx *ctx, const ol_db_desc *db);

/* ---- query --------------------------------------------------------------- */

/* Retrieve the top-N of every (bundle, frame, subspace) (Alg. 1) and,
 * if `aggregate`, fuse every bundle (Alg. 2).  frames: [n_bundles][M][K] fp32,
 * host or device (on_device).  Asynchronous on the context stream: a host
 * `frames` buffer is read before return; results stay valid until the next
 * ol_query.  With world > 1:
 *   - context with a NCCL communicator (ol_config.nccl_unique_id): the call is
 *     collective -- every rank calls it with identical arguments -- and it does the
 *     whole cross-GPU step on the context stream: a MIN all-reduce of the seeded
 *     thresholds before the scan (each rank's seed bounds the global N-th best, so
 *     the least one is still exact), then an all-gather of the per-rank top-N
 *     records and their merge.  Every rank ends with the global results.
 *   - without a communicator it produces only this rank's top-N (the "payload");
 *     the caller all-gathers payloads and calls ol_finalize (or ol_p2p_finalize).
 * Errors: NOT_READY (no database), INVALID_ARGUMENT (n_bundles = 0, M even or
 * 0 or > OL_MAX_M, N = 0 or > OL_MAX_N, top_c = 0 or > OL_MAX_TOP_C,
 * toler_per outside (0, 1], radius_m <= 0, tile_m <= 0, a bundle with more than
 * 8192 candidates when aggregating), NONFINITE (host frames; device frames
 * are checked on the device and reported by the next ol_get_*), OOM, CUDA,
 * NCCL (a collective failed to enqueue, or the communicator reports an
 * asynchronous error; ol_get_* poll it as well). */
OL_API ol_status ol_query(ol_ctx *ctx, uint32_t n_bundles, uint32_t M, const float *frames,
                   int32_t on_device, const ol_params *p, int32_t aggregate);

/* This rank's per-(frame, subspace) top-N as 16-byte records
 * {u32 acc_bits, u32 frame, i32 x, i32 y} in [frame][subspace][N] order, padded
 * with acc_bits = frame = 0xFFFFFFFF.  *dev_ptr is owned by the context. */
OL_API ol_status ol_payload(ol_ctx *ctx, const void **dev_ptr, uint64_t *bytes);

/* Copy this rank's payload (ol_payload) to `dst` (device memory, at least the
 * payload's bytes), stream-ordered; e.g. into a buffer the caller all-gathers. */
OL_API ol_status ol_payload_copy(ol_ctx *ctx, void *dst);

/* Merge `world` payloads gathered back to back at `gathered` (device, world *
 * payload bytes, rank order) into the global top-N, then build candidates and
 * (if requested in ol_query) estimates.  Identical on every rank.  Errors:
 * NOT_READY (no preceding ol_query), INVALID_ARGUMENT (world mismatch), CUDA. */
OL_API ol_status ol_finalize(ol_ctx *ctx, const void *gathered, int32_t world);

/* The pruning thresholds of the last query: [frames][subspace] acc bits (fp32, ordered
 * as unsigned), owned by the context, valid until the next ol_query.  Before the scan
 * they hold the seed (an upper bound of the N-th smallest acc of every (frame,
 * subspace)); after it, the running minimum the scan converged to.  Introspection and
 * multi-rank experiments (option "tc_debug" 512 stops ol_query after the seed; 64 makes
 * the next ol_query start from the values found here instead of seeding -- exact only if
 * they are such upper bounds).  Errors: INVALID_ARGUMENT, NOT_READY. */
OL_API ol_status ol_thresholds(ol_ctx *ctx, void **dev_ptr, uint64_t *count);

/* ---- peer-memory exchange (NVLink / NVSwitch, one node) --------------------
 * The cross-GPU step as one kernel instead of an NCCL all-gather +
 * ol_finalize: every rank stores its payload straight into slot `rank` of every
 * rank's mailbox over peer memory, signals each receiver (system-scope release
 * counter), waits for all ranks' slots in its own mailbox and merges them into
 * the global top-N; then candidates and estimates as ol_finalize.  Identical
 * results to ol_finalize on every rank.  Collective: every rank calls each of
 * these in the same order. */

/* Allocate this rank's mailbox (2 x world x max_payload_bytes + 256 B of
 * counters; max_payload_bytes >= the ol_payload bytes of every later query, a
 * multiple of 16) and write its CUDA IPC handle (64 bytes) to handle_out (may be
 * NULL when the caller emulates ranks on one GPU).  1 <= world <= 8.  Replaces
 * an earlier mailbox.  Errors: INVALID_ARGUMENT, OOM, CUDA. */
OL_API ol_status ol_p2p_open(ol_ctx *ctx, int32_t world, int32_t rank, uint64_t max_payload_bytes,
                             void *handle_out);

/* Open every other rank's mailbox: `handles` = world x 64 bytes in rank order
 * (the caller all-gathers the ol_p2p_open handles, e.g. over torch.distributed).
 * Errors: NOT_READY (no ol_p2p_open), INVALID_ARGUMENT, CUDA (IPC unavailable). */
OL_API ol_status ol_p2p_connect(ol_ctx *ctx, const void *handles);

/* After ol_query on every rank: exchange + merge + candidates (+ estimates), one
 * cooperative kernel for the exchange and merge, stream-ordered.  Errors:
 * NOT_READY (no query / not connected), INVALID_ARGUMENT (payload larger than
 * the mailbox), CUDA. */
OL_API ol_status ol_p2p_finalize(ol_ctx *ctx);

/* Tests: the same kernel emulating `world` ranks on ONE GPU as one cooperative
 * launch (group g = rank g, mailboxes local): ctxs[g] opened with
 * ol_p2p_open(world, g, ..), each after its ol_query.  Synchronises. */
OL_API ol_status ol_p2p_emulate(ol_ctx **ctxs, int32_t world);

/* Tests / measurements: link `world` contexts on ONE device as if they were ranks sharing
 * thresholds during the scan (what NCCL mode does over peer memory at world > 1): each
 * context's tensor-core scan MIN-s every threshold it publishes into the other contexts'
 * threshold arrays.  Use only with contexts that query the same frames in lock-step, each
 * after all of them ran that shape once (the arrays must be allocated); destroying a
 * context unlinks it; world = 1 unlinks ctxs[0].  Nothing waits on anything, so the
 * contexts' queries may run concurrently on separate streams.  Errors: INVALID_ARGUMENT
 * (NULL, different devices, a context owning a NCCL communicator). */
OL_API ol_status ol_tau_share_emulate(ol_ctx **ctxs, int32_t world);

/* ---- results ------------------------------------------------------------- */

/* Number of candidates of the last query: n_bundles * M * sum_i min(N, |n_i|). */
OL_API ol_status ol_candidate_count(const ol_ctx *ctx, uint64_t *count);

/* Copy the candidates to a caller-owned host buffer in (bundle, frame, subspace,
 * rank) order.  Synchronises the stream.  Errors: INVALID_ARGUMENT
 * (capacity too small), NOT_READY, NONFINITE (device frames held NaN/Inf), CUDA. */
OL_API ol_status ol_get_topk(ol_ctx *ctx, ol_candidate *out, uint64_t capacity, uint64_t *written);

/* Device pointer to the same candidate array (owned by the context; valid until
 * the next ol_query).  Does not synchronise. */
OL_API ol_status ol_topk_device(ol_ctx *ctx, const ol_candidate **dev_ptr, uint64_t *count);

/* Copy the n_bundles estimates to a caller-owned host buffer.  Synchronises.
 * Errors: EMPTY (aggregation was not requested), INVALID_ARGUMENT (capacity),
 * NOT_READY, CUDA. */
OL_API ol_status ol_get_estimates(ol_ctx *ctx, ol_estimate *out, uint32_t capacity);

/* Both at once with ONE stream synchronisation (the latency configurations: a second
 * D2H + sync costs ~15 us on a 20 us query): the candidates as ol_get_topk into
 * cand_out (cand_capacity) and, when the query aggregated and est_out is non-NULL,
 * the n_bundles estimates as ol_get_estimates into est_out (est_capacity).
 * *written = the candidate count.  Errors: those of ol_get_topk / ol_get_estimates
 * (EMPTY only if est_out is non-NULL and aggregation was not requested). */
OL_API ol_status ol_get_results(ol_ctx *ctx, ol_candidate *cand_out, uint64_t cand_capacity, uint64_t *written,
                                ol_estimate *est_out, uint32_t est_capacity);

/* ---- standalone pieces --------------------------------------------------- */

/* Algorithm 2 alone on caller-provided candidate tiles: bundle b owns
 * xy[offsets[b] .. offsets[b+1]) (pairs of int32).  offsets/xy host or device
 * (on_device); out is a host array of n_bundles.  Synchronous.  Tiles rank by
 * count, then signed (y, x) ascending (R7), for any int32 tile.
 * Errors: EMPTY (a bundle with zero candidates), OUT_OF_RANGE (a tile
 * outside the uploaded database's grid 0 <= x < grid_w, 0 <= y < grid_h -- a
 * DB/grid mismatch, S:102, S:262 -- or, with no database uploaded, outside
 * [-2^30, 2^30)), INVALID_ARGUMENT (parameters as in ol_query; a bundle with
 * more than 8192 candidates), CUDA. */
OL_API ol_status ol_aggregate(ol_ctx *ctx, uint32_t n_bundles, const uint32_t *offsets,
                       const int32_t *xy, int32_t on_device, const ol_params *p,
                       ol_estimate *out);

/* selectNearbyFrames (Alg. 1 step 2; window shape P:139): the window
 * of frames around m, of length min(M, n_frames), shifted to stay inside the
 * sequence.  Pure host function.  Errors: INVALID_ARGUMENT (M even or 0),
 * OUT_OF_RANGE (m >= n_frames). */
OL_API ol_status ol_select_window(uint32_t n_frames, uint32_t m, uint32_t M, uint32_t *first,
                           uint32_t *len);

/* ---- NEXT-1: shift-resolved re-scoring and heading ------------------------ */

/* Upload the omnidirectional profiles ("one-dimensional omnidirectional
 * vector"; W azimuth columns, fp32) of this rank's database rows, in the same
 * subspace / shard order as ol_upload_db's features ([rows][W], host or device).
 * Replaces previous profiles; synchronous.  Errors: NOT_READY (no database),
 * INVALID_ARGUMENT (W outside 8..1024, NULL), NONFINITE, OOM, CUDA. */
OL_API ol_status ol_upload_profiles(ol_ctx *ctx, const float *profiles, uint32_t W, int32_t on_device);

/* For every candidate of the last finalized query: the circular shift s in
 * [0, W) minimising the fp32 chain  acc_s = +0; for w = 0..W-1:
 * d = RN32(q[(w+s) mod W] - p[w]); acc_s = fma32(d, d, acc_s)  between the query
 * frame's profile q and the candidate's database profile p (the north star's
 * "score ... over all circular shifts"), and that minimum; ties -> smallest s.
 * s is the heading difference in columns (2 pi s / W radians).
 * query_profiles: [n_bundles * M][W], host or device.  Candidates whose frame
 * lies in another rank's shard get the key INT64_MAX, so ranks combine with a
 * MIN reduction over ol_shift_keys: done inside this call (collective, NCCL
 * all-reduce on the context stream) when the context owns a communicator, else by
 * the caller.  Asynchronous.  Errors: NOT_READY (no finalized query or no
 * profiles), INVALID_ARGUMENT, NONFINITE (host input), CUDA, NCCL. */
OL_API ol_status ol_shift_rescore(ol_ctx *ctx, const float *query_profiles, int32_t on_device);

/* The same re-scoring with the database profiles of exactly the final candidates
 * supplied by the caller ([n_cand][W] fp32 in candidate order, ol_get_topk's order;
 * host or device like query_profiles), instead of profiles of every database row
 * uploaded with ol_upload_profiles ("W = 256 fp32 = 1 KB/entry, for final candidates
 * only").  Every candidate is scored on this rank (no MIN reduction
 * needed).  8 <= W <= 1024.  Asynchronous.  Errors: NOT_READY (no finalized query),
 * INVALID_ARGUMENT, NONFINITE (host input), CUDA. */
OL_API ol_status ol_shift_rescore_cands(ol_ctx *ctx, const float *query_profiles, const float *cand_profiles,
                                        uint32_t W, int32_t on_device);

/* Device array (owned by the context) of the last ol_shift_rescore, one key per
 * candidate in candidate order: (bits(min acc) << 32) | s, or INT64_MAX. */
OL_API ol_status ol_shift_keys(ol_ctx *ctx, uint64_t **dev_keys, uint64_t *count);

/* Copy those keys to `dst` (device memory, >= 8 bytes per candidate), stream-ordered;
 * e.g. into a buffer the caller MIN-reduces across ranks. */
OL_API ol_status ol_shift_keys_copy(ol_ctx *ctx, void *dst);

/* Host copy of the keys as shift[i], dist2[i] (dist2 = +inf, shift = UINT32_MAX
 * for INT64_MAX keys).  Synchronises.  Errors: NOT_READY, INVALID_ARGUMENT, CUDA. */
OL_API ol_status ol_get_shifts(ol_ctx *ctx, uint32_t *shift, float *dist2, uint64_t capacity);

/* ---- descriptor extraction (NEXT-3, the step before the path) -------------- */

/* The paper's rotation-invariant feature of omnidirectional profiles ("The
 * FFT magnitude of the one-dimensional omnidirectional vector"): for each
 * profile x[0..W-1], X[k] = sum_w x[w] e^{-2 pi i k w / W} for k = 1..64 (DC
 * dropped), m_k = |X[k]|, descriptor = m / ||m|| if ||m|| > 1e-12, else all-zero
 * and flagged degenerate (reading R4).  Binary64 arithmetic on the GPU: an FFT
 * (one warp per profile) for W = 128, 256, 512, a direct sum for other W.
 *   profiles:    [n][W] binary64, host (on_device = 0) or device memory
 *   out32:       [n][64] fp32 descriptors, RN of the binary64 values (the database /
 *                query format of ol_upload_db and ol_query); may be NULL
 *   out64:       [n][64] binary64 descriptors; may be NULL
 *   degenerate:  [n] bytes, 1 = degenerate; may be NULL
 *   profile_out: [n][W] fp32, RN of (x - mean x) / ||m|| (all-zero if degenerate):
 *                the NEXT-1 stored profile, whose |DFT| on bins 1..64 is the
 *                descriptor, so the shift distance of two of them is at least
 *                (2/W) x the squared descriptor distance (Parseval); may be NULL
 * Outputs live where the input lives (host or device; caller-owned).  Host calls
 * synchronise; device calls are stream-ordered.  65 <= W <= 2048.
 * Errors: INVALID_ARGUMENT (W, NULL profiles), NONFINITE (host input with NaN/Inf),
 * CUDA. */
OL_API ol_status ol_extract_features(ol_ctx *ctx, const double *profiles, uint64_t n, uint32_t W,
                                     int32_t on_device, float *out32, double *out64, uint8_t *degenerate,
                                     float *profile_out);

/* ---- tuning / introspection (never changes results) ---------------------- */

/* Launch-shape knobs for schedule-independence tests and tuning.  None of them can
 * change a result: every path computes the exact top-N of R3 (tests force each one).
 *   "chunk"         entries per work item (0 = automatic)
 *   "qtile"         query frames per CTA tile of the CUDA-core scans (0 = automatic)
 *   "tau_seed"      1 (default) / 0: seed pruning thresholds before the scan
 *   "seed_samples"  rows sampled per (frame, subspace) by the exact seed (16..32768; default 0:
 *                   8192 for >= 1,024 (frame, subspace) jobs, else 4096; at most 8192 when the
 *                   one-CTA-per-job seed kernel runs)
 *   "seed_select"   0 (default) / 1: the two-kernel seed's select step: a warp per job gathering
 *                   the values below a strided-subset bound when 2,048 <= samples <= 4,096 and
 *                   N <= 32 /
 *                   the CTA-per-job or radix selects everywhere
 *   "seed_kernel"   1 (default) / 0: two-kernel seed (sample rows reused across frames; one CTA
 *                   per job when its scratch would exceed 2^28 entries) / one CTA per
 *                   (frame, subspace, split) job
 *   "tc"            -1 (default: automatic, >= tc_min_frames frames) / 1 / 0: the certified
 *                   tensor-core filter (needs |f| < 65000 and ||f|| < 300 in the database)
 *   "tc_min_frames" frames per query below which the CUDA-core scans are used (default 0:
 *                   automatic, 4 when the filter plane has 64-B rows (tc_k = 32), else 16)
 *   "tc_seed"       0 (default) / 1 / 2: tensor-core bound pre-pass as the seed (N <= 16);
 *                   2 runs it after the exact sampled seed
 *   "tc_k"          0 (default: 32 when every subspace holds >= 8M rows on this rank, else
 *                   64) / 16 / 32 / 48 / 64: dimensions (a prefix) the certified tensor-core
 *                   filter scores; fewer halve its MMA work, more pairs reach the exact
 *                   re-score.  Results are identical.  Takes effect at the next ol_upload_db
 *   "pair"          1 (default: with the 128-B filter plane and >= 10M rows on the rank) / 2
 *                   (always) / 0 (never): CTA
 *                   pairs (tcgen05 cta_group::2) for the tensor-core scan
 *   "cluster"       1 (default) / 2 / 4 / 8: thread-block clusters over a work item's query
 *                   blocks when pairs are off
 *   "scan2"         1 (default: the TMA-fed kernel for 1-2 frames per tile, the row-pair
 *                   streaming kernel up to 16) / 2 (TMA-fed up to 16) / 0 (the general kernel):
 *                   small-batch CUDA-core kernel choice
 *   "ctas"          cap on resident CTAs (0 = automatic)
 *   "time_kernels"  1 / 0: per-stage CUDA-event timing (stats "time_{seed,scan,merge,final}_ns")
 *   "tc_debug"      profiling only (results invalid when nonzero; host-side bits 64 = keep
 *                   the thresholds found in ol_thresholds instead of seeding, 512 = stop
 *                   after the seed)
 *   "tau_share"     1 (default) / 0: NCCL mode at world > 1: the tensor-core scan MIN-s every
 *                   threshold it publishes into the other ranks' threshold arrays over peer
 *                   memory (handles exchanged collectively through the communicator); any
 *                   rank's published threshold bounds the global N-th best, so results are
 *                   identical and small shards prune as well as the whole database
 *   "micro"         1 (default) / 0: world-1 queries with <= 8,192 rows per subspace and <= 65,536
 *                   (frame, row) pairs run as ONE kernel (NK10: a cluster of 1-8 CTAs per
 *                   (frame, subspace) scores its shares of the rows exactly, rank 0 merges
 *                   the shares' top-N over distributed shared memory and writes the candidate
 *                   rows, each bundle's last job runs Algorithm 2) instead of the launch
 *                   sequence; not used when "tc", "chunk" or "qtile" force a path or schedule
 *   "agg_block"     0 (default) / 1: tests: Algorithm 2 by the CTA-wide kernel for bundles of
 *                   <= 32 candidates too (default: one warp, shuffles only); same results
 *   "inline_rescore" -1 (default: when the subspaces average <= 65,536 rows) / 1 / 0: the tensor-core
 *                   scan's epilogue warps re-score their own survivors (per-frame list locks)
 *                   instead of queueing them to the two exact warps -- for small databases
 *                   (many small subspaces: C2 1.61 -> 1.00 ms), not for large ones (C3:
 *                   0.39 -> 0.70 ms); single CTAs only (CTA pairs keep the exact warps)
 *   "merge_scan"    0 (default) / 1: tests: the per-rank merge takes its fallback (N rounds of
 *                   a CTA-wide minimum over every work-item list) instead of gathering the keys
 *                   <= min over lists of list[N-1]; same results
 *   "poison"        0 (default) / 1: tests (an initcheck stand-in): the next uploads fill padding
 *                   rows and coords with NaN bytes instead of zeros, and every query first
 *                   fills its scratch and output buffers with garbage; results must not change
 *   "graph"         0 (default) / 1: CUDA-graph replay for repeated query shapes (world 1,
 *                   time_kernels off).  The first ol_query of a shape runs eagerly and then
 *                   captures its launch sequence on a private stream; later calls with the
 *                   same frames pointer (device frames; host frames are copied into the
 *                   context's own buffer first), n_bundles, M, params and aggregate flag
 *                   replay it as one cudaGraphLaunch on the context stream.  Results are
 *                   identical.  Up to 16 shapes are kept (least recently used evicted).
 *                   Any ol_set_option or ol_upload_db retires them.  If a capture fails
 *                   that shape keeps running eagerly (no error).
 * Every call (any key) retires the captured query graphs.
 * Errors: INVALID_ARGUMENT (unknown key or value). */
OL_API ol_status ol_set_option(ol_ctx *ctx, const char *key, int64_t value);

/* Read statistics of the last query: "nccl" (1 if the context owns a communicator),
 * "tau_peers" (other ranks' threshold arrays the tensor-core scan publishes into),
 * "used_micro" (1 if the last query ran as the single small-problem kernel),
 * "nccl_version" (of the loaded NCCL, 0 if none), "survivors" (pairs that passed the coarse
 * bound), "pairs" (pairs scanned), "kernels" (kernel launches of the last
 * ol_query + ol_finalize), "used_tc" / "used_pair" (1 if the tensor-core scan / CTA pairs
 * ran), "graph_replays" (queries served by graph replay so far), "tc_k" (the filter's dimensions), "items" / "chunk" (work items and rows per item), "time_{seed,scan,merge,final}_ns"
 * (accumulated stage times while option "time_kernels" is 1; reading resets them).
 * Unknown key: INVALID_ARGUMENT.  Synchronises. */
OL_API ol_status ol_get_stat(ol_ctx *ctx, const char *key, int64_t *value);

#ifdef __cplusplus
}
#endif
#endif /* OMNILOC_H */
