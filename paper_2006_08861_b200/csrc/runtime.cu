// runtime.cu -- the omniloc C-ABI (include/omniloc.h): context, database layout
// in HBM, work decomposition, launch sequence and result retrieval.
//
// Launch sequence of one ol_query:
//   [check_finite]  device frames only
//   tau_seed        NK3  thresholds from a row sample         (one CTA / (frame, subspace))
//   scan<kc>        NK2  coarse prefix + fine completion + CTA top-N (the hot loop)
//   merge_chunks    NK4  per-rank top-N per (frame, subspace) + tiles -> payload
//   -- world == 1: finalize immediately; world > 1: caller all-gathers payloads --
//   merge_ranks     NK4' N smallest of the W gathered payloads   (world > 1 only)
//   candidates           records -> ol_candidate rows, SPEC order
//   aggregate       NK5  Algorithm 2 per bundle                  (if requested)
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <mutex>
#include <nccl.h>   // types and signatures only: the library is loaded on demand (dlopen)
#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a profiler attaches

#include "ol_internal.h"

using namespace ol;

// ---------------------------------------------------------------- NCCL, loaded on demand
// The cross-GPU step of SURVEY §8e (all-gather of the per-rank top-N, plus the MIN
// all-reduce of the seeded thresholds) runs on a communicator the context owns.  NCCL is
// dlopen'ed the first time a context asks for it, so a world-1 process never needs it;
// "libnccl.so.2" resolves to the copy already in the process when there is one (torch's),
// else the system library; OL_NCCL_LIB overrides the path.
struct NcclApi {
    decltype(&ncclGetUniqueId) getUniqueId;
    decltype(&ncclCommInitRank) commInitRank;
    decltype(&ncclCommDestroy) commDestroy;
    decltype(&ncclCommAbort) commAbort;
    decltype(&ncclCommGetAsyncError) commGetAsyncError;
    decltype(&ncclAllGather) allGather;
    decltype(&ncclAllReduce) allReduce;
    decltype(&ncclGetErrorString) getErrorString;
    decltype(&ncclGetVersion) getVersion;
};

static const NcclApi *nccl_api(std::string *why) {
    static std::once_flag once;
    static NcclApi api;
    static bool ok = false;
    static std::string err;
    std::call_once(once, [] {
        const char *env = getenv("OL_NCCL_LIB");
        void *h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { err = std::string("dlopen NCCL: ") + dlerror(); return; }
        bool all = true;
        auto sym = [&](const char *n) { void *f = dlsym(h, n); if (!f) { all = false; err = std::string("NCCL lacks ") + n; } return f; };
        api.getUniqueId = (decltype(api.getUniqueId))sym("ncclGetUniqueId");
        api.commInitRank = (decltype(api.commInitRank))sym("ncclCommInitRank");
        api.commDestroy = (decltype(api.commDestroy))sym("ncclCommDestroy");
        api.commAbort = (decltype(api.commAbort))sym("ncclCommAbort");
        api.commGetAsyncError = (decltype(api.commGetAsyncError))sym("ncclCommGetAsyncError");
        api.allGather = (decltype(api.allGather))sym("ncclAllGather");
        api.allReduce = (decltype(api.allReduce))sym("ncclAllReduce");
        api.getErrorString = (decltype(api.getErrorString))sym("ncclGetErrorString");
        api.getVersion = (decltype(api.getVersion))sym("ncclGetVersion");
        ok = all;
    });
    if (!ok && why) *why = err;
    return ok ? &api : nullptr;
}

static thread_local std::string g_thread_err = "no error";

// bumped whenever grow() (re)allocates a buffer: a captured query graph holds raw
// device pointers, so it is valid only in the allocation epoch it was captured in
static std::atomic<uint64_t> g_alloc_epoch{0};

struct ol_ctx {
    int device = 0, rank = 0, world = 1, kc = 16;
    cudaStream_t stream = nullptr;  // borrowed (NULL = legacy default stream)
    ncclComm_t comm = nullptr;      // owned; set when ol_config carried a NCCL unique id
    uint4 *gather_d = nullptr; size_t gather_cap = 0;   // [world][payload] all-gathered records
    // in-scan threshold sharing (NCCL mode at world > 1, option "tau_share"): the other ranks'
    // threshold arrays, opened by CUDA IPC after a collective exchange of handles whenever the
    // (identically sized) arrays are reallocated
    void *tau_peer[kXchgMax] = {};
    size_t tau_shared_cap = 0;
    unsigned char *hbuf_d = nullptr;
    int64_t opt_tau_share = 1;
    int64_t opt_poison = 0;            // tests: fill padding and per-query outputs with garbage first
    std::vector<ol_ctx *> emu_peers;   // tests: contexts on this device linked by ol_tau_share_emulate
    std::string err = "no error";
    // database
    bool db_ready = false;
    uint32_t n_sub = 0;
    uint64_t rows = 0, rows_pad = 0;
    int32_t grid_w = 0, grid_h = 0;
    std::vector<SubInfo> subs;
    SubInfo *subs_d = nullptr;
    float *coarse = nullptr, *fine = nullptr;
    int32_t *coords = nullptr;
    // tensor-core filter operands (tcscan.cu): fp16 rows + per-row bound terms
    void *plane16 = nullptr;       // fp16 rows [rows][64]
    float2 *blk = nullptr;         // per 32-row block: (min RD||f||^2/2, max RU e_f) of the row bound terms
    uint32_t *tcstat_d = nullptr;  // [0] database norm bound bits, [1] max |f| bits,
                                   // [2] batch norm bound bits, [3] force_all
    bool tc_ok = false;
    float nf_max = 0.f;
    CUtensorMap map_rows, map_rows_half;   // 256-row boxes; 128-row boxes (CTA pairs)
    void *q16 = nullptr; size_t q16_cap = 0;
    float4 *qmeta = nullptr; size_t qmeta_cap = 0;
    bool used_tc = false;
    bool used_pair = false;
    // NEXT-1 profiles and shift keys
    float *prof = nullptr; uint32_t prof_W = 0;
    float *qprof_d = nullptr; size_t qprof_cap = 0;
    u64 *shift_keys = nullptr; size_t shift_cap = 0;
    bool shift_ready = false;
    // work items, one immutable table per chunk size: a captured query graph holds the
    // device pointers of the table it ran with, so a table is never rewritten in place
    // (rewriting items / chunk ranges under a graph of another shape made it
    // scan the wrong rows).  Dropped only with the database, or all at once (gen++) when
    // more than kMaxTables chunk sizes were seen.
    struct ItemTable {
        uint64_t chunk;
        std::vector<WorkItem> items;
        WorkItem *items_d;
        SubInfo *subs_d;          // the subspaces with this table's chunk_begin / chunk_end
        uint32_t max_lists;       // the most work items of one subspace
    };
    static constexpr size_t kMaxTables = 16;
    std::deque<ItemTable> tables;    // (a deque: push_back keeps `cur` valid)
    const ItemTable *cur = nullptr;  // the table of the last query_body
    WorkItem *items_d = nullptr;     // == cur->items_d
    uint64_t items_chunk = 0;
    size_t n_items() const { return cur ? cur->items.size() : 0; }
    uint32_t *seed_scratch = nullptr; size_t seed_scratch_cap = 0;
    // tensor-core bound pre-pass (tau seed) over the strided view rows 0, S, 2S, ...
    uint32_t seed_stride = 0;     // 0: not available (fp16 path off or tiny database)
    CUtensorMap map_srows;
    std::vector<WorkItem> sitems;
    WorkItem *sitems_d = nullptr;
    size_t sitems_cap = 0;
    uint64_t sitems_chunk = 0;
    // per-query buffers
    float *q_d = nullptr; size_t q_cap = 0;
    uint32_t *tau0_d = nullptr; size_t tau_cap = 0;
    u64 *partial_d = nullptr; size_t partial_cap = 0;
    uint4 *payload_d = nullptr; size_t payload_cap = 0;
    uint4 *final_d = nullptr; size_t final_cap = 0;
    // peer-memory exchange (ol_p2p_*): this rank's mailbox (256 B of arrival counters, then
    // 2 x world x max_records records) and the peers' mailboxes opened by CUDA IPC
    unsigned char *mbox_d = nullptr;
    void *peer_base[kXchgMax] = {};
    uint64_t mbox_records = 0;
    int p2p_world = 0, p2p_rank = 0;
    bool p2p_ready = false;
    uint32_t p2p_epoch = 0;
    ol_candidate *cand_d = nullptr; size_t cand_cap = 0;
    ol_estimate *est_d = nullptr; size_t est_cap = 0;
    // device prefixes of min(N, |n_i|), one immutable array per N (same reason as tables)
    std::vector<std::pair<uint32_t, uint32_t *>> prefixes;
    uint32_t *prefix_d = nullptr;   // the prefix of the last ensure_prefix
    bool cand_fused = false;  // world 1: merge_chunks_kernel wrote the candidate rows
    uint32_t *agg_off_d = nullptr; size_t agg_off_cap = 0;
    uint32_t *bcount_d = nullptr; size_t bcount_cap = 0;   // NK10 per-bundle job counters (kept zero)
    bool used_micro = false;
    int64_t opt_micro = 1;
    int64_t opt_inline = -1;     // tensor-core scan: epilogue warps re-score their own survivors (-1 auto: short items)
    int64_t opt_merge_scan = 0;  // 1: the merge's N-round scan over every key (tests: the fallback)
    int64_t opt_agg_block = 0;   // 1: Algorithm 2 by the CTA-wide kernel for bundles <= 32 too (tests)
    int32_t *agg_xy_d = nullptr; size_t agg_xy_cap = 0;
    int *flags_d = nullptr;                // [0] nonfinite frames, [1] aggregation error
    unsigned long long *stat_d = nullptr;  // [0] survivors
    unsigned long long *prof_d = nullptr;  // [16] tcscan per-role cycle counters (tc_debug & 8)
    // last query
    bool q_ready = false, finalized = false;
    uint32_t nb = 0, M = 0, N = 0, nq = 0, qt = 0;
    int aggregate = 0;
    ol_params params{};
    uint64_t n_cand = 0, per_bundle = 0, pairs = 0;
    int launches = 0;
    // options
    int64_t opt_chunk = 0, opt_qtile = 0, opt_tau_seed = 1, opt_ctas = 0, opt_time = 0, opt_seed_samples = 0, opt_seed_select = 0;
    int64_t opt_tc = -1;         // tensor-core filter: -1 auto (>= tc_min_frames frames), 0 off, 1 always
    int64_t opt_tc_min_frames = 0;    // 0 = automatic: 4 with the 64-B plane (kf = 32), else 16.  Round 1, C4:
                                      // 64-B plane: 4 frames scan2 0.94 vs tc 1.02 ms, 8: 1.28 vs 1.02;
                                      // 128-B plane: 8 frames 1.37 vs 1.77, 16: 2.42 vs 1.77
    int64_t opt_tc_debug = 0;
    int64_t opt_seed_kernel = 1;   // 1: two-kernel seed (rows reused across frames), 0: one CTA per (frame, subspace)
    int64_t opt_tc_k = 0;        // tensor-core filter dimensions (prefix; applied at upload); 0 = auto
    uint32_t tc_kf = 64;
    uint32_t tc_pw = 64;         // fp16 plane row width (halves): 32 when tc_kf = 32
    int64_t opt_tc_seed = 0;     // tensor-core path: 1 = seed thresholds with the bound pre-pass (off: the exact sampled seed is as fast at C4 and tighter at C3)
    int64_t opt_cluster = 1;     // tensor-core path: CTAs per cluster (query blocks sharing rows)
    int64_t opt_pair = 1;        // tensor-core path: CTA pairs (cta_group::2, M = 256): 0 off, 1 auto, 2 on
    int64_t opt_scan2 = 1;       // small batches (<= 16 frames per tile): 1 auto (scan3 for <= 2, else scan2), 2 scan3, 0 scan_kernel    // profiling experiments only (results invalid when nonzero)
    // per-kernel-class CUDA-event timing (option "time_kernels"): pairs recorded on
    // the context stream around each launch; summed and released by ol_get_stat
    enum { T_SEED, T_SCAN, T_MERGE, T_FINAL, T_COUNT };
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[T_COUNT];
    std::vector<cudaEvent_t> ev_pool;
    // CUDA-graph replay of repeated query shapes (option "graph"): the
    // launch sequence of ol_query after the host->device copy of the frames, captured
    // on a private stream after one eager run and replayed while the key matches.
    // Any ol_set_option / ol_upload_db bumps `gen` and so retires the graph.
    struct QueryKey {
        const float *q; uint32_t nb, M, on_device, aggregate; ol_params p; uint64_t gen, epoch;
        bool operator==(const QueryKey &o) const {
            return q == o.q && nb == o.nb && M == o.M && on_device == o.on_device && aggregate == o.aggregate &&
                   gen == o.gen && epoch == o.epoch && !memcmp(&p, &o.p, sizeof(p));
        }
    };
    struct QueryState {   // what the launch sequence leaves on the host side
        bool used_tc, used_pair;
        uint32_t nb, M, N, nq, qt;
        int aggregate;
        ol_params params;
        uint64_t n_cand, per_bundle, pairs;
        int launches;
        const ItemTable *cur;   // the (immutable) tables the captured launches read
        uint32_t *prefix_d;
        bool used_micro;
    };
    struct GraphEntry {
        QueryKey key;
        QueryState state;
        cudaGraphExec_t exec;   // NULL: the capture failed, this shape runs eagerly
        uint64_t last_use;
    };
    static constexpr size_t kMaxGraphs = 16;   // shapes kept (least recently used evicted)
    int64_t opt_graph = 0;
    uint64_t gen = 0, graph_clock = 0;
    std::vector<GraphEntry> graphs;
    cudaStream_t cap_stream = nullptr;
    uint64_t graph_replays = 0;
};

static cudaEvent_t take_event(ol_ctx *c) {
    if (!c->ev_pool.empty()) { cudaEvent_t e = c->ev_pool.back(); c->ev_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// NVTX range (host timeline of the launch sequence, for nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct TimeScope {  // a stage of the launch sequence: an NVTX range, and an event pair when timing is on
    ol_ctx *c; int cls; cudaEvent_t a = nullptr;
    NvtxRange nv;
    static const char *name(int cls) {
        static const char *n[] = {"ol.seed", "ol.scan", "ol.merge", "ol.finalize"};
        return n[cls];
    }
    TimeScope(ol_ctx *c_, int cls_) : c(c_), cls(cls_), nv(name(cls_)) {
        if (c->opt_time) { a = take_event(c); cudaEventRecord(a, c->stream); }
    }
    ~TimeScope() {
        if (a) { cudaEvent_t b = take_event(c); cudaEventRecord(b, c->stream); c->ev[cls].push_back({a, b}); }
    }
};

// ---------------------------------------------------------------- helpers
static ol_status fail(ol_ctx *c, ol_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    g_thread_err = buf;
    return s;
}

#define OL_CUDA(c, call)                                                                   \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail((c), e_ == cudaErrorMemoryAllocation ? OL_ERR_OOM : OL_ERR_CUDA,    \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define OL_NCCL(c, call)                                                                     \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            return fail((c), OL_ERR_NCCL, "%s: %s (%s:%d)", #call, nccl_api(nullptr)->getErrorString(r_), \
                        __FILE__, __LINE__);                                                 \
    } while (0)

// a communicator error raised asynchronously (a peer died, a network fault)
static ol_status fail(ol_ctx *c, ol_status s, const char *fmt, ...);
static ol_status nccl_poll(ol_ctx *c) {
    if (!c->comm) return OL_OK;
    ncclResult_t a = ncclSuccess;
    const NcclApi *api = nccl_api(nullptr);
    const ncclResult_t r = api->commGetAsyncError(c->comm, &a);
    if (r != ncclSuccess) return fail(c, OL_ERR_NCCL, "ncclCommGetAsyncError: %s", api->getErrorString(r));
    if (a != ncclSuccess && a != ncclInProgress)
        return fail(c, OL_ERR_NCCL, "NCCL communicator error: %s", api->getErrorString(a));
    return OL_OK;
}

#define OL_LAUNCH(c, call)  \
    do {                    \
        OL_CUDA(c, call);   \
        ++(c)->launches;    \
    } while (0)

template <typename T>
static cudaError_t grow(T **p, size_t *cap, size_t n) {
    if (n <= *cap && *p) return cudaSuccess;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    size_t want = n < 1 ? 1 : n;
    g_alloc_epoch.fetch_add(1);
    cudaError_t e = cudaMalloc((void **)p, want * sizeof(T));
    if (e == cudaSuccess) *cap = want;
    return e;
}

static ol_status check_params(ol_ctx *c, const ol_params *p, bool need_agg) {
    if (!p) return fail(c, OL_ERR_INVALID_ARGUMENT, "params is NULL");
    if (p->N == 0 || p->N > OL_MAX_N)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "N=%u outside 1..%d", p->N, OL_MAX_N);
    if (need_agg) {
        if (p->top_c == 0 || p->top_c > OL_MAX_TOP_C)
            return fail(c, OL_ERR_INVALID_ARGUMENT, "top_c=%u outside 1..%d", p->top_c, OL_MAX_TOP_C);
        if (!(p->toler_per > 0.0 && p->toler_per <= 1.0))
            return fail(c, OL_ERR_INVALID_ARGUMENT, "toler_per=%g outside (0,1]", p->toler_per);
        if (!(p->radius_m > 0.0) || !std::isfinite(p->radius_m))
            return fail(c, OL_ERR_INVALID_ARGUMENT, "radius_m=%g must be > 0", p->radius_m);
        if (!(p->tile_m > 0.0) || !std::isfinite(p->tile_m))
            return fail(c, OL_ERR_INVALID_ARGUMENT, "tile_m=%g must be > 0", p->tile_m);
    }
    return OL_OK;
}

static void free_tables(ol_ctx *c) {
    for (auto &t : c->tables) { cudaFree(t.items_d); cudaFree(t.subs_d); }
    c->tables.clear();
    c->cur = nullptr;
    c->items_d = nullptr;
    c->items_chunk = 0;
    for (auto &p : c->prefixes) cudaFree(p.second);
    c->prefixes.clear();
    c->prefix_d = nullptr;
}

static void free_db(ol_ctx *c) {
    free_tables(c);
    cudaFree(c->coarse); cudaFree(c->fine); cudaFree(c->coords); cudaFree(c->subs_d);
    cudaFree(c->plane16); cudaFree(c->blk); cudaFree(c->prof);
    c->prof = nullptr; c->prof_W = 0;
    c->coarse = c->fine = nullptr; c->coords = nullptr; c->subs_d = nullptr;
    c->plane16 = nullptr; c->blk = nullptr; c->tc_ok = false;
    c->db_ready = false;
    c->sitems_chunk = 0;
    c->seed_stride = 0;
}

extern "C" {

// ---------------------------------------------------------------- lifetime
ol_status ol_create(const ol_config *cfg, ol_ctx **out) {
    if (!out) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!cfg) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "cfg is NULL");
    if (cfg->K != OL_K) return fail(nullptr, OL_ERR_DIMENSION_MISMATCH, "K=%u, library needs %d", cfg->K, OL_K);
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world)
        return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "rank=%d world=%d", cfg->rank, cfg->world);
    int kc = cfg->coarse_k == 0 ? OL_K : (int)cfg->coarse_k;
    if (kc != 8 && kc != 16 && kc != 32 && kc != 64)
        return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "coarse_k=%u not in {0,8,16,32,64}", cfg->coarse_k);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, OL_ERR_CUDA, "no CUDA device: %s", cudaGetErrorString(e));
    if (cfg->device < 0 || cfg->device >= ndev)
        return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "device %d of %d", cfg->device, ndev);
    ol_ctx *c = new ol_ctx();
    c->device = cfg->device; c->rank = cfg->rank; c->world = cfg->world; c->kc = kc;
    e = cudaSetDevice(c->device);
    if (e == cudaSuccess) {
        c->stream = (cudaStream_t)cfg->cuda_stream;  // borrowed; NULL = legacy default stream
    }
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->flags_d, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->stat_d, 4 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->tcstat_d, 8 * sizeof(uint32_t));
    if (e == cudaSuccess) e = cudaMalloc((void **)&c->prof_d, 1024 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(c->flags_d, 0, 4 * sizeof(int));
    if (e != cudaSuccess) {
        fail(nullptr, OL_ERR_CUDA, "ol_create: %s", cudaGetErrorString(e));
        ol_destroy(c);
        return OL_ERR_CUDA;
    }
    if (cfg->nccl_unique_id) {   // collective: every rank of `world` calls ol_create with the same id
        std::string why;
        const NcclApi *api = nccl_api(&why);
        if (!api) { ol_destroy(c); return fail(nullptr, OL_ERR_NCCL, "%s", why.c_str()); }
        ncclUniqueId id;
        memcpy(&id, cfg->nccl_unique_id, sizeof(id));
        const ncclResult_t r = api->commInitRank(&c->comm, c->world, id, c->rank);
        if (r != ncclSuccess) {
            c->comm = nullptr;
            ol_destroy(c);
            return fail(nullptr, OL_ERR_NCCL, "ncclCommInitRank(world %d, rank %d): %s", cfg->world, cfg->rank,
                        api->getErrorString(r));
        }
    }
    *out = c;
    return OL_OK;
}

ol_status ol_nccl_unique_id(void *out) {
    if (!out) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "out is NULL");
    std::string why;
    const NcclApi *api = nccl_api(&why);
    if (!api) return fail(nullptr, OL_ERR_NCCL, "%s", why.c_str());
    ncclUniqueId id;
    const ncclResult_t r = api->getUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, OL_ERR_NCCL, "ncclGetUniqueId: %s", api->getErrorString(r));
    static_assert(sizeof(id) == OL_NCCL_ID_BYTES, "ncclUniqueId size");
    memcpy(out, &id, sizeof(id));
    return OL_OK;
}


// release the peer mailboxes opened by IPC and this rank's own
static void p2p_close(ol_ctx *c) {
    for (int p = 0; p < kXchgMax; ++p)
        if (c->peer_base[p]) { cudaIpcCloseMemHandle(c->peer_base[p]); c->peer_base[p] = nullptr; }
    cudaFree(c->mbox_d);
    c->mbox_d = nullptr;
    c->p2p_ready = false;
    c->p2p_world = 0;
}

void ol_destroy(ol_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->comm) {   // a communicator in error state cannot be destroyed cleanly: abort it
        const NcclApi *api = nccl_api(nullptr);
        ncclResult_t a = ncclSuccess;
        if (api->commGetAsyncError(c->comm, &a) == ncclSuccess && a == ncclSuccess) api->commDestroy(c->comm);
        else api->commAbort(c->comm);
        c->comm = nullptr;
    }
    cudaFree(c->gather_d);
    for (auto &p : c->tau_peer)
        if (p) { cudaIpcCloseMemHandle(p); p = nullptr; }
    cudaFree(c->hbuf_d);
    for (ol_ctx *o : c->emu_peers) {   // unlink from the emulated group
        auto &v = o->emu_peers;
        for (size_t i = 0; i < v.size(); ++i)
            if (v[i] == c) { v.erase(v.begin() + i); break; }
    }
    free_db(c);
    cudaFree(c->seed_scratch); cudaFree(c->sitems_d); cudaFree(c->q_d); cudaFree(c->tau0_d); cudaFree(c->partial_d);
    cudaFree(c->payload_d); cudaFree(c->final_d); cudaFree(c->cand_d); cudaFree(c->est_d);
    p2p_close(c);
    cudaFree(c->agg_off_d); cudaFree(c->bcount_d); cudaFree(c->agg_xy_d);
    cudaFree(c->flags_d); cudaFree(c->stat_d); cudaFree(c->tcstat_d); cudaFree(c->prof_d);
    cudaFree(c->q16); cudaFree(c->qmeta); cudaFree(c->qprof_d); cudaFree(c->shift_keys);
    for (auto &v : c->ev)
        for (auto &p : v) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    for (auto &g : c->graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    delete c;
}

const char *ol_last_error(const ol_ctx *c) { return c ? c->err.c_str() : g_thread_err.c_str(); }

ol_status ol_set_stream(ol_ctx *c, void *stream) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    c->stream = (cudaStream_t)stream;
    return OL_OK;
}

ol_status ol_shard_range(uint64_t n, int32_t rank, int32_t world, uint64_t *begin,
                         uint64_t *count) {
    if (world < 1 || rank < 0 || rank >= world || !begin || !count)
        return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "rank=%d world=%d", rank, world);
    // floor(r * n / w) without overflow for n < 2^63, w < 2^31
    uint64_t b = (n / world) * rank + (n % world) * rank / world;
    uint64_t e = (n / world) * (rank + 1) + (n % world) * (rank + 1) / world;
    *begin = b;
    *count = e - b;
    return OL_OK;
}

ol_status ol_select_window(uint32_t n_frames, uint32_t m, uint32_t M, uint32_t *first,
                           uint32_t *len) {
    if (M == 0 || M % 2 == 0) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "M=%u must be odd", M);
    if (m >= n_frames) return fail(nullptr, OL_ERR_OUT_OF_RANGE, "m=%u >= n_frames=%u", m, n_frames);
    if (!first || !len) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "NULL output");
    const uint32_t L = M < n_frames ? M : n_frames;
    const uint32_t h = (M - 1) / 2;
    uint32_t f = m > h ? m - h : 0;          // centred window, clipped at the start ...
    if (f > n_frames - L) f = n_frames - L;  // ... and shifted back from the end
    *first = f;
    *len = L;
    return OL_OK;
}

// ---------------------------------------------------------------- database
ol_status ol_upload_db(ol_ctx *c, const ol_db_desc *db) {
    NvtxRange nv("ol_upload_db");
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!db || db->n_subspaces == 0 || !db->global_sizes || !db->features || !db->coords)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "database descriptor incomplete");
    if ((db->shard_begin == nullptr) != (db->shard_count == nullptr))
        return fail(c, OL_ERR_INVALID_ARGUMENT, "shard_begin and shard_count must both be set or NULL");
    if (db->grid_w <= 0 || db->grid_h <= 0)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "grid %dx%d", db->grid_w, db->grid_h);
    OL_CUDA(c, cudaSetDevice(c->device));
    const uint32_t ns = db->n_subspaces;
    std::vector<SubInfo> subs(ns);
    std::vector<uint64_t> src_begin(ns);   // row offset of subspace i in the caller's arrays
    uint64_t rows = 0, rows_pad = 0;       // device rows: each subspace starts on a 256-row tile (kPadRows)
    for (uint32_t i = 0; i < ns; ++i) {
        const uint64_t gs = db->global_sizes[i];
        if (gs == 0 || gs > 0xFFFFFFFEull)
            return fail(c, OL_ERR_INVALID_ARGUMENT, "subspace %u size %llu outside 1..2^32-2", i,
                        (unsigned long long)gs);
        uint64_t b, n;
        if (db->shard_begin) { b = db->shard_begin[i]; n = db->shard_count[i]; }
        else ol_shard_range(gs, c->rank, c->world, &b, &n);
        if (b + n > gs)
            return fail(c, OL_ERR_INVALID_ARGUMENT, "shard [%llu,+%llu) outside subspace %u of %llu",
                        (unsigned long long)b, (unsigned long long)n, i, (unsigned long long)gs);
        src_begin[i] = rows;
        subs[i].row_begin = rows_pad;
        subs[i].count = n;
        subs[i].shard_begin = (uint32_t)b;
        subs[i].global_size = (uint32_t)gs;
        rows += n;
        rows_pad += (n + kPadRows - 1) / kPadRows * kPadRows;
    }
    // validate inputs (S:32 finite values; S:102 coords inside the grid)
    if (!db->on_device) {
        for (uint64_t t = 0; t < rows * OL_K; ++t)
            if (!std::isfinite(db->features[t]))
                return fail(c, OL_ERR_NONFINITE, "feature value %llu is not finite", (unsigned long long)t);
        for (uint64_t t = 0; t < rows; ++t) {
            int32_t x = db->coords[2 * t], y = db->coords[2 * t + 1];
            if (x < 0 || x >= db->grid_w || y < 0 || y >= db->grid_h)
                return fail(c, OL_ERR_OUT_OF_RANGE, "coord (%d,%d) of row %llu outside %dx%d grid", x, y,
                            (unsigned long long)t, db->grid_w, db->grid_h);
        }
    }
    free_db(c);
    const int kc = c->kc;
    const uint64_t R = rows_pad ? rows_pad : 32;
    OL_CUDA(c, cudaMalloc((void **)&c->coarse, sizeof(float) * R * kc));
    // padding rows = 0 (option "poison": NaN bytes, so a padding element that is ever read shows)
    const int fillb = c->opt_poison ? 0xFF : 0;
    OL_CUDA(c, cudaMemsetAsync(c->coarse, fillb, sizeof(float) * R * kc, c->stream));
    OL_CUDA(c, cudaMalloc((void **)&c->fine, sizeof(float) * R * OL_K));   // (full rows: fine_off)
    OL_CUDA(c, cudaMemsetAsync(c->fine, fillb, sizeof(float) * R * OL_K, c->stream));
    OL_CUDA(c, cudaMalloc((void **)&c->coords, sizeof(int32_t) * 2 * R));
    OL_CUDA(c, cudaMemsetAsync(c->coords, fillb, sizeof(int32_t) * 2 * R, c->stream));
    OL_CUDA(c, cudaMalloc((void **)&c->subs_d, sizeof(SubInfo) * ns));
    const float *src = db->features;
    float *tmp = nullptr;
    if (rows) {
        const cudaMemcpyKind kind = db->on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        if (db->on_device) {
            OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, 2 * sizeof(int), c->stream));
            OL_CUDA(c, launch_check_finite(db->features, rows * OL_K, c->flags_d, c->stream));
            OL_CUDA(c, launch_check_coords(db->coords, rows, 0, db->grid_w, 0, db->grid_h, c->flags_d + 1,
                                           c->stream));
            int fl[2];
            OL_CUDA(c, cudaMemcpyAsync(fl, c->flags_d, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
            OL_CUDA(c, cudaStreamSynchronize(c->stream));
            OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, 2 * sizeof(int), c->stream));
            if (fl[0]) { free_db(c); return fail(c, OL_ERR_NONFINITE, "device features hold NaN/Inf"); }
            if (fl[1]) { free_db(c); return fail(c, OL_ERR_OUT_OF_RANGE, "device coords outside the grid"); }
        } else {
            OL_CUDA(c, cudaMalloc((void **)&tmp, sizeof(float) * rows * OL_K));
            OL_CUDA(c, cudaMemcpyAsync(tmp, db->features, sizeof(float) * rows * OL_K,
                                       cudaMemcpyHostToDevice, c->stream));
            src = tmp;
        }
        for (uint32_t i = 0; i < ns; ++i) {   // subspace i -> its tile-aligned device rows
            if (!subs[i].count) continue;
            OL_CUDA(c, cudaMemcpyAsync(c->coords + 2 * subs[i].row_begin, db->coords + 2 * src_begin[i],
                                       sizeof(int32_t) * 2 * subs[i].count, kind, c->stream));
            OL_CUDA(c, launch_relayout(src + src_begin[i] * OL_K, subs[i].count, subs[i].row_begin, kc, c->coarse,
                                       c->fine, c->stream));
        }
        // tile-padding rows repeat their subspace's last row (never reported: every kernel
        // bounds rows by the subspace count), so per-block row terms stay tight
        OL_CUDA(c, cudaMemcpyAsync(c->subs_d, subs.data(), sizeof(SubInfo) * ns, cudaMemcpyHostToDevice,
                                   c->stream));
        OL_CUDA(c, launch_pad_rows(c->subs_d, ns, kc, c->coarse, c->fine, c->stream));
        if (c->opt_tc != 0) {
            // the filter on the first 32 dimensions halves the MMA work but passes more
            // pairs to the exact path; automatic mode takes 32 once every subspace holds >= 8M
            // rows on this rank.  Round 2 (survivor rows read in halves, best pair setting each,
            // 1,024 frames, kf 32 vs 64): 6M rows 0.868 vs 0.857 ms, 10M 1.216 vs 1.271, 12.5M
            // 1.414 vs 1.507, 25M 2.379 vs 2.716, 50M 4.289 vs 5.432 (round 1 crossed at ~32M)
            uint64_t minc = ~0ull;
            for (auto &sb : subs) minc = sb.count < minc ? sb.count : minc;
            c->tc_kf = c->opt_tc_k ? (uint32_t)c->opt_tc_k : (minc >= 8000000ull ? 32u : 64u);
            // kf = 32: the plane holds only those dimensions (64-B rows): half the bytes
            // streamed, and what makes few-frame batches HBM-bound at half the time
            c->tc_pw = c->tc_kf == 32 ? 32u : 64u;
            OL_CUDA(c, cudaMalloc(&c->plane16, sizeof(uint16_t) * rows_pad * c->tc_pw));
            OL_CUDA(c, cudaMalloc((void **)&c->blk, sizeof(float2) * (rows_pad / 32)));
            OL_CUDA(c, cudaMemsetAsync(c->tcstat_d, 0, 8 * sizeof(uint32_t), c->stream));
            OL_CUDA(c, launch_tc_prep_rows(c->coarse, c->fine, kc, rows_pad, c->plane16, c->blk, c->tcstat_d,
                                           c->tc_kf, c->tc_pw, c->stream));
        }
    }
    OL_CUDA(c, cudaMemcpyAsync(c->subs_d, subs.data(), sizeof(SubInfo) * ns, cudaMemcpyHostToDevice,
                               c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    if (tmp) cudaFree(tmp);
    if (c->plane16 && rows) {
        uint32_t st[2];
        OL_CUDA(c, cudaMemcpy(st, c->tcstat_d, sizeof(st), cudaMemcpyDeviceToHost));
        const float nf = *reinterpret_cast<float *>(&st[0]), amax = *reinterpret_cast<float *>(&st[1]);
        c->nf_max = nf;
        // fp16 operands need |f| and ||f||^2 / 2 inside the fp16 range, and the row count
        // must fit a TMA coordinate
        c->tc_ok = std::isfinite(nf) && amax < 65000.f && nf < 300.f && rows_pad < (1ull << 31) &&
                   make_tc_map(&c->map_rows, c->plane16, rows_pad, 256, c->tc_pw) &&
                   make_tc_map(&c->map_rows_half, c->plane16, rows_pad, 128, c->tc_pw);
        // bound pre-pass view: ~128k sampled rows, at most 1/64 of the database
        uint64_t S = 64;
        while (rows_pad / (S * 2) >= 131072) S *= 2;
        c->seed_stride = c->tc_ok && rows_pad / S >= 2048 &&
                         make_tc_map(&c->map_srows, c->plane16, rows_pad, 256, c->tc_pw, (uint32_t)S) ? (uint32_t)S : 0;
    }
    c->subs = subs;
    c->rows_pad = rows_pad;
    c->n_sub = ns;
    c->rows = rows;
    c->grid_w = db->grid_w;
    c->grid_h = db->grid_h;
    c->db_ready = true;
    ++c->gen;
    c->q_ready = false;
    return OL_OK;
}

// ---------------------------------------------------------------- work decomposition
static ol_status build_items(ol_ctx *c, uint64_t chunk) {
    for (auto &t : c->tables)
        if (t.chunk == chunk) {
            c->cur = &t; c->items_d = t.items_d; c->items_chunk = chunk;
            return OL_OK;
        }
    if (c->tables.size() >= ol_ctx::kMaxTables) {   // retire every graph before freeing tables
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        for (auto &t : c->tables) { cudaFree(t.items_d); cudaFree(t.subs_d); }
        c->tables.clear();
        c->cur = nullptr;
        ++c->gen;
    }
    std::vector<WorkItem> items;
    std::vector<SubInfo> subs = c->subs;
    for (uint32_t i = 0; i < c->n_sub; ++i) {
        SubInfo &s = subs[i];
        s.chunk_begin = (uint32_t)items.size();
        for (uint64_t o = 0; o < s.count; o += chunk) {
            WorkItem w;
            w.sub = i;
            w.count = (uint32_t)((s.count - o) < chunk ? (s.count - o) : chunk);
            w.row_begin = s.row_begin + o;
            w.frame_begin = (uint32_t)(s.shard_begin + o);
            w._pad = 0;
            items.push_back(w);
        }
        s.chunk_end = (uint32_t)items.size();
    }
    uint32_t max_lists = 0;
    for (auto &sb : subs) max_lists = sb.chunk_end - sb.chunk_begin > max_lists ? sb.chunk_end - sb.chunk_begin : max_lists;
    ol_ctx::ItemTable t{chunk, items, nullptr, nullptr, max_lists};
    OL_CUDA(c, cudaMalloc((void **)&t.items_d, sizeof(WorkItem) * (items.empty() ? 1 : items.size())));
    if (cudaMalloc((void **)&t.subs_d, sizeof(SubInfo) * c->n_sub) != cudaSuccess) {
        cudaFree(t.items_d);
        return fail(c, OL_ERR_OOM, "work-item table");
    }
    c->tables.push_back(t);
    ol_ctx::ItemTable &tb = c->tables.back();
    if (!items.empty())
        OL_CUDA(c, cudaMemcpyAsync(tb.items_d, tb.items.data(), sizeof(WorkItem) * items.size(),
                                   cudaMemcpyHostToDevice, c->stream));
    OL_CUDA(c, cudaMemcpyAsync(tb.subs_d, subs.data(), sizeof(SubInfo) * c->n_sub, cudaMemcpyHostToDevice,
                               c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));  // host vectors are pageable
    c->cur = &tb; c->items_d = tb.items_d; c->items_chunk = chunk;
    return OL_OK;
}

// Work items of the pre-pass view (rows 0, S, 2S, ... of the device planes): per
// subspace, its rows that are multiples of S, in chunks of `chunk` view rows.
static ol_status build_sitems(ol_ctx *c, uint64_t chunk) {
    if (chunk == c->sitems_chunk && !c->sitems.empty()) return OL_OK;
    const uint64_t S = c->seed_stride;
    std::vector<WorkItem> items;
    for (uint32_t i = 0; i < c->n_sub; ++i) {
        const SubInfo &s = c->subs[i];
        if (!s.count) continue;
        const uint64_t j0 = (s.row_begin + S - 1) / S, j1 = (s.row_begin + s.count - 1) / S;
        if (j1 < j0) continue;
        const uint64_t n = j1 - j0 + 1;
        for (uint64_t o = 0; o < n; o += chunk) {
            WorkItem w;
            w.sub = i;
            w.count = (uint32_t)((n - o) < chunk ? (n - o) : chunk);
            w.row_begin = j0 + o;
            w.frame_begin = 0;   // (the pre-pass reports no frames)
            w._pad = 0;
            items.push_back(w);
        }
    }
    // rewritten in place (the bound pre-pass is not the default): retire captured graphs
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    ++c->gen;
    OL_CUDA(c, grow(&c->sitems_d, &c->sitems_cap, items.size() ? items.size() : 1));
    if (!items.empty())
        OL_CUDA(c, cudaMemcpyAsync(c->sitems_d, items.data(), sizeof(WorkItem) * items.size(),
                                   cudaMemcpyHostToDevice, c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    c->sitems.swap(items);
    c->sitems_chunk = chunk;
    return OL_OK;
}

// device prefix of min(N, |n_i|) over the subspaces (candidate row offsets)
static ol_status ensure_prefix(ol_ctx *c, uint32_t N) {
    for (auto &p : c->prefixes)
        if (p.first == N) { c->prefix_d = p.second; return OL_OK; }
    const uint32_t ns = c->n_sub;
    std::vector<uint32_t> prefix(ns + 1, 0);
    for (uint32_t i = 0; i < ns; ++i)
        prefix[i + 1] = prefix[i] + (c->subs[i].global_size < N ? c->subs[i].global_size : N);
    uint32_t *d = nullptr;
    OL_CUDA(c, cudaMalloc((void **)&d, sizeof(uint32_t) * (ns + 1)));
    c->prefixes.push_back({N, d});   // at most OL_MAX_N entries of n_sub + 1 words
    OL_CUDA(c, cudaMemcpyAsync(d, prefix.data(), sizeof(uint32_t) * (ns + 1), cudaMemcpyHostToDevice, c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    c->prefix_d = d;
    return OL_OK;
}

static ol_status finalize_impl(ol_ctx *c, const uint4 *gathered, int world);
static ol_status query_body(ol_ctx *c, uint32_t nb, uint32_t M, const float *q, int32_t on_device,
                            const ol_params *p, int32_t aggregate, uint64_t per_q);

static ol_ctx::QueryState save_state(const ol_ctx *c) {
    return {c->used_tc, c->used_pair, c->nb, c->M, c->N, c->nq, c->qt, c->aggregate, c->params,
            c->n_cand, c->per_bundle, c->pairs, c->launches, c->cur, c->prefix_d, c->used_micro};
}

static void load_state(ol_ctx *c, const ol_ctx::QueryState &s) {
    c->used_tc = s.used_tc; c->used_pair = s.used_pair; c->nb = s.nb; c->M = s.M; c->N = s.N; c->nq = s.nq;
    c->qt = s.qt; c->aggregate = s.aggregate; c->params = s.params; c->n_cand = s.n_cand;
    c->per_bundle = s.per_bundle; c->pairs = s.pairs; c->launches = s.launches;
    c->cur = s.cur; c->items_d = s.cur ? s.cur->items_d : nullptr; c->items_chunk = s.cur ? s.cur->chunk : 0;
    c->prefix_d = s.prefix_d;
    c->used_micro = s.used_micro;
    c->q_ready = true;
    c->finalized = c->world == 1;
    c->shift_ready = false;
}

// Capture query_body's launch sequence (already run eagerly once, so its caches and
// buffers are warm and it makes no synchronising call) on the private stream.  A
// failed capture leaves the entry's exec NULL: this shape then runs eagerly.
static void capture_query(ol_ctx *c, const ol_ctx::QueryKey &k, uint32_t nb, uint32_t M, const float *q,
                          int32_t on_device, const ol_params *p, int32_t aggregate, uint64_t per_q) {
    if (c->graphs.size() >= ol_ctx::kMaxGraphs) {   // evict the least recently used shape
        size_t lru = 0;
        for (size_t i = 1; i < c->graphs.size(); ++i)
            if (c->graphs[i].last_use < c->graphs[lru].last_use) lru = i;
        if (c->graphs[lru].exec) cudaGraphExecDestroy(c->graphs[lru].exec);
        c->graphs.erase(c->graphs.begin() + lru);
    }
    const ol_ctx::QueryState st0 = save_state(c);
    ol_ctx::QueryKey k2 = k;
    k2.epoch = g_alloc_epoch.load();   // the eager run may have grown buffers ...
    k2.gen = c->gen;                   // ... or retired graphs (table cache full, pre-pass items)
    c->graphs.push_back({k2, st0, nullptr, ++c->graph_clock});
    ol_ctx::GraphEntry &ge = c->graphs.back();
    const std::string err0 = c->err;
    if (!c->cap_stream && cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    cudaStream_t s0 = c->stream;
    c->stream = c->cap_stream;
    cudaGraph_t g = nullptr;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess) {
        const ol_status st = query_body(c, nb, M, q, on_device, p, aggregate, per_q);
        const cudaError_t e = cudaStreamEndCapture(c->stream, &g);
        cudaGraphExec_t ex = nullptr;
        if (st == OL_OK && e == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) == cudaSuccess)
            ge.exec = ex;
        if (g) cudaGraphDestroy(g);
    }
    cudaGetLastError();
    c->stream = s0;
    c->err = err0;
    load_state(c, st0);
}

// ---------------------------------------------------------------- query
ol_status ol_query(ol_ctx *c, uint32_t nb, uint32_t M, const float *frames, int32_t on_device,
                   const ol_params *p, int32_t aggregate) {
    NvtxRange nv("ol_query");
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->db_ready) return fail(c, OL_ERR_NOT_READY, "no database uploaded");
    ol_status st = check_params(c, p, aggregate != 0);
    if (st) return st;
    if (nb == 0) return fail(c, OL_ERR_INVALID_ARGUMENT, "n_bundles = 0");
    if (M == 0 || M % 2 == 0 || M > OL_MAX_M)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "M=%u must be odd and <= %d", M, OL_MAX_M);
    if (!frames) return fail(c, OL_ERR_INVALID_ARGUMENT, "frames is NULL");
    const uint64_t nq64 = (uint64_t)nb * M;
    if (nq64 > (1u << 24)) return fail(c, OL_ERR_INVALID_ARGUMENT, "too many query frames");
    const uint32_t nq = (uint32_t)nq64, N = p->N;
    uint64_t per_q = 0;
    for (uint32_t i = 0; i < c->n_sub; ++i) per_q += c->subs[i].global_size < N ? c->subs[i].global_size : N;
    if (aggregate && per_q * M > (uint64_t)kAggMax)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "bundle of %llu candidates exceeds %d",
                    (unsigned long long)(per_q * M), kAggMax);
    OL_CUDA(c, cudaSetDevice(c->device));
    c->q_ready = c->finalized = false;
    c->shift_ready = false;
    const float *q = frames;
    if (!on_device) {
        for (uint64_t t = 0; t < nq64 * OL_K; ++t)
            if (!std::isfinite(frames[t]))
                return fail(c, OL_ERR_NONFINITE, "frame value %llu is not finite", (unsigned long long)t);
        OL_CUDA(c, grow(&c->q_d, &c->q_cap, (size_t)nq * OL_K));
        OL_CUDA(c, cudaMemcpyAsync(c->q_d, frames, sizeof(float) * nq * OL_K, cudaMemcpyHostToDevice,
                                   c->stream));
        q = c->q_d;
    }
    // graph replay: one launch for the whole sequence when this shape ran before
    const bool graph = c->opt_graph && !c->opt_time && c->world == 1 && !c->comm;
    const ol_ctx::QueryKey key{q, nb, M, (uint32_t)(on_device != 0), (uint32_t)(aggregate != 0), *p, c->gen,
                               g_alloc_epoch.load()};
    if (graph) {
        for (size_t i = 0; i < c->graphs.size();)   // retire the graphs of older generations / epochs
            if (c->graphs[i].key.gen != key.gen || c->graphs[i].key.epoch != key.epoch) {
                if (c->graphs[i].exec) cudaGraphExecDestroy(c->graphs[i].exec);
                c->graphs.erase(c->graphs.begin() + i);
            } else ++i;
        for (auto &ge : c->graphs) {
            if (!(ge.key == key)) continue;
            ge.last_use = ++c->graph_clock;
            if (!ge.exec) return query_body(c, nb, M, q, on_device, p, aggregate, per_q);
            OL_CUDA(c, cudaGraphLaunch(ge.exec, c->stream));
            load_state(c, ge.state);
            ++c->graph_replays;
            return OL_OK;
        }
    }
    st = query_body(c, nb, M, q, on_device, p, aggregate, per_q);
    if (st || !graph) return st;
    capture_query(c, key, nb, M, q, on_device, p, aggregate, per_q);
    return OL_OK;
}

// Threshold sharing: every rank's seeded threshold for a (frame, subspace) is
// the N-th smallest acc of N distinct rows of that subspace, so it bounds the GLOBAL N-th
// smallest from above, and so does the minimum over ranks.  Pruning stays strict (acc > tau),
// so every row of the global top-N survives on its rank and results stay exact; smaller
// shards no longer start from looser thresholds than the whole database would.
static ol_status share_tau(ol_ctx *c, uint32_t nq) {
    if (!c->comm) return OL_OK;
    OL_NCCL(c, nccl_api(nullptr)->allReduce(c->tau0_d, c->tau0_d, (size_t)nq * c->n_sub, ncclUint32, ncclMin,
                                            c->comm, c->stream));
    return OL_OK;
}

// Open the other ranks' threshold arrays for in-scan sharing.  Collective (NCCL mode): every
// rank reallocates its array at the same query (identical shapes), so every rank comes here at
// the same query.  Publishing into a peer's array is safe across queries because the seed MIN
// all-reduce of query k+1 completes on a rank only after every rank finished its scan of k and
// seeded k+1.  A handle that cannot be opened (no peer access) just leaves that peer out.
static ol_status ensure_tau_peers(ol_ctx *c) {
    if (!c->comm || c->world == 1 || !c->opt_tau_share || c->tau_shared_cap == c->tau_cap) return OL_OK;
    for (auto &p : c->tau_peer)
        if (p) { cudaIpcCloseMemHandle(p); p = nullptr; }
    constexpr size_t H = sizeof(cudaIpcMemHandle_t);
    std::vector<unsigned char> hs((size_t)c->world * H, 0);
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, c->tau0_d) == cudaSuccess) memcpy(&hs[(size_t)c->rank * H], &h, H);
    cudaGetLastError();
    if (!c->hbuf_d) OL_CUDA(c, cudaMalloc((void **)&c->hbuf_d, kXchgMax * H));
    OL_CUDA(c, cudaMemcpyAsync(c->hbuf_d + (size_t)c->rank * H, &hs[(size_t)c->rank * H], H, cudaMemcpyHostToDevice,
                               c->stream));
    OL_NCCL(c, nccl_api(nullptr)->allGather(c->hbuf_d + (size_t)c->rank * H, c->hbuf_d, H, ncclUint8, c->comm,
                                            c->stream));
    OL_CUDA(c, cudaMemcpyAsync(hs.data(), c->hbuf_d, (size_t)c->world * H, cudaMemcpyDeviceToHost, c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    for (int p = 0; p < c->world && p < kXchgMax; ++p) {
        if (p == c->rank) continue;
        bool any = false;
        for (size_t b = 0; b < H; ++b) any |= hs[(size_t)p * H + b] != 0;
        if (!any) continue;
        memcpy(&h, &hs[(size_t)p * H], H);
        if (cudaIpcOpenMemHandle(&c->tau_peer[p], h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
            c->tau_peer[p] = nullptr;
            cudaGetLastError();
        }
    }
    c->tau_shared_cap = c->tau_cap;
    return OL_OK;
}

// the peer threshold arrays the scan publishes into (NCCL mode, or an emulated group)
static uint32_t peer_taus(const ol_ctx *c, uint64_t need, uint32_t **out) {
    uint32_t n = 0;
    if (!c->opt_tau_share) return 0;
    if (c->comm) {
        for (int p = 0; p < kXchgMax && n < kXchgMax - 1; ++p)
            if (c->tau_peer[p]) out[n++] = (uint32_t *)c->tau_peer[p];
    } else {
        for (const ol_ctx *o : c->emu_peers)   // tests: all linked contexts ran this shape (tau_cap >= need)
            if (n < kXchgMax - 1 && o->tau0_d && o->tau_cap >= need) out[n++] = o->tau0_d;
    }
    return n;
}

static ol_status query_body(ol_ctx *c, uint32_t nb, uint32_t M, const float *q, int32_t on_device,
                            const ol_params *p, int32_t aggregate, uint64_t per_q) {
    const uint64_t nq64 = (uint64_t)nb * M;
    const uint32_t nq = (uint32_t)nq64, N = p->N;
    ol_status st;
    c->launches = 0;
    c->used_micro = false;

    // small world-1 problems (the latency configurations): the whole sequence in one kernel
    uint64_t max_rows = 0;
    for (auto &sb : c->subs) max_rows = sb.count > max_rows ? sb.count : max_rows;
    // (not when an option forces a scan path or schedule: tests of those paths keep them)
    if (c->opt_micro && c->opt_tc == -1 && !c->opt_chunk && !c->opt_qtile && !(c->opt_tc_debug & ~32) &&
        c->world == 1 && !c->comm && max_rows <= kMicroMaxRows && max_rows > 0 &&
        (uint64_t)nq * c->rows <= kMicroMaxPairs) {
        st = ensure_prefix(c, N);
        if (st) return st;
        OL_CUDA(c, grow(&c->cand_d, &c->cand_cap, per_q * nq));
        uint32_t cap = 0;
        if (aggregate) {
            OL_CUDA(c, grow(&c->est_d, &c->est_cap, nb));
            if (nb > c->bcount_cap || !c->bcount_d) {
                OL_CUDA(c, grow(&c->bcount_d, &c->bcount_cap, nb));
                OL_CUDA(c, cudaMemsetAsync(c->bcount_d, 0, sizeof(uint32_t) * c->bcount_cap, c->stream));
            }
            cap = 32;
            while (cap < per_q * M) cap <<= 1;
        }
        const uint32_t split = micro_split(max_rows, (uint64_t)nq * c->n_sub);   // (a cluster per job)
        if (c->opt_poison) {   // (as below: outputs and scratch must be written before they are read)
            OL_CUDA(c, cudaMemsetAsync(c->cand_d, 0xA5, sizeof(ol_candidate) * c->cand_cap, c->stream));
            if (aggregate) OL_CUDA(c, cudaMemsetAsync(c->est_d, 0xA5, sizeof(ol_estimate) * c->est_cap, c->stream));
        }
        OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, 2 * sizeof(int), c->stream));
        MicroArgs ma;
        ma.split = split;
        ma.coarse = c->coarse; ma.fine = c->fine; ma.queries = q; ma.subs = c->subs_d; ma.coords = c->coords;
        ma.sub_prefix = c->prefix_d; ma.cand = c->cand_d; ma.bundle_count = c->bcount_d;
        ma.flag_nonfinite = c->flags_d;
        ma.nq = nq; ma.n_sub = c->n_sub; ma.N = N; ma.M = M; ma.kc = (uint32_t)c->kc;
        ma.check_finite = on_device ? 1 : 0;   // (host frames were checked on the host)
        ma.aggregate = aggregate ? 1 : 0;
        AggArgs &ag = ma.agg;
        ag.block_only = (uint32_t)c->opt_agg_block;
        ag.cand = c->cand_d; ag.per_bundle = (uint32_t)(per_q * M); ag.offsets = nullptr; ag.xy = nullptr;
        ag.out = c->est_d; ag.err_empty = c->flags_d + 1; ag.n_bundles = nb; ag.top_c = p->top_c;
        ag.toler_per = p->toler_per;
        const double r = p->radius_m / p->tile_m;
        ag.r2 = r * r; ag.tile_m = p->tile_m; ag.cap = cap;
        ma.prof = (c->opt_tc_debug & 32) ? c->prof_d : nullptr;
        if (ma.prof) OL_CUDA(c, cudaMemsetAsync(c->prof_d, 0, 64 * sizeof(unsigned long long), c->stream));
        {
            TimeScope ts(c, ol_ctx::T_SCAN);
            OL_LAUNCH(c, launch_micro(ma, micro_smem_bytes(max_rows, split, N, cap), c->stream));
        }
        c->used_tc = c->used_pair = false;
        c->used_micro = true;
        c->cand_fused = true;
        c->nb = nb; c->M = M; c->N = N; c->nq = nq; c->qt = 0; c->aggregate = aggregate; c->params = *p;
        c->per_bundle = per_q * M;
        c->n_cand = per_q * nq;
        c->pairs = (uint64_t)nq * c->rows;
        c->q_ready = true;
        c->finalized = true;
        return OL_OK;
    }

    // launch shape (results never depend on it): tensor-core filter or CUDA-core
    // scan, query tile, chunk size
    uint32_t tc_qb = 0, tc_stages = 0;
    // (round 2, seed + scan + merge, tensor cores vs CUDA cores: 64-B plane, 100M rows 4 frames
    // 1.014 vs 1.010 ms, 5: 1.019 vs 1.257; 10M rows 4: 0.191 vs 0.197, 5: 0.195 vs 0.223;
    // 128-B plane, 1M rows 12 frames 0.141 vs 0.128, 16: 0.140 vs 0.141)
    const uint32_t min_frames = c->opt_tc_min_frames ? (uint32_t)c->opt_tc_min_frames : (c->tc_pw == 32 ? 4u : 16u);
    const bool use_tc = c->tc_ok && (c->opt_tc == 1 || (c->opt_tc == -1 && nq >= min_frames)) &&
                        tc_shape(N, nq, c->tc_pw, &tc_qb, &tc_stages);
    uint32_t qt = c->opt_qtile > 0 ? (uint32_t)c->opt_qtile : kMaxQT;
    while (qt > 8 && scan_smem_bytes(qt, N) > 150 * 1024) qt -= 8;
    if (qt > kMaxQT) qt = kMaxQT;
    if (qt > nq) qt = nq;
    uint32_t n_qtiles = (nq + qt - 1) / qt;
    uint64_t chunk = (uint64_t)c->opt_chunk;
    if (use_tc) {
        n_qtiles = (nq + tc_qb - 1) / tc_qb;
        if (chunk == 0) {
            const uint64_t target = 148ull * 4;
            chunk = (c->rows * n_qtiles + target - 1) / target;
            if (chunk < 4096) chunk = 4096;
        }
        chunk = (chunk + 255) / 256 * 256;   // whole 256-row tiles
        if (chunk > (1ull << 24) - 256) chunk = (1ull << 24) - 256;
    } else if (chunk == 0) {
        const uint64_t target = 148ull * 8;
        chunk = (c->rows * n_qtiles + target - 1) / target;
        chunk = ((chunk + 255) / 256) * 256;
        if (chunk < 1024) chunk = 1024;
    }
    if (chunk > 0xFFFFFFFFull) chunk = 0xFFFFFFFFull;
    st = build_items(c, chunk);
    if (st) return st;
    const uint32_t n_items = (uint32_t)c->n_items();

    // buffers
    {   // (NCCL mode: whole powers of two, so the shared arrays are rarely reallocated and re-exchanged)
        size_t want = (size_t)nq * c->n_sub;
        if (c->comm && c->world > 1) { size_t r = 4096; while (r < want) r <<= 1; want = r; }
        OL_CUDA(c, grow(&c->tau0_d, &c->tau_cap, want));
    }
    // (collective in NCCL mode: every rank reaches it at the same query, whatever path it takes)
    st = ensure_tau_peers(c);
    if (st) return st;
    OL_CUDA(c, grow(&c->partial_d, &c->partial_cap, (size_t)nq * (n_items ? n_items : 1) * N));
    OL_CUDA(c, grow(&c->payload_d, &c->payload_cap, (size_t)nq * c->n_sub * N));
    if (c->opt_poison) {   // every per-query output must be written before it is read: fill them with garbage
        OL_CUDA(c, grow(&c->cand_d, &c->cand_cap, per_q * nq));
        OL_CUDA(c, grow(&c->final_d, &c->final_cap, (size_t)nq * c->n_sub * N));
        OL_CUDA(c, grow(&c->est_d, &c->est_cap, nb));
        OL_CUDA(c, cudaMemsetAsync(c->partial_d, 0xA5, sizeof(u64) * c->partial_cap, c->stream));
        OL_CUDA(c, cudaMemsetAsync(c->payload_d, 0xA5, sizeof(uint4) * c->payload_cap, c->stream));
        OL_CUDA(c, cudaMemsetAsync(c->cand_d, 0xA5, sizeof(ol_candidate) * c->cand_cap, c->stream));
        OL_CUDA(c, cudaMemsetAsync(c->final_d, 0xA5, sizeof(uint4) * c->final_cap, c->stream));
        OL_CUDA(c, cudaMemsetAsync(c->est_d, 0xA5, sizeof(ol_estimate) * c->est_cap, c->stream));
        if (c->gather_d) OL_CUDA(c, cudaMemsetAsync(c->gather_d, 0xA5, sizeof(uint4) * c->gather_cap, c->stream));
        if (c->seed_scratch) OL_CUDA(c, cudaMemsetAsync(c->seed_scratch, 0xA5, sizeof(uint32_t) * c->seed_scratch_cap, c->stream));
        if (c->q16) OL_CUDA(c, cudaMemsetAsync(c->q16, 0xA5, sizeof(uint16_t) * c->q16_cap, c->stream));
        if (c->qmeta) OL_CUDA(c, cudaMemsetAsync(c->qmeta, 0xA5, sizeof(float4) * c->qmeta_cap, c->stream));
    }
    OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, 2 * sizeof(int), c->stream));
    OL_CUDA(c, cudaMemsetAsync(c->stat_d, 0, 2 * sizeof(unsigned long long), c->stream));
    if (on_device) OL_LAUNCH(c, launch_check_finite(q, nq64 * OL_K, c->flags_d, c->stream));

    const bool seed = c->opt_tau_seed != 0;
    // tensor-core path: seed with the bound pre-pass when every subspace has >= 32 N
    // sampled rows (N <= 16: register lists); otherwise the exact sampled seed
    // (the pre-pass needs upper bounds on the full distance: only with a full-K filter)
    bool tc_seed = use_tc && seed && c->opt_tc_seed && c->seed_stride && N <= 16 && c->tc_kf == OL_K;
    for (auto &sb : c->subs)
        if (tc_seed && sb.count / c->seed_stride < 256ull * N) tc_seed = false;   // >= one full item
    if (seed && (!tc_seed || c->opt_tc_seed == 2) && !(c->opt_tc_debug & 64)) {   // (tc_debug & 64: keep the last thresholds)
        SeedArgs sa;
        sa.coarse = c->coarse; sa.fine = c->fine; sa.queries = q; sa.subs = c->subs_d;
        sa.tau0 = c->tau0_d; sa.nq = nq; sa.n_sub = c->n_sub; sa.N = N; sa.kc = (uint32_t)c->kc;
        sa.rows_pad = c->rows_pad;
        sa.select_old = c->opt_seed_select == 1;
        // splits x (count/8, at most 4096) rows per subspace, about 64k sampled pairs per
        // row... i.e. more splits for few frames; below N rows per split: no seed (+inf)
        // automatic: 8,192 samples for >= 1,024 (frame, subspace) jobs (1,024 frames: 1M rows
        // 0.657 vs 0.679 ms seed + scan, 20M 2.75 vs 2.78, 100M even), else 4,096 (few frames
        // take more splits, each a full sample)
        uint32_t S = c->opt_seed_samples ? (uint32_t)c->opt_seed_samples
                                         : ((uint64_t)nq * c->n_sub >= 1024 ? 8192u : 4096u);
        uint64_t minc = ~0ull;
        for (auto &s : c->subs) { uint64_t v = s.count / 8; if (v < S) S = (uint32_t)v; if (s.count < minc) minc = s.count; }
        sa.samples = S < 1 ? 1 : S;
        uint32_t splits = 1;
        while (splits < 16 && (uint64_t)nq * c->n_sub * splits < 148 * 2 &&
               (uint64_t)sa.samples * splits * 2 * 8 <= minc) splits *= 2;
        sa.splits = splits;
        // the two-kernel seed's scratch (acc bits of every (frame, subspace, split, sample));
        // the one-CTA-per-(frame, subspace, split) kernel runs instead beyond 2^28 entries
        // (round 2, with the CTA-per-job select, tools/seed_small.py: 8 / 64 / 256 frames at
        // 100M rows 0.036 / 0.049 / 0.051 vs 0.084 / 0.284 / 0.280 ms, 10M rows 0.034 / 0.046 /
        // 0.044 vs 0.050 / 0.147 / 0.147 ms; round 1: 1,024 frames at 100M 0.24 vs 0.62 ms)
        const uint64_t nscr = (uint64_t)nq * c->n_sub * splits * sa.samples;
        sa.scratch = nullptr;
        if (nscr <= (1ull << 28) && c->opt_seed_kernel != 0) {
            OL_CUDA(c, grow(&c->seed_scratch, &c->seed_scratch_cap, (size_t)nscr));
            sa.scratch = c->seed_scratch;
        }
        if (!sa.scratch && sa.samples > 8192) sa.samples = 8192;   // tau_seed_kernel's shared-memory bound
        TimeScope ts(c, ol_ctx::T_SEED);
        OL_LAUNCH(c, launch_fill_u32(c->tau0_d, (uint64_t)nq * c->n_sub, kInfBits, c->stream));
        OL_LAUNCH(c, launch_tau_seed(sa, c->stream));
    }
    // NCCL mode: the seeds' MIN over the ranks, at one point of the launch sequence for every
    // scan path (the collective sequence must not depend on a rank's own data)
    if (seed && !(c->opt_tc_debug & 64)) { st = share_tau(c, nq); if (st) return st; }
    if (c->opt_tc_debug & 512) { c->nq = nq; return OL_OK; }   // profiling: stop after the seed (ol_thresholds reads it)
    c->used_tc = false;
    c->used_pair = false;
    if (n_items && use_tc) {
        // CTA pairs need an even number of query blocks: a lone block (<= 128 frames) or a
        // small odd count would pay for a padding CTA's MMAs (measured: 1 block 1.8 ms single
        // vs 2.6 ms paired at C4; 2 blocks 3.7 vs 3.3 ms).  Automatic mode also wants the
        // 128-B plane and >= 10M rows: pairs halve the re-reads of a chunk's rows, which pay
        // once the plane outgrows L2; with the 64-B plane they no longer do (1,024 frames,
        // single vs pairs, final kernel: 5M rows 0.99 vs 1.03 ms, 20M 2.73 vs 2.63 (128-B
        // plane); 50M 5.46 vs 5.73, 100M 10.61 vs 10.64 (64-B plane))
        const uint32_t nqb1 = (nq + tc_qb - 1) / tc_qb;
        const bool pair = (c->opt_pair == 2 || (c->opt_pair == 1 && c->tc_pw == 64 && c->rows >= 10000000)) &&
                          (nqb1 % 2 == 0 || nqb1 >= 5);
        const uint32_t qb = tc_qb, n_qblocks = ((nq + qb - 1) / qb + (pair ? 1 : 0)) / (pair ? 2 : 1) * (pair ? 2 : 1),
                       nq_pad = n_qblocks * qb;
        OL_CUDA(c, grow((uint16_t **)&c->q16, &c->q16_cap, (size_t)nq_pad * c->tc_pw));
        OL_CUDA(c, grow(&c->qmeta, &c->qmeta_cap, nq));
        OL_CUDA(c, cudaMemsetAsync(c->tcstat_d + 2, 0, 2 * sizeof(uint32_t), c->stream));
        OL_LAUNCH(c, launch_tc_prep_queries(q, nq, nq_pad, c->q16, c->qmeta, c->tcstat_d, c->tc_kf, c->tc_pw, c->stream));
        if ((!seed || (tc_seed && c->opt_tc_seed != 2)) && !(c->opt_tc_debug & 64))
            OL_LAUNCH(c, launch_fill_u32(c->tau0_d, (uint64_t)nq * c->n_sub, kInfBits, c->stream));
        CUtensorMap map_q;
        if (!make_tc_map(&map_q, c->q16, nq_pad, qb, c->tc_pw))
            return fail(c, OL_ERR_CUDA, "cuTensorMapEncodeTiled failed");
        TcScanArgs a;
        a.bound = 0;
        a.n_peer = 0;
        a.cluster = (uint32_t)c->opt_cluster;
        a.pair = pair ? 1u : 0u;
        a.items = c->items_d; a.blk = c->blk; a.n_blk = (uint32_t)(c->rows_pad / 32); a.qmeta = c->qmeta; a.bounds = c->tcstat_d; a.nf_max = c->nf_max;
        a.g_tau = c->tau0_d; a.queries = q; a.coarse = c->coarse; a.fine = c->fine;
        a.partial = c->partial_d; a.stat_survivors = c->stat_d; a.stat_flagged = c->stat_d + 1;
        a.nq = nq; a.n_items = n_items; a.n_qblocks = n_qblocks; a.qb = qb; a.n_sub = c->n_sub;
        a.kf = c->tc_kf; a.pw = c->tc_pw;
        a.N = N; a.kc = (uint32_t)c->kc; a.stages = tc_stages; a.inline_rescore = c->opt_inline == 1 || (c->opt_inline == -1 && c->rows <= (uint64_t)c->n_sub * kInlineMaxRowsPerSub); a.dbg = (uint32_t)c->opt_tc_debug; a.prof = c->prof_d;
        if (a.dbg & 32) OL_CUDA(c, cudaMemsetAsync(c->prof_d, 0, ((a.dbg & 2048) ? 1024 : 64) * sizeof(unsigned long long), c->stream));
        if (tc_seed && !(a.dbg & 64)) {
            // bound pre-pass: tensor-core scores of every S-th row give each (frame,
            // subspace) N distinct rows with certified upper bounds on their acc
            uint64_t sch = ((c->rows_pad / c->seed_stride) * n_qblocks + 148 * 2 - 1) / (148 * 2);
            // every epilogue thread sees a quarter of its item's rows as 16-row sets: keep at
            // least 4 N sets per thread, or its list never fills and publishes nothing
            if (sch < 256ull * N) sch = 256ull * N;
            sch = (sch + 255) / 256 * 256;
            st = build_sitems(c, sch);
            if (st) return st;
            if (!c->sitems.empty()) {
                TcScanArgs pa = a;
                pa.bound = 1; pa.items = c->sitems_d; pa.n_items = (uint32_t)c->sitems.size(); pa.partial = nullptr;
                TimeScope tp(c, ol_ctx::T_SEED);
                OL_LAUNCH(c, launch_tcscan(c->map_srows, map_q, pa, (int)(pa.n_items * n_qblocks), c->stream));
            }
        }
        a.n_peer = peer_taus(c, (uint64_t)nq * c->n_sub, a.peer_tau);

        TimeScope ts(c, ol_ctx::T_SCAN);
        OL_LAUNCH(c, launch_tcscan(pair ? c->map_rows_half : c->map_rows, map_q, a, (int)(n_items * n_qblocks), c->stream));
        c->used_tc = true;
        c->used_pair = pair;
    } else if (n_items) {
        ScanArgs a;
        a.coarse = c->coarse; a.fine = c->fine; a.queries = q; a.items = c->items_d;
        a.tau0 = seed ? c->tau0_d : nullptr; a.partial = c->partial_d; a.stat_survivors = c->stat_d;
        a.nq = nq; a.n_items = n_items; a.n_qtiles = n_qtiles; a.qt = qt; a.n_sub = c->n_sub; a.N = N;
        a.rows_pad = c->rows_pad;
        TimeScope ts(c, ol_ctx::T_SCAN);
        // few frames: the TMA-fed row-pair kernel for 1-2 frames per tile (it streams the coarse
        // plane faster: tools/scan3_sweep.py, 10M rows 0.121 vs 0.140 ms at 1 frame, 100M 0.916
        // vs 0.937), the row-pair f32x2 streaming kernel for more (4 frames: 1.10 vs 0.98 ms)
        // (scan3 bulk-copies whole 32-row tiles of the coarse plane: work items must start on one)
        const bool kc3 = (c->kc == 8 || c->kc == 16 || c->kc == 32) && chunk % 32 == 0, kc2 = c->kc == 8 || c->kc == 16 || c->kc == 32 || c->kc == 64;
        if (qt <= 16 && kc3 && (c->opt_scan2 == 2 || (c->opt_scan2 == 1 && qt <= 2)))
            OL_LAUNCH(c, launch_scan3(c->kc, a, scan3_smem_bytes(qt, N, c->kc), (int)(n_items * n_qtiles), c->stream));
        else if (qt <= 16 && kc2 && c->opt_scan2)
            OL_LAUNCH(c, launch_scan2(c->kc, a, scan2_smem_bytes(qt, N, c->kc), (int)(n_items * n_qtiles), c->stream));
        else
            OL_LAUNCH(c, launch_scan(c->kc, a, scan_smem_bytes(qt, N), (int)(n_items * n_qtiles), c->stream));
    }
    MergeArgs ma;
    ma.partial = c->partial_d; ma.subs = c->cur ? c->cur->subs_d : c->subs_d; ma.coords = c->coords; ma.records = c->payload_d;
    ma.nq = nq; ma.n_items = n_items; ma.n_sub = c->n_sub; ma.N = N;
    ma.cand = nullptr; ma.sub_prefix = nullptr; ma.M = M; ma.n_cand = per_q * nq;
    ma.max_lists = c->cur ? c->cur->max_lists : (uint32_t)n_items;
    ma.force_scan = (uint32_t)c->opt_merge_scan;
    c->cand_fused = false;
    if (c->world == 1) {   // the merge also writes the candidate rows (one launch fewer)
        st = ensure_prefix(c, N);
        if (st) return st;
        OL_CUDA(c, grow(&c->cand_d, &c->cand_cap, per_q * nq));
        ma.cand = c->cand_d; ma.sub_prefix = c->prefix_d;
        c->cand_fused = true;
    }
    {
        TimeScope ts(c, ol_ctx::T_MERGE);
        OL_LAUNCH(c, launch_merge_chunks(ma, c->stream));
    }

    c->nb = nb; c->M = M; c->N = N; c->nq = nq; c->qt = qt; c->aggregate = aggregate; c->params = *p;
    c->per_bundle = per_q * M;
    c->n_cand = per_q * nq;
    c->pairs = (uint64_t)nq * c->rows;
    c->q_ready = true;
    if (c->comm) {   // the exchange inside the call: all-gather the per-rank top-N, merge
        const size_t P = (size_t)nq * c->n_sub * N;
        OL_CUDA(c, grow(&c->gather_d, &c->gather_cap, P * c->world));
        {
            TimeScope ts(c, ol_ctx::T_FINAL);
            OL_NCCL(c, nccl_api(nullptr)->allGather(c->payload_d, c->gather_d, P * sizeof(uint4), ncclUint8, c->comm,
                                                    c->stream));
        }
        st = finalize_impl(c, c->gather_d, c->world);
        if (st) return st;
        return nccl_poll(c);
    }
    if (c->world == 1) return finalize_impl(c, c->payload_d, 1);
    return OL_OK;
}

ol_status ol_thresholds(ol_ctx *c, void **dev_ptr, uint64_t *count) {
    if (!c || !dev_ptr || !count) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->tau0_d) return fail(c, OL_ERR_NOT_READY, "no query");
    *dev_ptr = c->tau0_d;
    *count = (uint64_t)c->nq * c->n_sub;
    return OL_OK;
}

ol_status ol_payload(ol_ctx *c, const void **dev_ptr, uint64_t *bytes) {
    if (!c || !dev_ptr || !bytes) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->q_ready) return fail(c, OL_ERR_NOT_READY, "no query");
    *dev_ptr = c->payload_d;
    *bytes = (uint64_t)c->nq * c->n_sub * c->N * sizeof(uint4);
    return OL_OK;
}

ol_status ol_payload_copy(ol_ctx *c, void *dst) {
    if (!c || !dst) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->q_ready) return fail(c, OL_ERR_NOT_READY, "no query");
    OL_CUDA(c, cudaSetDevice(c->device));
    OL_CUDA(c, cudaMemcpyAsync(dst, c->payload_d, (size_t)c->nq * c->n_sub * c->N * sizeof(uint4),
                               cudaMemcpyDeviceToDevice, c->stream));
    return OL_OK;
}

static ol_status finalize_tail(ol_ctx *c, const uint4 *rec);

static ol_status finalize_impl(ol_ctx *c, const uint4 *gathered, int world) {
    TimeScope ts(c, ol_ctx::T_FINAL);
    const uint32_t nq = c->nq, N = c->N, ns = c->n_sub;
    const uint4 *rec = gathered;
    if (world > 1 || gathered != c->payload_d) {
        OL_CUDA(c, grow(&c->final_d, &c->final_cap, (size_t)nq * ns * N));
        RankMergeArgs ra;
        ra.gathered = gathered; ra.records = c->final_d; ra.nq = nq; ra.n_sub = ns; ra.N = N;
        ra.world = (uint32_t)world;
        OL_LAUNCH(c, launch_merge_ranks(ra, c->stream));
        rec = c->final_d;
    }
    return finalize_tail(c, rec);
}

// candidates (and estimates) from the merged records [nq][n_sub][N]
static ol_status finalize_tail(ol_ctx *c, const uint4 *rec) {
    const uint32_t nq = c->nq, N = c->N, ns = c->n_sub;
    if (!(c->cand_fused && rec == c->payload_d)) {
        ol_status st = ensure_prefix(c, N);
        if (st) return st;
        OL_CUDA(c, grow(&c->cand_d, &c->cand_cap, c->n_cand));
        CandArgs ca;
        ca.records = rec; ca.sub_prefix = c->prefix_d; ca.out = c->cand_d; ca.nq = nq; ca.n_sub = ns;
        ca.N = N; ca.M = c->M; ca.n_cand = c->n_cand;
        OL_LAUNCH(c, launch_candidates(ca, c->stream));
    }
    if (c->aggregate) {
        OL_CUDA(c, grow(&c->est_d, &c->est_cap, c->nb));
        AggArgs ag;
        ag.block_only = (uint32_t)c->opt_agg_block;
        ag.cand = c->cand_d; ag.per_bundle = (uint32_t)c->per_bundle; ag.offsets = nullptr;
        ag.xy = nullptr; ag.out = c->est_d; ag.err_empty = c->flags_d + 1; ag.n_bundles = c->nb;
        ag.top_c = c->params.top_c; ag.toler_per = c->params.toler_per;
        const double r = c->params.radius_m / c->params.tile_m;
        ag.r2 = r * r; ag.tile_m = c->params.tile_m;
        uint32_t cap = 32;
        while (cap < c->per_bundle) cap <<= 1;
        ag.cap = cap;
        OL_LAUNCH(c, launch_aggregate(ag, c->stream));
    }
    c->finalized = true;
    return OL_OK;
}

ol_status ol_finalize(ol_ctx *c, const void *gathered, int32_t world) {
    NvtxRange nv("ol_finalize");
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->q_ready) return fail(c, OL_ERR_NOT_READY, "no query to finalize");
    if (world != c->world || !gathered)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "world %d != context world %d", world, c->world);
    OL_CUDA(c, cudaSetDevice(c->device));
    return finalize_impl(c, (const uint4 *)gathered, world);
}

// ---------------------------------------------------------------- peer-memory exchange
static constexpr size_t kMboxFlagBytes = 256;

ol_status ol_p2p_open(ol_ctx *c, int32_t world, int32_t rank, uint64_t max_payload_bytes, void *handle_out) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (world < 1 || world > kXchgMax || rank < 0 || rank >= world)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "world %d / rank %d (1 <= world <= %d)", world, rank, kXchgMax);
    if (max_payload_bytes == 0 || max_payload_bytes % sizeof(uint4))
        return fail(c, OL_ERR_INVALID_ARGUMENT, "max_payload_bytes must be a positive multiple of 16");
    OL_CUDA(c, cudaSetDevice(c->device));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    p2p_close(c);
    const size_t bytes = kMboxFlagBytes + 2 * (size_t)world * max_payload_bytes;
    if (cudaMalloc(&c->mbox_d, bytes) != cudaSuccess) { c->mbox_d = nullptr; return fail(c, OL_ERR_OOM, "mailbox of %zu bytes", bytes); }
    OL_CUDA(c, cudaMemset(c->mbox_d, 0, kMboxFlagBytes));
    c->mbox_records = max_payload_bytes / sizeof(uint4);
    c->p2p_world = world; c->p2p_rank = rank; c->p2p_epoch = 0;
    if (handle_out) {
        cudaIpcMemHandle_t h;
        OL_CUDA(c, cudaIpcGetMemHandle(&h, c->mbox_d));
        memcpy(handle_out, &h, sizeof(h));
    }
    return OL_OK;
}

ol_status ol_p2p_connect(ol_ctx *c, const void *handles) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->mbox_d) return fail(c, OL_ERR_NOT_READY, "ol_p2p_open first");
    if (!handles && c->p2p_world > 1) return fail(c, OL_ERR_INVALID_ARGUMENT, "handles is NULL");
    OL_CUDA(c, cudaSetDevice(c->device));
    for (int p = 0; p < c->p2p_world; ++p) {
        if (p == c->p2p_rank) continue;
        cudaIpcMemHandle_t h;
        memcpy(&h, (const unsigned char *)handles + (size_t)p * sizeof(h), sizeof(h));
        OL_CUDA(c, cudaIpcOpenMemHandle(&c->peer_base[p], h, cudaIpcMemLazyEnablePeerAccess));
    }
    c->p2p_ready = true;
    return OL_OK;
}

static void xchg_fill(XchgArgs &x, ol_ctx *c, int p, void *base) {
    x.flag[p] = reinterpret_cast<unsigned int *>(base);
    x.mbox[p] = reinterpret_cast<uint4 *>(static_cast<unsigned char *>(base) + kMboxFlagBytes);
    (void)c;
}

ol_status ol_p2p_finalize(ol_ctx *c) {
    NvtxRange nv("ol_p2p_finalize");
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->q_ready) return fail(c, OL_ERR_NOT_READY, "no query to finalize");
    if (!c->p2p_ready) return fail(c, OL_ERR_NOT_READY, "ol_p2p_connect first");
    const uint64_t P = (uint64_t)c->nq * c->n_sub * c->N;
    if (P > c->mbox_records) return fail(c, OL_ERR_INVALID_ARGUMENT, "payload of %llu records exceeds the mailbox (%llu)",
                                        (unsigned long long)P, (unsigned long long)c->mbox_records);
    OL_CUDA(c, cudaSetDevice(c->device));
    TimeScope ts(c, ol_ctx::T_FINAL);
    OL_CUDA(c, grow(&c->final_d, &c->final_cap, (size_t)P));
    XchgArgs x = {};
    for (int p = 0; p < c->p2p_world; ++p) xchg_fill(x, c, p, p == c->p2p_rank ? (void *)c->mbox_d : c->peer_base[p]);
    x.payload[0] = c->payload_d; x.records[0] = c->final_d;
    x.rank0 = (uint32_t)c->p2p_rank; x.world = (uint32_t)c->p2p_world; x.blocks = kXchgBlocks;
    x.epoch = ++c->p2p_epoch; x.nq = c->nq; x.n_sub = c->n_sub; x.N = c->N;
    OL_LAUNCH(c, launch_xchg_merge(x, 1, c->stream));
    return finalize_tail(c, c->final_d);
}

ol_status ol_p2p_emulate(ol_ctx **ctxs, int32_t world) {
    if (!ctxs || world < 1 || world > kXchgMax) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctxs / world");
    ol_ctx *c0 = ctxs[0];
    for (int g = 0; g < world; ++g) {
        ol_ctx *c = ctxs[g];
        if (!c || !c->mbox_d || c->p2p_world != world || c->p2p_rank != g || c->device != c0->device)
            return fail(c ? c : c0, OL_ERR_INVALID_ARGUMENT, "context %d: ol_p2p_open(world, rank = %d) on one device", g, g);
        if (!c->q_ready) return fail(c, OL_ERR_NOT_READY, "context %d has no query to finalize", g);
        if (c->nq != c0->nq || c->n_sub != c0->n_sub || c->N != c0->N || c->p2p_epoch != c0->p2p_epoch)
            return fail(c, OL_ERR_INVALID_ARGUMENT, "context %d: a different query shape or epoch", g);
        if ((uint64_t)c->nq * c->n_sub * c->N > c->mbox_records) return fail(c, OL_ERR_INVALID_ARGUMENT, "mailbox too small");
    }
    OL_CUDA(c0, cudaSetDevice(c0->device));
    XchgArgs x = {};
    for (int g = 0; g < world; ++g) {
        ol_ctx *c = ctxs[g];
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        OL_CUDA(c, grow(&c->final_d, &c->final_cap, (size_t)c->nq * c->n_sub * c->N));
        xchg_fill(x, c, g, c->mbox_d);
        x.payload[g] = c->payload_d; x.records[g] = c->final_d;
        ++c->p2p_epoch;
    }
    x.rank0 = 0; x.world = (uint32_t)world; x.blocks = kXchgBlocks; x.epoch = c0->p2p_epoch;
    x.nq = c0->nq; x.n_sub = c0->n_sub; x.N = c0->N;
    OL_LAUNCH(c0, launch_xchg_merge(x, (uint32_t)world, c0->stream));
    OL_CUDA(c0, cudaStreamSynchronize(c0->stream));
    for (int g = 0; g < world; ++g) {
        ol_status st = finalize_tail(ctxs[g], ctxs[g]->final_d);
        if (st) return st;
    }
    return OL_OK;
}

ol_status ol_tau_share_emulate(ol_ctx **ctxs, int32_t world) {
    if (!ctxs || world < 1 || world > kXchgMax) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctxs / world");
    for (int g = 0; g < world; ++g) {
        if (!ctxs[g] || ctxs[g]->device != ctxs[0]->device || ctxs[g]->comm)
            return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "context %d: NULL, another device, or owns a communicator", g);
    }
    for (int g = 0; g < world; ++g) {   // unlink from any earlier group, then link to this one
        ol_ctx *c = ctxs[g];
        for (ol_ctx *o : c->emu_peers) {
            auto &v = o->emu_peers;
            for (size_t i = 0; i < v.size(); ++i)
                if (v[i] == c) { v.erase(v.begin() + i); break; }
        }
        c->emu_peers.clear();
    }
    for (int g = 0; g < world; ++g)
        for (int o = 0; o < world; ++o)
            if (o != g) ctxs[g]->emu_peers.push_back(ctxs[o]);
    return OL_OK;
}

// ---------------------------------------------------------------- results
static ol_status check_flags(ol_ctx *c) {
    if (ol_status e = nccl_poll(c)) return e;
    int fl[2];
    OL_CUDA(c, cudaMemcpyAsync(fl, c->flags_d, sizeof(fl), cudaMemcpyDeviceToHost, c->stream));
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    if (fl[0]) return fail(c, OL_ERR_NONFINITE, "query frames hold NaN/Inf");
    if (fl[1] == 1) return fail(c, OL_ERR_EMPTY, "a bundle has no candidates");
    if (fl[1] == 2) return fail(c, OL_ERR_INVALID_ARGUMENT, "a bundle exceeds %d candidates", kAggMax);
    return OL_OK;
}

ol_status ol_candidate_count(const ol_ctx *c, uint64_t *count) {
    if (!c || !count) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->finalized) return fail(const_cast<ol_ctx *>(c), OL_ERR_NOT_READY, "no finalized query");
    *count = c->n_cand;
    return OL_OK;
}

ol_status ol_get_topk(ol_ctx *c, ol_candidate *out, uint64_t capacity, uint64_t *written) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->finalized) return fail(c, OL_ERR_NOT_READY, "no finalized query");
    if (!out || capacity < c->n_cand)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "capacity %llu < %llu candidates",
                    (unsigned long long)capacity, (unsigned long long)c->n_cand);
    OL_CUDA(c, cudaSetDevice(c->device));
    OL_CUDA(c, cudaMemcpyAsync(out, c->cand_d, sizeof(ol_candidate) * c->n_cand, cudaMemcpyDeviceToHost,
                               c->stream));
    ol_status st = check_flags(c);
    if (st) return st;
    if (written) *written = c->n_cand;
    return OL_OK;
}

ol_status ol_topk_device(ol_ctx *c, const ol_candidate **dev_ptr, uint64_t *count) {
    if (!c || !dev_ptr || !count) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->finalized) return fail(c, OL_ERR_NOT_READY, "no finalized query");
    *dev_ptr = c->cand_d;
    *count = c->n_cand;
    return OL_OK;
}

ol_status ol_get_estimates(ol_ctx *c, ol_estimate *out, uint32_t capacity) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->finalized) return fail(c, OL_ERR_NOT_READY, "no finalized query");
    if (!c->aggregate) return fail(c, OL_ERR_EMPTY, "aggregation was not requested");
    if (!out || capacity < c->nb)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "capacity %u < %u bundles", capacity, c->nb);
    OL_CUDA(c, cudaSetDevice(c->device));
    OL_CUDA(c, cudaMemcpyAsync(out, c->est_d, sizeof(ol_estimate) * c->nb, cudaMemcpyDeviceToHost,
                               c->stream));
    return check_flags(c);
}

ol_status ol_get_results(ol_ctx *c, ol_candidate *cand_out, uint64_t cand_capacity, uint64_t *written,
                         ol_estimate *est_out, uint32_t est_capacity) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->finalized) return fail(c, OL_ERR_NOT_READY, "no finalized query");
    if (!cand_out || cand_capacity < c->n_cand)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "capacity %llu < %llu candidates",
                    (unsigned long long)cand_capacity, (unsigned long long)c->n_cand);
    if (est_out && !c->aggregate) return fail(c, OL_ERR_EMPTY, "aggregation was not requested");
    if (est_out && est_capacity < c->nb)
        return fail(c, OL_ERR_INVALID_ARGUMENT, "capacity %u < %u bundles", est_capacity, c->nb);
    OL_CUDA(c, cudaSetDevice(c->device));
    OL_CUDA(c, cudaMemcpyAsync(cand_out, c->cand_d, sizeof(ol_candidate) * c->n_cand, cudaMemcpyDeviceToHost,
                               c->stream));
    if (est_out)
        OL_CUDA(c, cudaMemcpyAsync(est_out, c->est_d, sizeof(ol_estimate) * c->nb, cudaMemcpyDeviceToHost,
                                   c->stream));
    ol_status st = check_flags(c);   // (one synchronisation for both copies)
    if (st) return st;
    if (written) *written = c->n_cand;
    return OL_OK;
}

ol_status ol_aggregate(ol_ctx *c, uint32_t nb, const uint32_t *offsets, const int32_t *xy,
                       int32_t on_device, const ol_params *p, ol_estimate *out) {
    NvtxRange nv("ol_aggregate");
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    ol_status st = check_params(c, p, true);
    if (st) return st;
    if (nb == 0 || !offsets || !xy || !out) return fail(c, OL_ERR_INVALID_ARGUMENT, "empty/NULL input");
    OL_CUDA(c, cudaSetDevice(c->device));
    // tiles must lie in the database's grid when one is uploaded (a coordinate
    // outside the grid signals a DB/grid mismatch), else in [-2^30, 2^30) so that the circle
    // test's dx^2 + dy^2 cannot overflow int64
    const bool grid = c->db_ready;
    const int32_t x0 = grid ? 0 : -(1 << 30), x1 = grid ? c->grid_w : (1 << 30);
    const int32_t y0 = grid ? 0 : -(1 << 30), y1 = grid ? c->grid_h : (1 << 30);
    const uint32_t *off_d = offsets;
    const int32_t *xy_d = xy;
    uint32_t cap = 0;   // device offsets: sizes unknown on the host, kAggMax
    if (!on_device) {
        uint32_t mx = 1;
        for (uint32_t b = 0; b < nb; ++b)
            if (offsets[b + 1] > offsets[b] && offsets[b + 1] - offsets[b] > mx) mx = offsets[b + 1] - offsets[b];
        cap = 32;
        while (cap < mx && cap < (uint32_t)kAggMax) cap <<= 1;
        for (uint32_t b = 0; b < nb; ++b) {
            if (offsets[b + 1] < offsets[b]) return fail(c, OL_ERR_INVALID_ARGUMENT, "offsets decrease");
            if (offsets[b + 1] == offsets[b]) return fail(c, OL_ERR_EMPTY, "bundle %u has no candidates", b);
            if (offsets[b + 1] - offsets[b] > (uint32_t)kAggMax)
                return fail(c, OL_ERR_INVALID_ARGUMENT, "bundle %u exceeds %d candidates", b, kAggMax);
        }
        const uint64_t tot = offsets[nb];
        for (uint64_t t = offsets[0]; t < tot; ++t) {
            const int32_t x = xy[2 * t], y = xy[2 * t + 1];
            if (x < x0 || x >= x1 || y < y0 || y >= y1)
                return fail(c, OL_ERR_OUT_OF_RANGE, "tile (%d,%d) of candidate %llu outside [%d,%d)x[%d,%d)%s", x, y,
                            (unsigned long long)t, x0, x1, y0, y1, grid ? " (the database grid)" : "");
        }
        OL_CUDA(c, grow(&c->agg_off_d, &c->agg_off_cap, nb + 1));
        OL_CUDA(c, grow(&c->agg_xy_d, &c->agg_xy_cap, 2 * (tot ? tot : 1)));
        OL_CUDA(c, cudaMemcpyAsync(c->agg_off_d, offsets, sizeof(uint32_t) * (nb + 1),
                                   cudaMemcpyHostToDevice, c->stream));
        OL_CUDA(c, cudaMemcpyAsync(c->agg_xy_d, xy, sizeof(int32_t) * 2 * tot, cudaMemcpyHostToDevice,
                                   c->stream));
        off_d = c->agg_off_d;
        xy_d = c->agg_xy_d;
    }
    OL_CUDA(c, grow(&c->est_d, &c->est_cap, nb));
    OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, 3 * sizeof(int), c->stream));
    if (on_device) {   // the tiles' range, checked on the device (ol_aggregate is synchronous anyway)
        uint32_t ends[2];
        OL_CUDA(c, cudaMemcpyAsync(&ends[0], offsets, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaMemcpyAsync(&ends[1], offsets + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        if (ends[1] > ends[0])
            OL_CUDA(c, launch_check_coords(xy + 2 * (uint64_t)ends[0], ends[1] - ends[0], x0, x1, y0, y1,
                                           c->flags_d + 2, c->stream));
    }
    AggArgs ag;
    ag.block_only = (uint32_t)c->opt_agg_block;
    ag.cand = nullptr; ag.per_bundle = 0; ag.offsets = off_d; ag.xy = xy_d; ag.out = c->est_d;
    ag.err_empty = c->flags_d + 1; ag.n_bundles = nb; ag.top_c = p->top_c; ag.toler_per = p->toler_per;
    const double r = p->radius_m / p->tile_m;
    ag.r2 = r * r; ag.tile_m = p->tile_m;
    ag.cap = cap;
    OL_CUDA(c, launch_aggregate(ag, c->stream));
    OL_CUDA(c, cudaMemcpyAsync(out, c->est_d, sizeof(ol_estimate) * nb, cudaMemcpyDeviceToHost, c->stream));
    int oor = 0;
    OL_CUDA(c, cudaMemcpyAsync(&oor, c->flags_d + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    st = check_flags(c);
    c->finalized = false;  // est_d now holds these estimates, not the last query's
    if (st) return st;
    if (oor) return fail(c, OL_ERR_OUT_OF_RANGE, "device tiles outside [%d,%d)x[%d,%d)%s", x0, x1, y0, y1,
                         grid ? " (the database grid)" : "");
    return OL_OK;
}

// ---------------------------------------------------------------- NEXT-1 shift re-scoring
ol_status ol_upload_profiles(ol_ctx *c, const float *profiles, uint32_t W, int32_t on_device) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->db_ready) return fail(c, OL_ERR_NOT_READY, "upload the database first");
    if (!profiles || W < 8 || W > 1024) return fail(c, OL_ERR_INVALID_ARGUMENT, "W=%u outside 8..1024", W);
    OL_CUDA(c, cudaSetDevice(c->device));
    if (!on_device) {
        for (uint64_t t = 0; t < c->rows * W; ++t)
            if (!std::isfinite(profiles[t]))
                return fail(c, OL_ERR_NONFINITE, "profile value %llu is not finite", (unsigned long long)t);
    } else {
        OL_CUDA(c, cudaMemsetAsync(c->flags_d, 0, sizeof(int), c->stream));
        OL_CUDA(c, launch_check_finite(profiles, c->rows * W, c->flags_d, c->stream));
        int fl = 0;
        OL_CUDA(c, cudaMemcpyAsync(&fl, c->flags_d, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        if (fl) return fail(c, OL_ERR_NONFINITE, "device profiles hold NaN/Inf");
    }
    cudaFree(c->prof);
    c->prof = nullptr;
    c->prof_W = 0;
    const uint64_t R = c->rows_pad ? c->rows_pad : 32;
    OL_CUDA(c, cudaMalloc((void **)&c->prof, sizeof(float) * R * W));
    const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    uint64_t src = 0;
    for (auto &s : c->subs) {   // same tile-aligned row placement as the features
        if (s.count)
            OL_CUDA(c, cudaMemcpyAsync(c->prof + s.row_begin * W, profiles + src * W, sizeof(float) * s.count * W,
                                       kind, c->stream));
        src += s.count;
    }
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    c->prof_W = W;
    return OL_OK;
}

ol_status ol_extract_features(ol_ctx *c, const double *profiles, uint64_t n, uint32_t W, int32_t on_device,
                              float *out32, double *out64, uint8_t *degenerate, float *profile_out) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (W <= (uint32_t)OL_K || W > 2048) return fail(c, OL_ERR_INVALID_ARGUMENT, "W = %u outside 65..2048", W);
    if (n == 0) return OL_OK;
    if (!profiles) return fail(c, OL_ERR_INVALID_ARGUMENT, "profiles is NULL");
    OL_CUDA(c, cudaSetDevice(c->device));
    if (on_device) {
        OL_LAUNCH(c, launch_extract(profiles, n, W, out32, out64, degenerate, profile_out, c->stream));
        return OL_OK;
    }
    for (uint64_t t = 0; t < n * W; ++t)
        if (!std::isfinite(profiles[t]))
            return fail(c, OL_ERR_NONFINITE, "profile value %llu is not finite", (unsigned long long)t);
    double *dp = nullptr, *d64 = nullptr;
    float *d32 = nullptr, *dpo = nullptr;
    uint8_t *dd = nullptr;
    ol_status st = OL_OK;
    auto cleanup = [&]() { cudaFree(dp); cudaFree(d64); cudaFree(d32); cudaFree(dd); cudaFree(dpo); };
#define OL_EX(x)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) { cleanup(); return fail(c, OL_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); } \
    } while (0)
    OL_EX(cudaMalloc((void **)&dp, sizeof(double) * n * W));
    if (out64) OL_EX(cudaMalloc((void **)&d64, sizeof(double) * n * OL_K));
    if (out32) OL_EX(cudaMalloc((void **)&d32, sizeof(float) * n * OL_K));
    if (degenerate) OL_EX(cudaMalloc((void **)&dd, n));
    if (profile_out) OL_EX(cudaMalloc((void **)&dpo, sizeof(float) * n * W));
    OL_EX(cudaMemcpyAsync(dp, profiles, sizeof(double) * n * W, cudaMemcpyHostToDevice, c->stream));
    OL_EX(launch_extract(dp, n, W, d32, d64, dd, dpo, c->stream));
    ++c->launches;
    if (out64) OL_EX(cudaMemcpyAsync(out64, d64, sizeof(double) * n * OL_K, cudaMemcpyDeviceToHost, c->stream));
    if (out32) OL_EX(cudaMemcpyAsync(out32, d32, sizeof(float) * n * OL_K, cudaMemcpyDeviceToHost, c->stream));
    if (degenerate) OL_EX(cudaMemcpyAsync(degenerate, dd, n, cudaMemcpyDeviceToHost, c->stream));
    if (profile_out) OL_EX(cudaMemcpyAsync(profile_out, dpo, sizeof(float) * n * W, cudaMemcpyDeviceToHost, c->stream));
    OL_EX(cudaStreamSynchronize(c->stream));
#undef OL_EX
    cleanup();
    return st;
}

static ol_status shift_rescore_impl(ol_ctx *c, const float *qprof, const float *cprof, uint32_t Wc, int32_t on_device) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    NvtxRange nv("ol_shift_rescore");
    if (!c->finalized) return fail(c, OL_ERR_NOT_READY, "no finalized query");
    if (!cprof && !c->prof) return fail(c, OL_ERR_NOT_READY, "no profiles uploaded");
    if (!qprof) return fail(c, OL_ERR_INVALID_ARGUMENT, "query_profiles is NULL");
    if (cprof && (Wc < 8 || Wc > 1024)) return fail(c, OL_ERR_INVALID_ARGUMENT, "W=%u outside 8..1024", Wc);
    OL_CUDA(c, cudaSetDevice(c->device));
    const uint32_t W = cprof ? Wc : c->prof_W;
    const float *qp = qprof, *cp = cprof;
    if (!on_device) {
        for (uint64_t t = 0; t < (uint64_t)c->nq * W; ++t)
            if (!std::isfinite(qprof[t]))
                return fail(c, OL_ERR_NONFINITE, "query profile value %llu is not finite", (unsigned long long)t);
        if (cprof)
            for (uint64_t t = 0; t < c->n_cand * W; ++t)
                if (!std::isfinite(cprof[t]))
                    return fail(c, OL_ERR_NONFINITE, "candidate profile value %llu is not finite", (unsigned long long)t);
        OL_CUDA(c, grow(&c->qprof_d, &c->qprof_cap, (size_t)c->nq * W + (cprof ? c->n_cand * W : 0)));
        OL_CUDA(c, cudaMemcpyAsync(c->qprof_d, qprof, sizeof(float) * c->nq * W, cudaMemcpyHostToDevice, c->stream));
        qp = c->qprof_d;
        if (cprof) {
            OL_CUDA(c, cudaMemcpyAsync(c->qprof_d + (size_t)c->nq * W, cprof, sizeof(float) * c->n_cand * W,
                                       cudaMemcpyHostToDevice, c->stream));
            cp = c->qprof_d + (size_t)c->nq * W;
        }
    }
    OL_CUDA(c, grow(&c->shift_keys, &c->shift_cap, c->n_cand));
    ShiftArgs sa;
    sa.cand = c->cand_d; sa.subs = c->subs_d; sa.prof = c->prof; sa.cprof = cp; sa.qprof = qp; sa.keys = c->shift_keys;
    sa.n_cand = c->n_cand; sa.W = W; sa.M = c->M; sa.nq = c->nq;
    if (c->n_cand) OL_LAUNCH(c, launch_shift(sa, c->stream));
    if (!cprof && c->comm && c->n_cand)   // ranks scored only their own rows: keep the least key of every candidate
        OL_NCCL(c, nccl_api(nullptr)->allReduce(c->shift_keys, c->shift_keys, c->n_cand, ncclUint64, ncclMin, c->comm,
                                                c->stream));
    c->shift_ready = true;
    return OL_OK;
}

ol_status ol_shift_rescore(ol_ctx *c, const float *qprof, int32_t on_device) {
    return shift_rescore_impl(c, qprof, nullptr, 0, on_device);
}

ol_status ol_shift_rescore_cands(ol_ctx *c, const float *qprof, const float *cand_prof, uint32_t W, int32_t on_device) {
    if (!cand_prof) return fail(c, OL_ERR_INVALID_ARGUMENT, "cand_prof is NULL");
    return shift_rescore_impl(c, qprof, cand_prof, W, on_device);
}

ol_status ol_shift_keys(ol_ctx *c, uint64_t **dev_keys, uint64_t *count) {
    if (!c || !dev_keys || !count) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->shift_ready) return fail(c, OL_ERR_NOT_READY, "no shift re-scoring");
    *dev_keys = reinterpret_cast<uint64_t *>(c->shift_keys);
    *count = c->n_cand;
    return OL_OK;
}

ol_status ol_shift_keys_copy(ol_ctx *c, void *dst) {
    if (!c || !dst) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!c->shift_ready) return fail(c, OL_ERR_NOT_READY, "no shift re-scoring");
    OL_CUDA(c, cudaSetDevice(c->device));
    if (c->n_cand)
        OL_CUDA(c, cudaMemcpyAsync(dst, c->shift_keys, sizeof(u64) * c->n_cand, cudaMemcpyDeviceToDevice, c->stream));
    return OL_OK;
}

ol_status ol_get_shifts(ol_ctx *c, uint32_t *shift, float *dist2, uint64_t capacity) {
    if (!c) return fail(nullptr, OL_ERR_INVALID_ARGUMENT, "ctx is NULL");
    if (!c->shift_ready) return fail(c, OL_ERR_NOT_READY, "no shift re-scoring");
    if (!shift || !dist2 || capacity < c->n_cand) return fail(c, OL_ERR_INVALID_ARGUMENT, "capacity too small");
    std::vector<u64> k(c->n_cand);
    if (c->n_cand) {
        OL_CUDA(c, cudaMemcpyAsync(k.data(), c->shift_keys, sizeof(u64) * c->n_cand, cudaMemcpyDeviceToHost, c->stream));
    }
    OL_CUDA(c, cudaStreamSynchronize(c->stream));
    for (uint64_t i = 0; i < c->n_cand; ++i) {
        if (k[i] == kShiftPad) { shift[i] = 0xFFFFFFFFu; dist2[i] = INFINITY; continue; }
        shift[i] = (uint32_t)k[i];
        const uint32_t b = (uint32_t)(k[i] >> 32);
        memcpy(&dist2[i], &b, 4);
    }
    return OL_OK;
}

// ---------------------------------------------------------------- options / stats
ol_status ol_set_option(ol_ctx *c, const char *key, int64_t v) {
    if (!c || !key) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!strcmp(key, "chunk")) { if (v < 0) goto bad; c->opt_chunk = v; }
    else if (!strcmp(key, "qtile")) { if (v < 0 || v > kMaxQT) goto bad; c->opt_qtile = v; }
    else if (!strcmp(key, "tau_seed")) { if (v != 0 && v != 1) goto bad; c->opt_tau_seed = v; }
    else if (!strcmp(key, "seed_select")) { if (v < 0 || v > 1) goto bad; c->opt_seed_select = v; }
    else if (!strcmp(key, "seed_samples")) { if (v != 0 && (v < 16 || v > 32768)) goto bad; c->opt_seed_samples = v; }
    else if (!strcmp(key, "ctas")) { if (v < 0) goto bad; c->opt_ctas = v; }
    else if (!strcmp(key, "time_kernels")) { if (v != 0 && v != 1) goto bad; c->opt_time = v; }
    else if (!strcmp(key, "tc")) { if (v < -1 || v > 1) goto bad; c->opt_tc = v; }
    else if (!strcmp(key, "pair")) { if (v < 0 || v > 2) goto bad; c->opt_pair = v; }
    else if (!strcmp(key, "cluster")) { if (v != 1 && v != 2 && v != 4 && v != 8) goto bad; c->opt_cluster = v; }
    else if (!strcmp(key, "seed_kernel")) { if (v != 0 && v != 1) goto bad; c->opt_seed_kernel = v; }
    else if (!strcmp(key, "tc_k")) { if (v != 0 && (v < 16 || v > 64 || v % 16)) goto bad; c->opt_tc_k = v; }
    else if (!strcmp(key, "tc_seed")) { if (v < 0 || v > 2) goto bad; c->opt_tc_seed = v; }
    else if (!strcmp(key, "scan2")) { if (v < 0 || v > 2) goto bad; c->opt_scan2 = v; }
    else if (!strcmp(key, "tc_min_frames")) { if (v < 0) goto bad; c->opt_tc_min_frames = v; }
    else if (!strcmp(key, "tc_debug")) { if (v < 0 || v > 65535) goto bad; c->opt_tc_debug = v; }
    else if (!strcmp(key, "graph")) { if (v != 0 && v != 1) goto bad; c->opt_graph = v; }
    else if (!strcmp(key, "tau_share")) { if (v != 0 && v != 1) goto bad; c->opt_tau_share = v; }
    else if (!strcmp(key, "micro")) { if (v != 0 && v != 1) goto bad; c->opt_micro = v; }
    else if (!strcmp(key, "agg_block")) { if (v != 0 && v != 1) goto bad; c->opt_agg_block = v; }
    else if (!strcmp(key, "merge_scan")) { if (v != 0 && v != 1) goto bad; c->opt_merge_scan = v; }
    else if (!strcmp(key, "inline_rescore")) { if (v < -1 || v > 1) goto bad; c->opt_inline = v; }
    else if (!strcmp(key, "poison")) { if (v != 0 && v != 1) goto bad; c->opt_poison = v; }
    else return fail(c, OL_ERR_INVALID_ARGUMENT, "unknown option '%s'", key);
    ++c->gen;   // every option can change the launch sequence: retire a captured graph
    return OL_OK;
bad:
    return fail(c, OL_ERR_INVALID_ARGUMENT, "bad value %lld for '%s'", (long long)v, key);
}

ol_status ol_get_stat(ol_ctx *c, const char *key, int64_t *value) {
    if (!c || !key || !value) return fail(c, OL_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!strcmp(key, "survivors") && c->used_micro) *value = (int64_t)c->pairs;   // (NK10: every pair scored)
    else if (!strcmp(key, "survivors")) {
        unsigned long long v = 0;
        OL_CUDA(c, cudaMemcpyAsync(&v, c->stat_d, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        *value = (int64_t)v;
    } else if (!strcmp(key, "flagged")) {
        unsigned long long v = 0;
        OL_CUDA(c, cudaMemcpyAsync(&v, c->stat_d + 1, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        *value = (int64_t)v;
    } else if (!strncmp(key, "prof", 4)) {
        unsigned long long v[1024];
        OL_CUDA(c, cudaMemcpyAsync(v, c->prof_d, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        *value = (int64_t)v[atoi(key + 4)];
    } else if (!strcmp(key, "pairs")) *value = (int64_t)c->pairs;
    else if (!strcmp(key, "kernels")) *value = c->launches;
    else if (!strcmp(key, "graph_replays")) *value = (int64_t)c->graph_replays;
    else if (!strcmp(key, "qtile")) *value = c->qt;
    else if (!strcmp(key, "chunk")) *value = (int64_t)c->items_chunk;
    else if (!strcmp(key, "items")) *value = (int64_t)c->n_items();
    else if (!strcmp(key, "used_tc")) *value = c->used_tc ? 1 : 0;
    else if (!strcmp(key, "used_pair")) *value = c->used_pair ? 1 : 0;
    else if (!strcmp(key, "used_micro")) *value = c->used_micro ? 1 : 0;
    else if (!strcmp(key, "tc_k")) *value = (int64_t)c->tc_kf;
    else if (!strcmp(key, "tc_ok")) *value = c->tc_ok ? 1 : 0;
    else if (!strcmp(key, "nccl")) *value = c->comm ? 1 : 0;
    else if (!strcmp(key, "check") || !strcmp(key, "check_reset")) {
        // checked library only (-DOL_CHECKED): the first failed device bounds check, as
        // (translation unit << 24 | source line), 0 = none; always 0 in the product library
        OL_CUDA(c, cudaDeviceSynchronize());
        const bool r = key[5] != 0;
        uint32_t v = 0;
        for (uint32_t x : {check_scan(r), check_merge(r), check_aggregate(r), check_tcscan(r), check_shift(r),
                           check_extract(r)})
            if (!v) v = x;
        *value = v;
    }
    else if (!strcmp(key, "checked")) {
#ifdef OL_CHECKED
        *value = 1;
#else
        *value = 0;
#endif
    }
    else if (!strcmp(key, "tau_peers")) {
        uint32_t *pp[kXchgMax];
        *value = peer_taus(c, (uint64_t)c->nq * c->n_sub, pp);
    }
    else if (!strcmp(key, "nccl_version")) {
        int v = 0;
        const NcclApi *api = nccl_api(nullptr);
        if (api) api->getVersion(&v);
        *value = v;
    }
    else if (!strncmp(key, "time_", 5)) {
        // time_seed_ns / time_scan_ns / time_merge_ns / time_final_ns: summed over the
        // launches since the last read (then released); time_*_n: how many launches
        static const char *names[] = {"seed", "scan", "merge", "final"};
        int cls = -1;
        for (int k = 0; k < 4; ++k)
            if (!strncmp(key + 5, names[k], strlen(names[k]))) cls = k;
        if (cls < 0) return fail(c, OL_ERR_INVALID_ARGUMENT, "unknown stat '%s'", key);
        const bool count = strstr(key, "_n") && key[strlen(key) - 1] == 'n' && key[strlen(key) - 2] == '_';
        if (count) { *value = (int64_t)c->ev[cls].size(); return OL_OK; }
        OL_CUDA(c, cudaStreamSynchronize(c->stream));
        double ns = 0;
        for (auto &p : c->ev[cls]) {
            float ms = 0;
            OL_CUDA(c, cudaEventElapsedTime(&ms, p.first, p.second));
            ns += ms * 1e6;
            c->ev_pool.push_back(p.first);
            c->ev_pool.push_back(p.second);
        }
        c->ev[cls].clear();
        *value = (int64_t)ns;
    }
    else return fail(c, OL_ERR_INVALID_ARGUMENT, "unknown stat '%s'", key);
    return OL_OK;
}

}  // extern "C"
