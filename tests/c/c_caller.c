/*
 * c_caller.c -- the boundary used from plain C, no Python and no torch ("a C
 * caller gets the global top-N from ol_query alone").  A world-1 context WITH a NCCL
 * communicator (ol_nccl_unique_id -> ol_config.nccl_unique_id, so ol_query runs the
 * in-library exchange), a small two-subspace database of random unit vectors, bundles of
 * M = 3 frames, Algorithm 2 on; then the same query compared, field by field, with the
 * CPU oracle (liboracle.so, test infrastructure -- linked by this test only).
 *
 *   gcc -O2 -I include tests/c/c_caller.c -L paper_2006_08861_b200 -lomniloc -L oracle -loracle -lm \
 *       -Wl,-rpath,... -o c_caller && ./c_caller
 * Exit status 0 = every candidate and estimate equal; prints one summary line.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "omniloc.h"

/* the oracle's C entry points (oracle/oracle.c) */
int64_t oracle_retrieve(int n_sub, const int64_t *sub_sizes, const float *feats, const int32_t *coords, int K,
                        int n_bundles, int M, const float *frames, int N, int use_select, uint32_t *o_sub,
                        uint32_t *o_frame, uint32_t *o_bundle, uint32_t *o_qframe, float *o_acc, float *o_dist,
                        int32_t *o_x, int32_t *o_y, int64_t capacity);
int oracle_aggregate(int64_t total, const int32_t *xy, int top_c, double toler_per, double radius_m, double tile_m,
                     int32_t *out_x, int32_t *out_y, double *out_conf, int *out_low, int *out_n_ranked,
                     int32_t *ranked_xy, uint32_t *ranked_count, uint32_t *ranked_circle);

#define CHECK(call)                                                                        \
    do {                                                                                   \
        ol_status s_ = (call);                                                             \
        if (s_ != OL_OK) {                                                                 \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, s_, ol_last_error(ctx));        \
            return 2;                                                                      \
        }                                                                                  \
    } while (0)

static uint64_t rng = 0x9E3779B97F4A7C15ull;
static double urand(void) {   /* SplitMix64 -> [0, 1) */
    uint64_t z = (rng += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return (double)((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
}

int main(void) {
    enum { K = OL_K, NB = 4, M = 3, N = 10 };
    const uint64_t sizes[2] = {3000, 1700};
    const int64_t sizes64[2] = {3000, 1700};
    const uint64_t rows = sizes[0] + sizes[1];
    float *F = malloc(sizeof(float) * rows * K);
    int32_t *C = malloc(sizeof(int32_t) * rows * 2);
    for (uint64_t r = 0; r < rows; ++r) {
        double n2 = 0.0, v[K];
        for (int k = 0; k < K; ++k) { v[k] = urand(); n2 += v[k] * v[k]; }
        for (int k = 0; k < K; ++k) F[r * K + k] = (float)(v[k] / sqrt(n2));
        C[2 * r] = (int32_t)(urand() * 40);
        C[2 * r + 1] = (int32_t)(urand() * 40);
    }
    float Q[NB * M * K];
    for (int j = 0; j < NB * M; ++j) {
        const uint64_t r = (uint64_t)(urand() * rows);
        for (int k = 0; k < K; ++k) Q[j * K + k] = F[r * K + k] + (float)(1e-3 * (urand() - 0.5));
    }
    ol_ctx *ctx = NULL;
    unsigned char id[OL_NCCL_ID_BYTES];
    CHECK(ol_nccl_unique_id(id));
    ol_config cfg = {0, 0, 1, NULL, OL_K, 16, id};
    CHECK(ol_create(&cfg, &ctx));
    ol_db_desc db = {2, sizes, NULL, NULL, F, C, 40, 40, 0};
    CHECK(ol_upload_db(ctx, &db));
    CHECK(ol_set_option(ctx, "micro", 0));   /* the full launch sequence with the exchange */
    ol_params p = {N, 10, 0.2, 3.0, 0.3};
    CHECK(ol_query(ctx, NB, M, Q, 0, &p, 1));
    int64_t nccl = 0;
    CHECK(ol_get_stat(ctx, "nccl", &nccl));
    uint64_t n = 0, w = 0;
    CHECK(ol_candidate_count(ctx, &n));
    ol_candidate *got = malloc(sizeof(ol_candidate) * n);
    CHECK(ol_get_topk(ctx, got, n, &w));
    ol_estimate est[NB];
    CHECK(ol_get_estimates(ctx, est, NB));
    /* the one-synchronisation fetch gives the same bytes */
    ol_candidate *got2 = malloc(sizeof(ol_candidate) * n);
    ol_estimate est2[NB];
    uint64_t w2 = 0;
    CHECK(ol_get_results(ctx, got2, n, &w2, est2, NB));
    const int same = w2 == n && !memcmp(got, got2, sizeof(ol_candidate) * n) && !memcmp(est, est2, sizeof(est));

    /* the oracle on the same inputs */
    uint32_t *os = malloc(4 * n), *of = malloc(4 * n), *ob = malloc(4 * n), *oq = malloc(4 * n);
    float *oa = malloc(4 * n), *od = malloc(4 * n);
    int32_t *ox = malloc(4 * n), *oy = malloc(4 * n);
    const int64_t m = oracle_retrieve(2, sizes64, F, C, K, NB, M, Q, N, 0, os, of, ob, oq, oa, od, ox, oy, (int64_t)n);
    int bad = (m != (int64_t)n) || (w != n) || nccl != 1 || !same;
    for (uint64_t i = 0; !bad && i < n; ++i) {
        uint32_t ga, ra, gd, rd;
        memcpy(&ga, &got[i].dist2, 4); memcpy(&ra, &oa[i], 4);
        memcpy(&gd, &got[i].dist, 4); memcpy(&rd, &od[i], 4);
        if (got[i].subspace != os[i] || got[i].frame != of[i] || got[i].bundle != ob[i] ||
            got[i].query_frame != oq[i] || ga != ra || gd != rd || got[i].x != ox[i] || got[i].y != oy[i]) {
            fprintf(stderr, "candidate %llu differs\n", (unsigned long long)i);
            bad = 1;
        }
    }
    const uint64_t per = n / NB;
    for (int b = 0; !bad && b < NB; ++b) {
        int32_t xy[2 * 1024], rxy[2 * 64], x, y;
        uint32_t rc[64], rci[64];
        double conf;
        int low, nr;
        for (uint64_t i = 0; i < per; ++i) { xy[2 * i] = ox[b * per + i]; xy[2 * i + 1] = oy[b * per + i]; }
        oracle_aggregate((int64_t)per, xy, 10, 0.2, 3.0, 0.3, &x, &y, &conf, &low, &nr, rxy, rc, rci);
        if (est[b].x != x || est[b].y != y || est[b].confidence != conf || (int)est[b].low_confidence != low ||
            (int)est[b].n_ranked != nr) {
            fprintf(stderr, "estimate %d differs\n", b);
            bad = 1;
        }
    }
    printf("c_caller: %llu candidates and %d estimates from a world-1 NCCL context, %s the oracle\n",
           (unsigned long long)n, NB, bad ? "DIFFERENT from" : "equal to");
    ol_destroy(ctx);
    return bad;
}
