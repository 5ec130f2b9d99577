/*
 * oracle.c -- the plain, slow, obviously-correct CPU ORACLE for the hot path of
 * arXiv 2006.08861 (Hu, Zhu, Zhang, "GPU-accelerated Hierarchical Panoramic
 * Image Feature Retrieval for Indoor Localization", ICMR'16).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_2006_08861_b200/) never links, imports or executes it,
 * and it shares no code, header, table or constant with the CUDA path.
 *
 * Citation key:  P:n = /root/reference/PAPER.md line n,  S:n = SPEC.md line n.
 *
 * Every function below is the plain definition of the step it names, written
 * in the paper's order.  The precision contract is DESIGN.md reading R3
 * (SURVEY D3): fp32 inputs, d = RN32(q_k - f_k), acc = fmaf(d, d, acc) for
 * k = 0..K-1 in order, starting from +0; distance = sqrtf(acc); ranking on
 * (acc, frame index).  Compile with -ffp-contract=off so the compiler cannot
 * fuse or reorder any of it.
 *
 * Pins (tests/test_oracle_*.py): closed forms of S:56-57/S:66-67, numpy.fft
 * for the DFT, an exact rational emulation of the fmaf chain, brute-force
 * sort in Python, the paper's 825-candidate count, and
 * hand-constructed aggregation cases.
 * Parity unpinned: nothing (every function has at least one external pin).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_ERR_INVALID (-1)
#define OR_ERR_EMPTY (-2)
#define OR_ERR_RANGE (-3)
#define OR_ERR_CAPACITY (-4)

/* ------------------------------------------------------------------------ */
/* Feature: |DFT| bins 1..K of the circular profile, L2-normalised.          */
/* P:121 ("The FFT magnitude of the one-dimensional omnidirectional vector   */
/* is used as a rotation-invariant omnidirectional feature"); S:53 fixes the  */
/* unnormalised forward DFT X[k] = sum_w x[w] e^{-2 pi i k w / W}, bins       */
/* k = 1..K (DC dropped), coeffs = m/||m|| if ||m|| > 1e-12 else all-zero     */
/* and flagged degenerate.  Direct O(W*K) summation, binary64.               */
/* ------------------------------------------------------------------------ */
int oracle_extract_feature(const double *profile, int W, int K, double *coeffs,
                           int *degenerate) {
    if (W < 1 || K < 1 || K >= W) return OR_ERR_INVALID;
    double norm2 = 0.0;
    for (int k = 1; k <= K; ++k) {
        double re = 0.0, im = 0.0;
        for (int w = 0; w < W; ++w) {
            /* angle reduced exactly: (k*w) mod W, so large k*w loses nothing */
            long long r = ((long long)k * (long long)w) % W;
            double ang = 2.0 * M_PI * (double)r / (double)W;
            re += profile[w] * cos(ang);
            im -= profile[w] * sin(ang);
        }
        double m = sqrt(re * re + im * im);
        coeffs[k - 1] = m;
        norm2 += m * m;
    }
    double norm = sqrt(norm2);
    if (norm > 1e-12) {
        for (int k = 0; k < K; ++k) coeffs[k] /= norm;
        *degenerate = 0;
    } else {
        for (int k = 0; k < K; ++k) coeffs[k] = 0.0;
        *degenerate = 1;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1 stored profile: the mean-removed profile scaled  */
/* by 1/||m||, ||m|| = the norm of the |DFT| bins 1..K the descriptor is      */
/* normalised by (oracle_extract_feature above).  With this scaling the */
/* descriptor c = m/||m|| is exactly |DFT(x_hat)| on bins 1..K, so Parseval    */
/* and the reverse triangle inequality give, for every circular shift s,      */
/*   sum_w (x_hat_q[(w+s) mod W] - x_hat_d[w])^2 >= (2/W) ||c_q - c_d||^2     */
/* (bins k and W-k both contribute for a real profile, K < W/2).  Degenerate  */
/* profiles (||m|| <= 1e-12) give all zeros.  Binary64; out32 = RN32 of it.   */
/* ------------------------------------------------------------------------ */
int oracle_shift_profile(const double *profile, int W, int K, double *out64, float *out32) {
    if (W < 1 || K < 1 || K >= W) return OR_ERR_INVALID;
    double *coeffs = (double *)malloc(sizeof(double) * (size_t)K);
    /* ||m|| is the descriptor's normaliser: recompute the bins, keep the norm */
    double norm2 = 0.0;
    for (int k = 1; k <= K; ++k) {
        double re = 0.0, im = 0.0;
        for (int w = 0; w < W; ++w) {
            long long r = ((long long)k * (long long)w) % W;
            double ang = 2.0 * M_PI * (double)r / (double)W;
            re += profile[w] * cos(ang);
            im -= profile[w] * sin(ang);
        }
        double m = sqrt(re * re + im * im);
        coeffs[k - 1] = m;
        norm2 += m * m;
    }
    free(coeffs);
    double norm = sqrt(norm2);
    double mean = 0.0;
    for (int w = 0; w < W; ++w) mean += profile[w];
    mean /= (double)W;
    for (int w = 0; w < W; ++w) {
        double v = norm > 1e-12 ? (profile[w] - mean) / norm : 0.0;
        if (out64) out64[w] = v;
        if (out32) out32[w] = (float)v;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* calculateDistance (Alg. 1 step 7; Euclidean per P:202).  The fp32  */
/* fixed-order chain of reading R3.  Returns acc = squared distance.         */
/* ------------------------------------------------------------------------ */
float oracle_acc(const float *q, const float *f, int K) {
    float acc = 0.0f;
    for (int k = 0; k < K; ++k) {
        float d = q[k] - f[k];
        acc = fmaf(d, d, acc);
    }
    return acc;
}

float oracle_distance(const float *q, const float *f, int K) {
    return sqrtf(oracle_acc(q, f, K));
}

/* acc for one query against n rows of F ([n][K], row-major).  Each entry's  */
/* chain is independent of every other entry's, so the loop over entries may */
/* run on several host threads without changing any arithmetic.             */
void oracle_acc_many(const float *q, const float *F, int64_t n, int K, float *acc) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; ++t) acc[t] = oracle_acc(q, F + t * (int64_t)K, K);
}

/* ------------------------------------------------------------------------ */
/* selectTopCandidates (Alg. 1 step 10; "top N"): the N        */
/* smallest distances of one subspace, ascending, ties by ascending frame    */
/* index; if |n_i| < N all of them.  Sort-all definition.    */
/* ------------------------------------------------------------------------ */
typedef struct { float acc; uint32_t t; } or_pair;

static int cmp_pair(const void *a, const void *b) {
    const or_pair *x = (const or_pair *)a, *y = (const or_pair *)b;
    if (x->acc < y->acc) return -1;
    if (x->acc > y->acc) return 1;
    return (x->t < y->t) ? -1 : (x->t > y->t) ? 1 : 0;
}

int64_t oracle_topn_sortall(const float *acc, int64_t n, int N, uint32_t *idx_out,
                            float *acc_out) {
    if (n <= 0 || N <= 0) return 0;
    or_pair *p = (or_pair *)malloc(sizeof(or_pair) * (size_t)n);
    if (!p) return OR_ERR_INVALID;
    for (int64_t t = 0; t < n; ++t) { p[t].acc = acc[t]; p[t].t = (uint32_t)t; }
    qsort(p, (size_t)n, sizeof(or_pair), cmp_pair);
    int64_t c = n < N ? n : N;
    for (int64_t r = 0; r < c; ++r) { idx_out[r] = p[r].t; acc_out[r] = p[r].acc; }
    free(p);
    return c;
}

/* The same definition ("the N smallest under (acc, index)") computed by one */
/* pass that keeps the N smallest seen so far in a sorted array: for DBs too */
/* large to sort per query.  tests/test_oracle_retrieval.py checks it equals */
/* the sort-all version, ties included.                                       */
int64_t oracle_topn_select(const float *acc, int64_t n, int N, uint32_t *idx_out,
                           float *acc_out) {
    if (n <= 0 || N <= 0) return 0;
    int64_t c = 0;
    for (int64_t t = 0; t < n; ++t) {
        float a = acc[t];
        /* (a, t) is larger than every kept element with equal acc (t grows). */
        if (c == N && !(a < acc_out[c - 1])) continue;
        int64_t pos = (c == N) ? N - 1 : c;
        while (pos > 0 && a < acc_out[pos - 1]) {
            acc_out[pos] = acc_out[pos - 1];
            idx_out[pos] = idx_out[pos - 1];
            --pos;
        }
        acc_out[pos] = a;
        idx_out[pos] = (uint32_t)t;
        if (c < N) ++c;
    }
    return c;
}

/* ------------------------------------------------------------------------ */
/* selectNearbyFrames (Alg. 1 step 2; window shape P:139): frames     */
/* m-(M-1)/2 .. m+(M-1)/2, shifted to stay inside the sequence and keeping   */
/* min(M, n_frames) frames.                                          */
/* ------------------------------------------------------------------------ */
int oracle_select_window(uint32_t n_frames, uint32_t m, uint32_t M, uint32_t *first,
                         uint32_t *len) {
    if (M == 0 || (M % 2) == 0) return OR_ERR_INVALID;
    if (m >= n_frames) return OR_ERR_RANGE;
    uint32_t L = M < n_frames ? M : n_frames;
    int64_t f = (int64_t)m - (int64_t)((M - 1) / 2);
    if (f < 0) f = 0;
    if (f > (int64_t)(n_frames - L)) f = (int64_t)(n_frames - L);
    *first = (uint32_t)f;
    *len = L;
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 as a whole: for every bundle b, query frame j and       */
/* subspace i, compare q_j with every f_t^i (t = 1..|n_i|) and keep    */
/* the top N.  Output concatenated in (bundle, frame, subspace, rank) order   */
/* with the geo-referenced tile of each candidate.     */
/* feats: all subspaces' rows back to back, [sum |n_i|][K]; coords [..][2].   */
/* ------------------------------------------------------------------------ */
int64_t oracle_retrieve(int n_sub, const int64_t *sub_sizes, const float *feats,
                        const int32_t *coords, int K, int n_bundles, int M,
                        const float *frames, int N, int use_select,
                        uint32_t *o_sub, uint32_t *o_frame, uint32_t *o_bundle,
                        uint32_t *o_qframe, float *o_acc, float *o_dist, int32_t *o_x,
                        int32_t *o_y, int64_t capacity) {
    if (n_sub <= 0 || K <= 0 || N <= 0 || M <= 0 || n_bundles < 0) return OR_ERR_INVALID;
    int64_t *off = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_sub + 1));
    int64_t maxn = 0;
    off[0] = 0;
    for (int i = 0; i < n_sub; ++i) {
        if (sub_sizes[i] <= 0) { free(off); return OR_ERR_INVALID; }
        off[i + 1] = off[i] + sub_sizes[i];
        if (sub_sizes[i] > maxn) maxn = sub_sizes[i];
    }
    float *acc = (float *)malloc(sizeof(float) * (size_t)maxn);
    uint32_t *idx = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)N);
    float *tacc = (float *)malloc(sizeof(float) * (size_t)N);
    int64_t w = 0;
    int rc = OR_OK;
    for (int b = 0; b < n_bundles && rc == OR_OK; ++b) {
        for (int j = 0; j < M && rc == OR_OK; ++j) {
            const float *q = frames + ((int64_t)b * M + j) * K;
            for (int i = 0; i < n_sub; ++i) {
                const float *F = feats + off[i] * K;
                oracle_acc_many(q, F, sub_sizes[i], K, acc);
                int64_t c = use_select ? oracle_topn_select(acc, sub_sizes[i], N, idx, tacc)
                                       : oracle_topn_sortall(acc, sub_sizes[i], N, idx, tacc);
                if (c < 0) { rc = OR_ERR_INVALID; break; }
                if (w + c > capacity) { rc = OR_ERR_CAPACITY; break; }
                for (int64_t r = 0; r < c; ++r, ++w) {
                    o_sub[w] = (uint32_t)i;
                    o_frame[w] = idx[r];
                    o_bundle[w] = (uint32_t)b;
                    o_qframe[w] = (uint32_t)j;
                    o_acc[w] = tacc[r];
                    o_dist[w] = sqrtf(tacc[r]);
                    o_x[w] = coords[(off[i] + idx[r]) * 2 + 0];
                    o_y[w] = coords[(off[i] + idx[r]) * 2 + 1];
                }
            }
        }
    }
    free(acc); free(idx); free(tacc); free(off);
    return rc == OR_OK ? w : rc;
}

/* ------------------------------------------------------------------------ */
/* Algorithm 2 with the prose of P:197:                          */
/*   1. bin every candidate into its 30 cm tile (locationDistriArray);       */
/*   2. rank the non-zero tiles by count, descending (ties (y, x) ascending,  */
/*      S:270), keep the first TopC;                                          */
/*   3. for each ranked tile in order, count the candidates inside the       */
/*      tolerance circle of radius radius_m around it ("count the total      */
/*      number of candidates within this circle"; tile-centre          */
/*      distance, inclusive) and return the first whose count is      */
/*      > NumOfAllCandidates x tolerPer (strict);                     */
/*   4. if none passes (the listing leaves FinalPosition unset):   */
/*      the ranked tile with the largest circle count, earliest rank on ties, */
/*      flagged low-confidence.                                */
/* The circle count is the literal definition: a loop over all candidates.   */
/* ------------------------------------------------------------------------ */
typedef struct { int32_t x, y; uint32_t count; } or_tile;

static int cmp_yx(const void *a, const void *b) {
    const int32_t *p = (const int32_t *)a, *q = (const int32_t *)b; /* (x, y) */
    if (p[1] != q[1]) return p[1] < q[1] ? -1 : 1;
    if (p[0] != q[0]) return p[0] < q[0] ? -1 : 1;
    return 0;
}

static int cmp_rank(const void *a, const void *b) {
    const or_tile *p = (const or_tile *)a, *q = (const or_tile *)b;
    if (p->count != q->count) return p->count > q->count ? -1 : 1;
    if (p->y != q->y) return p->y < q->y ? -1 : 1;
    if (p->x != q->x) return p->x < q->x ? -1 : 1;
    return 0;
}

int oracle_aggregate(int64_t total, const int32_t *xy, int top_c, double toler_per,
                     double radius_m, double tile_m, int32_t *out_x, int32_t *out_y,
                     double *out_conf, int *out_low, int *out_n_ranked,
                     int32_t *ranked_xy, uint32_t *ranked_count, uint32_t *ranked_circle) {
    if (total <= 0) return OR_ERR_EMPTY;
    if (top_c <= 0 || !(toler_per > 0.0 && toler_per <= 1.0) || !(radius_m > 0.0) ||
        !(tile_m > 0.0))
        return OR_ERR_INVALID;
    /* step 1: 2-D binning -- sort a copy by tile, count runs */
    int32_t *s = (int32_t *)malloc(sizeof(int32_t) * 2 * (size_t)total);
    memcpy(s, xy, sizeof(int32_t) * 2 * (size_t)total);
    qsort(s, (size_t)total, 2 * sizeof(int32_t), cmp_yx);
    or_tile *tiles = (or_tile *)malloc(sizeof(or_tile) * (size_t)total);
    int64_t nt = 0;
    for (int64_t c = 0; c < total; ++c) {
        if (nt > 0 && tiles[nt - 1].x == s[2 * c] && tiles[nt - 1].y == s[2 * c + 1]) {
            tiles[nt - 1].count++;
        } else {
            tiles[nt].x = s[2 * c]; tiles[nt].y = s[2 * c + 1]; tiles[nt].count = 1; ++nt;
        }
    }
    /* step 2: rank, keep TopC */
    qsort(tiles, (size_t)nt, sizeof(or_tile), cmp_rank);
    int nr = (int)(nt < top_c ? nt : top_c);
    /* step 3: tolerance circles (radius in tiles; squared in binary64) */
    double r = radius_m / tile_m;
    double r2 = r * r;
    double thresh = toler_per * (double)total;
    int chosen = -1, best = 0;
    for (int i = 0; i < nr; ++i) {
        uint32_t circle = 0;
        for (int64_t c = 0; c < total; ++c) {
            int64_t dx = (int64_t)xy[2 * c] - tiles[i].x;
            int64_t dy = (int64_t)xy[2 * c + 1] - tiles[i].y;
            if ((double)(dx * dx + dy * dy) <= r2) ++circle;
        }
        ranked_xy[2 * i] = tiles[i].x;
        ranked_xy[2 * i + 1] = tiles[i].y;
        ranked_count[i] = tiles[i].count;
        ranked_circle[i] = circle;
        if (chosen < 0 && (double)circle > thresh) chosen = i;
        if (circle > ranked_circle[best]) best = i; /* strict: earliest rank on ties */
    }
    int low = 0;
    if (chosen < 0) { chosen = best; low = 1; }
    *out_x = tiles[chosen].x;
    *out_y = tiles[chosen].y;
    *out_conf = (double)ranked_circle[chosen] / (double)total;
    *out_low = low;
    *out_n_ranked = nr;
    free(s); free(tiles);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* NEXT-1: explicit circular-shift distance between two           */
/* omnidirectional profiles -- the north star's "score ... over all circular  */
/* shifts (rotations)", P:121 ("FFT magnitude ... rotation-invariant" is the  */
/* descriptor this complements).  For every shift s = 0..W-1 the same fp32    */
/* fixed-order chain as oracle_acc (DESIGN R3) over w = 0..W-1 of             */
/* d = RN32(q[(w+s) mod W] - p[w]); returns the minimum and its smallest      */
/* argmin (a rotation of the camera heading by s columns).                    */
/* ------------------------------------------------------------------------ */
float oracle_shift_distance(const float *q, const float *p, int W, int *argmin) {
    float best = INFINITY;
    int bs = 0;
    for (int s = 0; s < W; ++s) {
        float acc = 0.0f;
        for (int w = 0; w < W; ++w) {
            float d = q[(w + s) % W] - p[w];
            acc = fmaf(d, d, acc);
        }
        if (acc < best) { best = acc; bs = s; }
    }
    *argmin = bs;
    return best;
}

/* Timing infrastructure (bench.py's cpu_baseline: single-thread and all-core rates); no
 * arithmetic.  n < 1 restores the OpenMP default. */
void oracle_set_threads(int n) { omp_set_num_threads(n > 0 ? n : omp_get_num_procs()); }
