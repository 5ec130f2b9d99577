// synth.cu -- seeded, counter-based synthetic building/campus/city generator "G".
//
// SHARED INPUT GENERATOR.  It produces the inputs both the CUDA
// product path and the CPU oracle consume: per-entry fp32 descriptors and int32
// floor tiles, plus query frames.  It holds none of the hot path's arithmetic
// (no distance, no top-N, no aggregation).  It renders a circular intensity
// profile per camera pose and takes |DFT| bins 1..K, L2-normalised (the
// paper's feature), because the hot path's input *is* that
// descriptor; the oracle has its own, independently written feature extraction
// that tests/test_generator.py compares against.
//
// World model (SURVEY §8d "G", after S:387-395):
//   floor: floor_w x floor_h tiles of 0.30 m, walls at y = 0 and floor_h;
//   landmarks: n_lm per floor layout, x ~ U(0, floor_w), y = wall + N(0, 3),
//     amplitude U(0.1, 0.5), angular width U(0.05, 0.3) rad, decay 1/(1 + d/20);
//     +dup_frac duplicates copied floor_w/2 away in x ("scene similarity");
//   floors: floor_reuse of floors reuse an earlier floor's landmark layout;
//   paths: `paths` straight paths along x at y = path_y0 + p*path_dy (P:200:
//     "5 parallel paths"), frames evenly spaced;
//   profile: W samples, 0.5 + bumps at (bearing - heading) + N(0, sigma^2);
//     heading ~ U[0, 2pi) per frame (rotation invariance is exercised);
//   atlas: floor f at tile offset ((f % cols)*atlas_dx, (f / cols)*atlas_dy).
// Every random draw is a pure function of (seed, domain, counter): any shard of
// any size generates independently, on the host (OpenMP) or on the device.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#ifdef __CUDACC__
#define SYN_HD __host__ __device__ __forceinline__
#else
#define SYN_HD inline
#endif

extern "C" {
typedef struct {
    uint64_t seed;
    int32_t n_floors, paths, frames_per_path;
    int32_t W, K, n_lm;
    double dup_frac, floor_reuse, noise_sigma;
    double floor_w, floor_h, path_y0, path_dy;
    int32_t atlas_cols, atlas_dx, atlas_dy, _pad;
} syn_spec;

typedef struct {
    int32_t floor;
    double x, y, heading;
    uint64_t noise_key;
} syn_point;
}

namespace {

constexpr int kMaxLm = 256;
constexpr double kTwoPi = 6.283185307179586476925286766559;

SYN_HD uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
SYN_HD uint64_t key3(uint64_t a, uint64_t b, uint64_t c) {
    return mix64(mix64(mix64(a) ^ b) ^ c);
}
SYN_HD double unif(uint64_t k) { return (double)(mix64(k) >> 11) * (1.0 / 9007199254740992.0); }
SYN_HD double normal(uint64_t k) {
    double u1 = unif(k), u2 = unif(k ^ 0xD1B54A32D192ED03ull);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(kTwoPi * u2);
}

struct Landmark { double x, y, amp, inv2w2; };

SYN_HD int n_landmarks(const syn_spec &s) {
    int n = s.n_lm + (int)(s.n_lm * s.dup_frac + 0.5);
    return n > kMaxLm ? kMaxLm : n;
}

SYN_HD int32_t layout_of(const syn_spec &s, int32_t f) {
    if (f > 0 && unif(key3(s.seed, 11, (uint64_t)f)) < s.floor_reuse)
        return (int32_t)(mix64(key3(s.seed, 12, (uint64_t)f)) % (uint64_t)f);
    return f;
}

SYN_HD void landmark(const syn_spec &s, int32_t layout, int j, Landmark &L) {
    int ndup = n_landmarks(s) - s.n_lm;
    int stride = (ndup > 0 && s.n_lm / ndup > 1) ? s.n_lm / ndup : 1;
    int base = j < s.n_lm ? j : ((j - s.n_lm) * stride) % s.n_lm;
    uint64_t k = key3(s.seed, 20 + (uint64_t)layout * 7919ull, (uint64_t)base);
    double x = unif(k ^ 1) * s.floor_w;
    double wall = unif(k ^ 2) < 0.5 ? 0.0 : s.floor_h;
    double y = wall + 3.0 * normal(k ^ 3);
    double amp = 0.1 + 0.4 * unif(k ^ 4);
    double wid = 0.05 + 0.25 * unif(k ^ 5);
    if (j >= s.n_lm) x = fmod(x + 0.5 * s.floor_w, s.floor_w);
    L.x = x; L.y = y; L.amp = amp; L.inv2w2 = 1.0 / (2.0 * wid * wid);
}

// landmark j as seen from pose p: azimuth phi = bearing - heading, amplitude
// amp / (1 + d/20) (written over L.x / L.amp)
SYN_HD void view(const syn_point &p, Landmark &L) {
    double dx = L.x - p.x, dy = L.y - p.y;
    double d = sqrt(dx * dx + dy * dy);
    L.x = atan2(dy, dx) - p.heading;
    L.amp = L.amp / (1.0 + d / 20.0);
}

SYN_HD void entry_point(const syn_spec &s, int64_t e, syn_point &p) {
    int64_t per_floor = (int64_t)s.paths * s.frames_per_path;
    int32_t f = (int32_t)(e / per_floor);
    int64_t r = e % per_floor;
    int32_t path = (int32_t)(r / s.frames_per_path);
    int32_t i = (int32_t)(r % s.frames_per_path);
    p.floor = f;
    p.x = (i + 0.5) * s.floor_w / s.frames_per_path;
    p.y = s.path_y0 + path * s.path_dy;
    uint64_t k = key3(s.seed, 1, (uint64_t)e);
    p.heading = kTwoPi * unif(k ^ 7);
    p.noise_key = k;
}

// one profile sample (azimuth column w); lm already passed through view()
SYN_HD double profile_sample(const syn_spec &s, const Landmark *lm, int nlm, const syn_point &p,
                             int w) {
    double theta = kTwoPi * (double)w / (double)s.W;
    double v = 0.5;
    for (int j = 0; j < nlm; ++j) {
        double delta = theta - lm[j].x;
        delta -= kTwoPi * floor(delta * (1.0 / kTwoPi) + 0.5);  // wrap to [-pi, pi)
        v += lm[j].amp * exp(-delta * delta * lm[j].inv2w2);
    }
    return v + s.noise_sigma * normal(key3(p.noise_key, 99, (uint64_t)w));
}

SYN_HD void tile_of(const syn_spec &s, const syn_point &p, int32_t *xy) {
    int32_t ox = (p.floor % s.atlas_cols) * s.atlas_dx;
    int32_t oy = (p.floor / s.atlas_cols) * s.atlas_dy;
    xy[0] = ox + (int32_t)floor(p.x + 0.5);
    xy[1] = oy + (int32_t)floor(p.y + 0.5);
}

// ---------------------------------------------------------------- host render
void render_host(const syn_spec &s, const syn_point &p, double *prof, float *desc, double *desc64) {
    Landmark lm[kMaxLm];
    int nlm = n_landmarks(s);
    int32_t lay = layout_of(s, p.floor);
    for (int j = 0; j < nlm; ++j) { landmark(s, lay, j, lm[j]); view(p, lm[j]); }
    for (int w = 0; w < s.W; ++w) prof[w] = profile_sample(s, lm, nlm, p, w);
    if (!desc && !desc64) return;
    double m[1024], cosT[4096], sinT[4096];
    for (int w = 0; w < s.W; ++w) {
        cosT[w] = cos(kTwoPi * w / s.W);
        sinT[w] = sin(kTwoPi * w / s.W);
    }
    double n2 = 0;
    for (int k = 1; k <= s.K; ++k) {
        double re = 0, im = 0;
        for (int w = 0, r = 0; w < s.W; ++w, r = (r + k >= s.W) ? r + k - s.W : r + k) {
            re += prof[w] * cosT[r];   // r = (k * w) mod W
            im -= prof[w] * sinT[r];
        }
        m[k - 1] = sqrt(re * re + im * im);
        n2 += m[k - 1] * m[k - 1];
    }
    double nrm = sqrt(n2);
    for (int k = 0; k < s.K; ++k) {
        double c = nrm > 1e-12 ? m[k] / nrm : 0.0;
        if (desc) desc[k] = (float)c;
        if (desc64) desc64[k] = c;
    }
}

// ---------------------------------------------------------------- device render
// One warp per point: lanes own azimuth samples, then DFT bins; twiddles in smem.
constexpr int kWarps = 4;
__global__ void render_kernel(syn_spec s, int64_t n, int mode, int64_t e_begin,
                              const syn_point *pts, float *desc, int32_t *tiles) {
    extern __shared__ double sm[];
    double *cosT = sm, *sinT = sm + s.W;
    double *prof = sm + 2 * s.W + (threadIdx.x / 32) * s.W;
    Landmark *lmw = reinterpret_cast<Landmark *>(sm + 2 * s.W + kWarps * s.W) + (threadIdx.x / 32) * kMaxLm;
    for (int w = threadIdx.x; w < s.W; w += blockDim.x) {
        cosT[w] = cos(kTwoPi * w / s.W);
        sinT[w] = sin(kTwoPi * w / s.W);
    }
    __syncthreads();
    int lane = threadIdx.x & 31;
    int nlm = n_landmarks(s);
    for (int64_t i = (int64_t)blockIdx.x * kWarps + threadIdx.x / 32; i < n;
         i += (int64_t)gridDim.x * kWarps) {
        syn_point p;
        if (mode == 0) entry_point(s, e_begin + i, p); else p = pts[i];
        int32_t lay = layout_of(s, p.floor);
        __syncwarp();
        for (int j = lane; j < nlm; j += 32) { landmark(s, lay, j, lmw[j]); view(p, lmw[j]); }
        __syncwarp();
        for (int w = lane; w < s.W; w += 32) prof[w] = profile_sample(s, lmw, nlm, p, w);
        __syncwarp();
        double mk[4];
        double n2 = 0;
        int nb = 0;
        for (int k = lane + 1; k <= s.K; k += 32, ++nb) {
            double re = 0, im = 0;
            for (int w = 0, r = 0; w < s.W; ++w, r = (r + k >= s.W) ? r + k - s.W : r + k) {
                re += prof[w] * cosT[r];   // r = (k * w) mod W
                im -= prof[w] * sinT[r];
            }
            mk[nb] = sqrt(re * re + im * im);
            n2 += mk[nb] * mk[nb];
        }
        for (int o = 16; o; o >>= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        double nrm = sqrt(n2);
        nb = 0;
        for (int k = lane + 1; k <= s.K; k += 32, ++nb)
            desc[i * s.K + (k - 1)] = (float)(nrm > 1e-12 ? mk[nb] / nrm : 0.0);
        if (lane == 0 && tiles) tile_of(s, p, tiles + 2 * i);
    }
}

}  // namespace

extern "C" {

int64_t syn_num_entries(const syn_spec *s) {
    return (int64_t)s->n_floors * s->paths * s->frames_per_path;
}

void syn_grid(const syn_spec *s, int32_t *gw, int32_t *gh) {
    int cols = s->n_floors < s->atlas_cols ? s->n_floors : s->atlas_cols;
    int rows = (s->n_floors + s->atlas_cols - 1) / s->atlas_cols;
    *gw = cols * s->atlas_dx;
    *gh = rows * s->atlas_dy;
}

void syn_entry_points(const syn_spec *s, int64_t e_begin, int64_t n, syn_point *out) {
    for (int64_t i = 0; i < n; ++i) entry_point(*s, e_begin + i, out[i]);
}

// Query poses.  mode 0: n random test positions (random floor, path, x; lateral
// offset `offset` tiles; own heading and noise).  mode 1: one test path video of
// n frames on (floor, path) with lateral offset `offset` ("offset
// test path").
void syn_query_points(const syn_spec *s, uint64_t qseed, int mode, int64_t n, int32_t floor,
                      int32_t path, double offset, syn_point *out) {
    for (int64_t j = 0; j < n; ++j) {
        uint64_t k = key3(qseed, 2, (uint64_t)j);
        syn_point &p = out[j];
        if (mode == 0) {
            p.floor = (int32_t)(mix64(k ^ 21) % (uint64_t)s->n_floors);
            int32_t pa = (int32_t)(mix64(k ^ 22) % (uint64_t)s->paths);
            p.x = unif(k ^ 23) * s->floor_w;
            p.y = s->path_y0 + pa * s->path_dy + offset;
        } else {
            p.floor = floor;
            p.x = (j + 0.5) * s->floor_w / (double)n;
            p.y = s->path_y0 + path * s->path_dy + offset;
        }
        p.heading = kTwoPi * unif(k ^ 24);
        p.noise_key = k;
    }
}

// Host render: profiles (optional, [n][W] f64), descriptors [n][K] f32 (and/or
// f64) and tiles [n][2].
void syn_render_host(const syn_spec *s, int64_t n, const syn_point *pts, double *prof_out,
                     float *desc, double *desc64, int32_t *tiles) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        double prof[4096];
        render_host(*s, pts[i], prof, desc ? desc + i * s->K : nullptr,
                    desc64 ? desc64 + i * s->K : nullptr);
        if (prof_out) memcpy(prof_out + i * s->W, prof, sizeof(double) * s->W);
        if (tiles) tile_of(*s, pts[i], tiles + 2 * i);
    }
}

void syn_db_host(const syn_spec *s, int64_t e_begin, int64_t n, float *desc, int32_t *tiles) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < n; ++i) {
        syn_point p;
        entry_point(*s, e_begin + i, p);
        double prof[4096];
        render_host(*s, p, prof, desc + i * s->K, nullptr);
        if (tiles) tile_of(*s, p, tiles + 2 * i);
    }
}

static size_t smem_bytes(const syn_spec *s) {
    return sizeof(double) * (2 * s->W + kWarps * s->W) + sizeof(Landmark) * kWarps * kMaxLm;
}

// Device render of DB entries [e_begin, e_begin + n) (mode 0) or of given poses
// (pts on device, mode 1).  desc/tiles are device pointers.  Returns cudaError.
int syn_render_device(const syn_spec *s, int64_t n, int mode, int64_t e_begin,
                      const syn_point *pts_dev, float *desc, int32_t *tiles, void *stream) {
    if (s->W > 1024 || s->K > 128) return -1;
    size_t sm = smem_bytes(s);
    cudaFuncSetAttribute(render_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int64_t blocks = (n + kWarps - 1) / kWarps;
    if (blocks > 148 * 64) blocks = 148 * 64;
    if (blocks < 1) blocks = 1;
    render_kernel<<<(unsigned)blocks, 32 * kWarps, sm, (cudaStream_t)stream>>>(
        *s, n, mode, e_begin, pts_dev, desc, tiles);
    return (int)cudaGetLastError();
}

}  // extern "C"
