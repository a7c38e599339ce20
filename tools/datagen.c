/*
 * Synthetic dataset generators for the benchmark and the parity tests.
 *
 * Two generators, both deterministic and bit-identical on any host with the
 * same libm (they use only splitmix64 integer draws plus sqrt/log/cos/sin in
 * double, exactly like the reference):
 *
 *  1. tsdg_make_synthetic / tsdg_make_synthetic_split — a restatement of the
 *     reference's Gaussian-mixture generator (bench.cpp:80-129, Rng64 from
 *     common.hpp:27-61).  Used for bit-exact parity inputs.  Pinned against
 *     the reference by tests/test_datagen.py.
 *
 *  2. tsdg_make_lowlid — the "low-LID clustered" recall/QPS generator of
 *     SURVEY.md §8(d) recipe 2: latent = make_synthetic_split(n, nq, L, ...),
 *     embedded with a fixed L x d matrix M (entries gauss()/sqrt(L)) and
 *     0.01*gauss() noise; gauss() = sqrt(-2 ln max(u1,1e-300)) cos(2 pi u2),
 *     all from one Rng64(seed ^ 0xABCDEF) stream: M row-major first, then the
 *     noise of the base rows, then of the queries (j ascending).  splitmix64 is
 *     a counter generator, so the noise stream is split across threads by
 *     jumping the state (draw i uses state seed + (i+1)*golden).
 *
 * Built into paper_2204_00824_b200/_lib/libtsdg_datagen.so (not the search
 * path; it only makes inputs).  Compiled with -ffp-contract=off.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL

static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t rng_next(uint64_t* s) {
    *s += GOLDEN;
    return mix64(*s);
}
static inline uint32_t rng_below(uint64_t* s, uint32_t n) { return (uint32_t)(rng_next(s) % n); }
static inline double rng_unit(uint64_t* s) {
    return (double)(rng_next(s) >> 11) * 0x1.0p-53;
}
static inline uint64_t rng_fork(uint64_t s, uint64_t i) {
    return mix64(s ^ (0xD1B54A32D192ED03ULL * (i + 1)));
}

/* bench.cpp:80-112 */
int tsdg_make_synthetic(uint32_t n, uint32_t d, uint32_t clusters, float spread,
                        uint64_t seed, float* out) {
    if (clusters < 1 || d < 1) return 1;
    const uint64_t base = seed;
    uint64_t center_rng = rng_fork(base, 0);
    float* centers = (float*)malloc(sizeof(float) * (size_t)clusters * d);
    if (!centers) return 2;
    for (size_t i = 0; i < (size_t)clusters * d; ++i) centers[i] = (float)rng_unit(&center_rng);
    const uint64_t row_base = rng_fork(base, 1);
    const double tau = 6.283185307179586;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        uint64_t rng = rng_fork(row_base, (uint64_t)i);
        const uint32_t c = rng_below(&rng, clusters);
        const float* center = centers + (size_t)c * d;
        float* row = out + (size_t)i * d;
        for (uint32_t j = 0; j < d; j += 2) {
            double u1 = rng_unit(&rng);
            if (u1 < 1e-300) u1 = 1e-300;
            const double u2 = rng_unit(&rng);
            const double r = sqrt(-2.0 * log(u1));
            const double z0 = r * cos(tau * u2);
            const double z1 = r * sin(tau * u2);
            row[j] = center[j] + spread * (float)z0;
            if (j + 1 < d) row[j + 1] = center[j + 1] + spread * (float)z1;
        }
    }
    free(centers);
    return 0;
}

/* bench.cpp:114-129: n + nq points from one mixture, split base | queries. */
int tsdg_make_synthetic_split(uint32_t n, uint32_t nq, uint32_t d, uint32_t clusters,
                              float spread, uint64_t seed, float* base, float* queries) {
    float* all = (float*)malloc(sizeof(float) * ((size_t)n + nq) * d);
    if (!all) return 2;
    const int rc = tsdg_make_synthetic(n + nq, d, clusters, spread, seed, all);
    if (rc == 0) {
        memcpy(base, all, sizeof(float) * (size_t)n * d);
        memcpy(queries, all + (size_t)n * d, sizeof(float) * (size_t)nq * d);
    }
    free(all);
    return rc;
}

static inline double gauss_at(uint64_t state) {
    /* two consecutive draws starting from `state` */
    uint64_t s = state;
    double u1 = rng_unit(&s);
    if (u1 < 1e-300) u1 = 1e-300;
    const double u2 = rng_unit(&s);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
}

/* SURVEY.md §8(d) recipe 2 ("low-LID clustered"). */
int tsdg_make_lowlid(uint32_t n, uint32_t nq, uint32_t d, uint32_t latent_dim,
                     uint32_t clusters, float spread, uint64_t seed, float noise,
                     float* base, float* queries) {
    const uint32_t L = latent_dim;
    float* lb = (float*)malloc(sizeof(float) * (size_t)n * L);
    float* lq = (float*)malloc(sizeof(float) * (size_t)nq * L);
    float* M = (float*)malloc(sizeof(float) * (size_t)L * d);
    if (!lb || !lq || !M) {
        free(lb); free(lq); free(M);
        return 2;
    }
    int rc = tsdg_make_synthetic_split(n, nq, L, clusters, spread, seed, lb, lq);
    if (rc != 0) {
        free(lb); free(lq); free(M);
        return rc;
    }
    const uint64_t s0 = seed ^ 0xABCDEFULL;
    const double inv = 1.0 / sqrt((double)L);
    for (size_t i = 0; i < (size_t)L * d; ++i) {
        M[i] = (float)(gauss_at(s0 + (uint64_t)(2 * i) * GOLDEN) * inv);
    }
    const uint64_t noise0 = (uint64_t)L * d;  /* gauss index of the first noise draw */
    const uint64_t total = (uint64_t)n + nq;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < (int64_t)total; ++r) {
        const float* lat = r < (int64_t)n ? lb + (size_t)r * L : lq + (size_t)(r - n) * L;
        float* out = r < (int64_t)n ? base + (size_t)r * d : queries + (size_t)(r - n) * d;
        for (uint32_t j = 0; j < d; ++j) {
            float acc = 0.0f;
            for (uint32_t l = 0; l < L; ++l) acc += lat[l] * M[(size_t)l * d + j];
            const uint64_t g = noise0 + (uint64_t)r * d + j;
            out[j] = acc + (float)(noise * gauss_at(s0 + 2 * g * GOLDEN));
        }
    }
    free(lb); free(lq); free(M);
    return 0;
}

/* FNV-1a over the raw bytes — dataset identity check (generator drift). */
uint64_t tsdg_fnv1a(const void* p, uint64_t nbytes) {
    const unsigned char* b = (const unsigned char*)p;
    uint64_t h = 0xcbf29ce484222325ULL;
    for (uint64_t i = 0; i < nbytes; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

/* Exact per-edge distances of a CSR graph: dist[j] = kernel(row(u), row(t_j)) in the
 * reference's sequential fp32 order (vectors.hpp:36-49; L2 only: metric 0 ->
 * squared L2, 1 -> 1 - dot, 2 -> -dot).  Used to rebuild a TSDG file from its
 * packed transport form; the result is checked against the original checksum. */
void tsdg_edge_distances(const float* base, uint32_t n, uint32_t d, int metric,
                         const uint64_t* offsets, const uint32_t* targets, float* out) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t u = 0; u < (int64_t)n; ++u) {
        const float* a = base + (size_t)u * d;
        for (uint64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
            const float* b = base + (size_t)targets[j] * d;
            float acc = 0.0f;
            if (metric == 0) {
                for (uint32_t i = 0; i < d; ++i) {
                    const float diff = a[i] - b[i];
                    acc += diff * diff;
                }
                out[j] = acc;
            } else {
                for (uint32_t i = 0; i < d; ++i) acc += a[i] * b[i];
                out[j] = metric == 1 ? 1.0f - acc : -acc;
            }
        }
    }
}
