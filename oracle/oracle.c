/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Never linked into the product library.
 *
 * A plain-C restatement of the reference's replication-runner path (arXiv 1501.01405
 * reference implementation, /root/reference/proj), used by tests/ to check the CUDA
 * path and cross-checked itself against oracle/_ref (the reference sources compiled
 * unmodified) and the reference's golden vectors (tests/golden/, see
 * tools/gen_golden.py). Built by oracle/Makefile with the reference's FP flags:
 * -O2 -ffp-contract=off (proj/CMakeLists.txt:12-13), so a*b+c is never fused.
 *
 * Parity pinned: taus88.golden (proj/taus88.golden), sweep_pi.golden
 * (proj/tests/golden/sweep_pi.golden) and per-replication outputs of the reference
 * itself (tests/golden/replications.json), see tests/test_oracle.py.
 *
 * Third-party arithmetic: mm1 calls glibc libm `log` exactly as the reference does
 * (models.hpp:67,75 via std::log). On x86-64 glibc 2.39 this is ifunc-dispatched; the
 * FMA variant is what an FMA-capable host runs. The device port of that variant lives
 * in paper_1501_01405_b200/csrc/glibc_log.cuh and is pinned against this libm.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* status codes: same values as include/wlp_b200.h */
enum { OK = 0, EDOMAIN = 1, ESPACING = 4, ENOMEM_ = 7 };

/* ---- rng (proj/src/rng.cpp) ------------------------------------------------------ */

/* make_rng_state, rng.cpp:29-34: components below 2/8/16 get the minimum OR-ed in. */
static void make_state(uint32_t s[3]) {
    if (s[0] < 2u) s[0] |= 2u;
    if (s[1] < 8u) s[1] |= 8u;
    if (s[2] < 16u) s[2] |= 16u;
}

/* splitmix64, rng.cpp:19-25. */
static uint64_t splitmix64(uint64_t* x) {
    *x += 0x9e3779b97f4a7c15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

/* rng_state_from_seed, rng.cpp:36-40: high halves of three splitmix64 outputs, passed as
 * make_rng_state(word(), word(), word()). C++ leaves the evaluation order of those three
 * calls unspecified; g++ on x86-64 (the reference's toolchain) evaluates them right to
 * left, so s3 gets the FIRST splitmix output and s1 the third. Pinned by
 * tests/golden/spacing.json ("master"), produced by the reference itself. */
int oracle_master_from_seed(uint64_t seed, uint32_t s[3]) {
    uint64_t x = seed;
    for (int i = 2; i >= 0; --i) s[i] = (uint32_t)(splitmix64(&x) >> 32);
    make_state(s);
    return OK;
}

/* taus_next, rng.cpp:42-51 — L'Ecuyer taus88, components (k,q,s) = (31,13,12),
 * (29,2,4), (28,3,17) (tests/support/taus_reference.hpp:21). */
static uint32_t taus_next(uint32_t s[3]) {
    uint32_t b;
    b = ((s[0] << 13) ^ s[0]) >> 19;
    s[0] = ((s[0] & 0xFFFFFFFEu) << 12) ^ b;
    b = ((s[1] << 2) ^ s[1]) >> 25;
    s[1] = ((s[1] & 0xFFFFFFF8u) << 4) ^ b;
    b = ((s[2] << 3) ^ s[2]) >> 11;
    s[2] = ((s[2] & 0xFFFFFFF0u) << 17) ^ b;
    return s[0] ^ s[1] ^ s[2];
}

/* uniform01, rng.cpp:53-55: exact u32 * 2^-32. */
static double uniform01(uint32_t s[3]) { return (double)taus_next(s) * 0x1p-32; }

int oracle_taus_stream(uint32_t a, uint32_t b, uint32_t c, int64_t n, uint32_t* out) {
    uint32_t s[3] = {a, b, c};
    make_state(s);
    for (int64_t i = 0; i < n; ++i) out[i] = taus_next(s);
    return OK;
}

/* random_spacing, rng.cpp:67-87: stream i = remap(next 3 master draws), redrawn while
 * it equals an earlier stream (std::set there, an open-addressing set here); 1000
 * rejections for one stream is an Error. */
int oracle_random_spacing(uint64_t master_seed, int64_t count, uint32_t* s1, uint32_t* s2,
                          uint32_t* s3) {
    uint32_t m[3];
    oracle_master_from_seed(master_seed, m);
    uint64_t cap = 16;
    while (cap < (uint64_t)count * 2) cap <<= 1;
    int64_t* slot = (int64_t*)malloc(cap * sizeof(int64_t));
    if (!slot) return ENOMEM_;
    for (uint64_t i = 0; i < cap; ++i) slot[i] = -1;
    for (int64_t i = 0; i < count; ++i) {
        int attempts = 0;
        for (;;) {
            uint32_t k[3];
            k[0] = taus_next(m);
            k[1] = taus_next(m);
            k[2] = taus_next(m);
            make_state(k);
            uint64_t h = ((uint64_t)k[0] * 0x9E3779B97F4A7C15ull) ^
                         ((uint64_t)k[1] * 0xC2B2AE3D27D4EB4Full) ^ ((uint64_t)k[2] << 17);
            uint64_t j = (h ^ (h >> 29)) & (cap - 1);
            int dup = 0;
            while (slot[j] >= 0) {
                int64_t o = slot[j];
                if (s1[o] == k[0] && s2[o] == k[1] && s3[o] == k[2]) {
                    dup = 1;
                    break;
                }
                j = (j + 1) & (cap - 1);
            }
            if (!dup) {
                slot[j] = i;
                s1[i] = k[0];
                s2[i] = k[1];
                s3[i] = k[2];
                break;
            }
            if (++attempts >= 1000) {
                free(slot);
                return ESPACING;
            }
        }
    }
    free(slot);
    return OK;
}

/* ---- models (proj/include/warpsim/models.hpp) ----------------------------------- */

/* pi_replication_u, models.hpp:49-59. */
double oracle_pi_replication(int64_t draws, const uint32_t seed[3]) {
    uint32_t s[3] = {seed[0], seed[1], seed[2]};
    double c = 0.0;
    for (int64_t i = 0; i < draws; ++i) {
        const double x = uniform01(s);
        const double y = uniform01(s);
        c = c + ((x * x + y * y <= 1.0) ? 1.0 : 0.0);
    }
    return (4.0 * c) / (double)draws;
}

/* mm1_replication_u, models.hpp:61-84 (Lindley recursion, glibc log). */
void oracle_mm1_replication(int64_t clients, double lambda, double mu, const uint32_t seed[3],
                            double out[3]) {
    uint32_t s[3] = {seed[0], seed[1], seed[2]};
    double w = 0.0, sv = 0.0, idle = 0.0, sumw = 0.0, sums = 0.0;
    for (int64_t i = 0; i < clients; ++i) {
        const double a = -log(1.0 - uniform01(s)) / lambda;
        const double t = (w + sv) - a;
        if (t < 0.0) {
            idle = idle - t;
            w = 0.0;
        } else {
            w = t;
        }
        sv = -log(1.0 - uniform01(s)) / mu;
        sumw = sumw + w;
        sums = sums + (w + sv);
    }
    out[0] = idle / (double)clients;
    out[1] = sumw / (double)clients;
    out[2] = sums / (double)clients;
}

/* walk_replication_u, models.hpp:86-108: direction floor(4u), second draw discarded,
 * final x folded into [0, chunks). */
double oracle_walk_replication(int64_t steps, int64_t chunks, const uint32_t seed[3]) {
    uint32_t s[3] = {seed[0], seed[1], seed[2]};
    double px = 0.0, py = 0.0;
    for (int64_t i = 0; i < steps; ++i) {
        const double u = uniform01(s);
        (void)uniform01(s);
        const int64_t d = (int64_t)floor(4.0 * u);
        if (d == 0)
            px = px + 1.0;
        else if (d == 1)
            px = px - 1.0;
        else if (d == 2)
            py = py + 1.0;
        else
            py = py - 1.0;
    }
    const double c = (double)chunks;
    return fmod(fmod(px, c) + c, c);
}

/* validate_params, models.cpp:26-44 (warning handled by the caller). */
typedef struct {
    int64_t replications, draws, clients;
    double lambda, mu;
    int64_t steps, chunks;
} oracle_params;

int oracle_validate(int model, const oracle_params* p) {
    if (p->replications < 1) return EDOMAIN;
    switch (model) {
        case 0: return p->draws < 1 ? EDOMAIN : OK;
        case 1:
            if (p->clients < 1) return EDOMAIN;
            if (!(p->lambda > 0.0) || !(p->mu > 0.0)) return EDOMAIN;
            return OK;
        case 2:
            if (p->steps < 1 || p->chunks < 2) return EDOMAIN;
            return OK;
    }
    return EDOMAIN;
}

/* The Sequential branch of run_model, models.cpp:345-376, over given streams. */
int oracle_replications(int model, const oracle_params* p, const uint32_t* s1,
                        const uint32_t* s2, const uint32_t* s3, int64_t count, double* o0,
                        double* o1, double* o2) {
    int st = oracle_validate(model, p);
    if (st) return st;
    for (int64_t r = 0; r < count; ++r) {
        const uint32_t seed[3] = {s1[r], s2[r], s3[r]};
        if (model == 0) {
            o0[r] = oracle_pi_replication(p->draws, seed);
        } else if (model == 1) {
            double m[3];
            oracle_mm1_replication(p->clients, p->lambda, p->mu, seed, m);
            o0[r] = m[0];
            o1[r] = m[1];
            o2[r] = m[2];
        } else {
            o0[r] = oracle_walk_replication(p->steps, p->chunks, seed);
        }
    }
    return OK;
}

/* run_model(..., Sequential, ...) outputs, models.cpp:329-376. */
int oracle_run_model(int model, const oracle_params* p, uint64_t seed, double* o0, double* o1,
                     double* o2) {
    int st = oracle_validate(model, p);
    if (st) return st;
    const int64_t R = p->replications;
    uint32_t* s = (uint32_t*)malloc((size_t)R * 3 * sizeof(uint32_t));
    if (!s) return ENOMEM_;
    st = oracle_random_spacing(seed, R, s, s + R, s + 2 * R);
    if (!st) st = oracle_replications(model, p, s, s + R, s + 2 * R, R, o0, o1, o2);
    free(s);
    return st;
}

/* ---- statistics (proj/src/models.cpp:61-119) -------------------------------------- */

/* inverse_normal_cdf, models.cpp:61-97: Acklam's rational guess + two Halley steps. */
int oracle_inverse_normal_cdf(double p, double* out) {
    static const double A[6] = {-3.969683028665376e+01, 2.209460984245205e+02,
                                -2.759285104469687e+02, 1.383577518672690e+02,
                                -3.066479806614716e+01, 2.506628277459239e+00};
    static const double B[5] = {-5.447609879822406e+01, 1.615858368580409e+02,
                                -1.556989798598866e+02, 6.680131188771972e+01,
                                -1.328068155288572e+01};
    static const double C[6] = {-7.784894002430293e-03, -3.223964580411365e-01,
                                -2.400758277161838e+00, -2.549732539343734e+00,
                                4.374664141464968e+00,  2.938163982698783e+00};
    static const double D[4] = {7.784695709041462e-03, 3.224671290700398e-01,
                                2.445134137142996e+00, 3.754408661907416e+00};
    if (!(p > 0.0 && p < 1.0)) return EDOMAIN;
    const double plow = 0.02425;
    double x;
    if (p < plow) {
        const double q = sqrt(-2.0 * log(p));
        x = (((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    } else if (p <= 1.0 - plow) {
        const double q = p - 0.5, r = q * q;
        x = (((((A[0] * r + A[1]) * r + A[2]) * r + A[3]) * r + A[4]) * r + A[5]) * q /
            (((((B[0] * r + B[1]) * r + B[2]) * r + B[3]) * r + B[4]) * r + 1.0);
    } else {
        const double q = sqrt(-2.0 * log(1.0 - p));
        x = -(((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    }
    /* std::numbers::sqrt2 and std::numbers::pi as exact double literals */
    const double sqrt2 = 1.4142135623730951, pi = 3.141592653589793;
    for (int k = 0; k < 2; ++k) {
        const double e = 0.5 * erfc(-x / sqrt2) - p;
        const double u = e * sqrt(2.0 * pi) * exp(x * x / 2.0);
        x = x - u / (1.0 + x * u / 2.0);
    }
    *out = x;
    return OK;
}

/* confidence_interval, models.cpp:99-119: naive two-pass mean / sum of squares. */
int oracle_confidence_interval(const double* v, int64_t n, double level, double* mean,
                               double* half_width, int* warn_small) {
    if (n < 2) return EDOMAIN;
    if (!(level > 0.0 && level < 1.0)) return EDOMAIN;
    double sum = 0.0;
    for (int64_t i = 0; i < n; ++i) sum += v[i];
    const double m = sum / (double)n;
    double ss = 0.0;
    for (int64_t i = 0; i < n; ++i) ss += (v[i] - m) * (v[i] - m);
    const double s = sqrt(ss / (double)(n - 1));
    double z;
    int st = oracle_inverse_normal_cdf(0.5 + level / 2.0, &z);
    if (st) return st;
    *mean = m;
    *half_width = z * s / sqrt((double)n);
    *warn_small = n < 30;
    return OK;
}

/* -log(1-u)/rate, rng.cpp:57-61 (glibc log). */
int oracle_exponential_from_u(const double* u, int64_t n, double rate, double* out) {
    if (!(rate > 0.0)) return EDOMAIN;
    for (int64_t i = 0; i < n; ++i) {
        if (!(u[i] >= 0.0 && u[i] < 1.0)) return EDOMAIN;
        out[i] = -log(1.0 - u[i]) / rate;
    }
    return OK;
}
