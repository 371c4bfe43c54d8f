// Bit-exact port of glibc 2.39's x86-64 FMA `log` (__log_fma) for host and device.
//
// Why: the mm1 model draws exponentials as -log(1-u)/rate (reference models.hpp:67,75;
// rng.cpp:60) through the host's libm. CUDA's log() rounds differently, so per-
// replication mm1 outputs would not be bit-identical to the CPU oracle. glibc's
// algorithm (sysdeps/ieee754/dbl-64/e_log.c, ARM optimized-routines, N = 128 table)
// is restated here in the exact operation order of the FMA build: the contractions
// below were read off the disassembly of libm.so.6's __log_fma;
// every plain + - * must stay unfused (host: -ffp-contract=off, device: --fmad=false),
// every fused step is an explicit fma().
//
// Pinned by tools/check_glibc_log.cpp: identical bits to libm's log for every input the
// model can produce, x = 1 - k*2^-32, k in [0, 2^32) (exhaustive), plus the generic
// paths (subnormals, specials) on samples.
//
// Device code passes the {invc, logc} table as a pointer (a shared-memory copy: the
// table index is data dependent, and a divergent __constant__ read serialises).
#pragma once

#include <stdint.h>

#include "glibc_log_data.h"

#if defined(__CUDACC__)
#define WLP_HD __host__ __device__ __forceinline__
#else
#define WLP_HD static inline
#include <math.h>
#include <string.h>
#endif

namespace wlp {

#if defined(__CUDACC__)
__device__ const double kLogTabDev[256] = WLP_LOG_TAB_INIT;  // global; kernels stage it in smem
#endif
static const double kLogTabHost[256] = WLP_LOG_TAB_INIT;

#if defined(__CUDA_ARCH__)
#define WLP_FMA(a, b, c) __fma_rn((a), (b), (c))
#define WLP_MUL(a, b) __dmul_rn((a), (b))
#define WLP_ADD(a, b) __dadd_rn((a), (b))
#define WLP_SUB(a, b) __dsub_rn((a), (b))
WLP_HD uint64_t wlp_as_u64(double x) { return static_cast<uint64_t>(__double_as_longlong(x)); }
WLP_HD double wlp_as_f64(uint64_t x) { return __longlong_as_double(static_cast<long long>(x)); }
WLP_HD int wlp_clz32(uint32_t x) { return __clz(static_cast<int>(x)); }
#else
#define WLP_FMA(a, b, c) fma((a), (b), (c))
#define WLP_MUL(a, b) ((a) * (b))
#define WLP_ADD(a, b) ((a) + (b))
#define WLP_SUB(a, b) ((a) - (b))
WLP_HD uint64_t wlp_as_u64(double x) {
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
}
WLP_HD double wlp_as_f64(uint64_t u) {
    double x;
    memcpy(&x, &u, sizeof x);
    return x;
}
WLP_HD int wlp_clz32(uint32_t x) { return x ? __builtin_clz(x) : 32; }
#endif

// Inputs 1 - 2^-4 <= x < 1 + 0x1.09p-4 take the table-free polynomial path.
constexpr uint64_t kLogNearLo = 0x3FEE000000000000ull;               // 1 - 0x1p-4
constexpr uint64_t kLogNearSpan = 0x3FF1090000000000ull - kLogNearLo;  // up to 1 + 0x1.09p-4
constexpr uint64_t kLogOff = 0x3fe6000000000000ull;  // table subintervals cover [OFF, 2*OFF)
constexpr uint64_t kOneBits = 0x3FF0000000000000ull;

WLP_HD bool log_is_near_one(uint64_t ix) { return ix - kLogNearLo < kLogNearSpan; }

// log(x) for x within 1 - 2^-4 .. 1 + 0x1.09p-4 (x != 1): r = x - 1 is exact, log1p(r)
// = r - r^2/2 + r^3 * P(r); the r^2/2 term is split hi/lo (rhi keeps 26 bits of r).
WLP_HD double log_near_one(double x) {
    const double r = WLP_SUB(x, 1.0);
    const double r2 = WLP_MUL(r, r);
    const double r3 = WLP_MUL(r, r2);
    constexpr double B[11] = WLP_LOG_POLY1_INIT;
    const double ta = WLP_FMA(r2, B[3], WLP_FMA(r, B[2], B[1]));
    const double tb = WLP_FMA(r2, B[6], WLP_FMA(r, B[5], B[4]));
    const double tc = WLP_FMA(r3, B[10], WLP_FMA(r2, B[9], WLP_FMA(r, B[8], B[7])));
    const double p = WLP_FMA(WLP_FMA(tc, r3, tb), r3, ta);
    const double rw = WLP_FMA(r, 0x1p27, r);
    const double rhi = WLP_FMA(-0x1p27, r, rw);
    const double rhi2 = WLP_MUL(rhi, rhi);
    const double rlo = WLP_SUB(r, rhi);
    const double hi = WLP_FMA(rhi2, B[0], r);
    double lo = WLP_FMA(rhi2, B[0], WLP_SUB(r, hi));
    lo = WLP_FMA(WLP_MUL(B[0], rlo), WLP_ADD(r, rhi), lo);
    return WLP_ADD(hi, WLP_FMA(p, r3, lo));
}

#if defined(__CUDACC__)
__constant__ double kLogPoly1Dev[11] = WLP_LOG_POLY1_INIT;

// log_near_one on the device with the coefficients as constant-bank operands of the
// DFMAs: from a constexpr array they are rebuilt in uniform registers on every call inside
// the mm1 batch loop (26 moves per batch). Same operations in the same order.
__device__ __forceinline__ double log_near_one_dev(double x) {
    const double* B = kLogPoly1Dev;
    const double r = __dsub_rn(x, 1.0);
    const double r2 = __dmul_rn(r, r);
    const double r3 = __dmul_rn(r, r2);
    const double ta = __fma_rn(r2, B[3], __fma_rn(r, B[2], B[1]));
    const double tb = __fma_rn(r2, B[6], __fma_rn(r, B[5], B[4]));
    const double tc = __fma_rn(r3, B[10], __fma_rn(r2, B[9], __fma_rn(r, B[8], B[7])));
    const double p = __fma_rn(__fma_rn(tc, r3, tb), r3, ta);
    const double rw = __fma_rn(r, 0x1p27, r);
    const double rhi = __fma_rn(-0x1p27, r, rw);
    const double rhi2 = __dmul_rn(rhi, rhi);
    const double rlo = __dsub_rn(r, rhi);
    const double hi = __fma_rn(rhi2, B[0], r);
    double lo = __fma_rn(rhi2, B[0], __dsub_rn(r, hi));
    lo = __fma_rn(__dmul_rn(B[0], rlo), __dadd_rn(r, rhi), lo);
    return __dadd_rn(hi, __fma_rn(p, r3, lo));
}
#endif

// log(x) for positive normal x outside the near-one window: x = 2^k * z, z in
// [OFF, 2*OFF); log x = k*ln2 + log(c) + log1p(z/c - 1), c from the 128-entry table
// `tab` = {invc, logc} pairs.
WLP_HD double log_table(uint64_t ix, const double* tab) {
    const uint64_t tmp = ix - kLogOff;
    const int i = static_cast<int>((tmp >> 45) & 127u);
    const int64_t k = static_cast<int64_t>(tmp) >> 52;
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double invc = tab[2 * i];
    const double logc = tab[2 * i + 1];
    const double z = wlp_as_f64(iz);
    const double kd = static_cast<double>(k);
    constexpr double A[5] = WLP_LOG_POLY_INIT;
    const double r = WLP_FMA(z, invc, -1.0);
    const double w = WLP_FMA(kd, WLP_LOG_LN2HI, logc);
    const double hi = WLP_ADD(r, w);
    const double lo = WLP_FMA(kd, WLP_LOG_LN2LO, WLP_ADD(WLP_SUB(w, hi), r));
    const double r2 = WLP_MUL(r, r);
    const double q = WLP_FMA(WLP_FMA(r, A[4], A[3]), r2, WLP_FMA(r, A[2], A[1]));
    const double y = WLP_FMA(WLP_MUL(r, r2), q, WLP_FMA(r2, A[0], lo));
    return WLP_ADD(y, hi);
}

// glibc log() semantics for every double (specials follow e_log.c: log(0) = -inf,
// log(<0) and log(nan) = nan, log(inf) = inf, subnormals normalised first).
WLP_HD double glibc_log_tab(double x, const double* tab) {
    uint64_t ix = wlp_as_u64(x);
    if (log_is_near_one(ix)) {
        if (ix == kOneBits) return 0.0;
        return log_near_one(x);
    }
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        if ((ix << 1) == 0) return -wlp_as_f64(0x7ff0000000000000ull);
        if (ix == 0x7ff0000000000000ull) return x;
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return wlp_as_f64(0x7ff8000000000000ull);
        ix = wlp_as_u64(WLP_MUL(x, 0x1p52)) - (52ull << 52);
    }
    return log_table(ix, tab);
}

#if !defined(__CUDA_ARCH__)
static inline double glibc_log(double x) { return glibc_log_tab(x, kLogTabHost); }
#endif

// Bits of x = 1 - n*2^-32 (the reference's `1.0 - next()`, exact) built with integer
// ops: m = 2^32 - n, x = m*2^-32 = 2^(-1-lz) * 1.f with lz = clz(m). n = 0 gives 1.0.
WLP_HD uint64_t one_minus_u32_bits(uint32_t n) {
    const uint32_t m = 0u - n;
    if (m == 0u) return kOneBits;
    const int lz = wlp_clz32(m);
    const uint32_t frac = (m << lz) << 1;  // mantissa bits below the leading one
    const uint32_t hi = (static_cast<uint32_t>(1022 - lz) << 20) | (frac >> 12);
    return (static_cast<uint64_t>(hi) << 32) | static_cast<uint64_t>(frac << 20);
}

#if defined(__CUDACC__)
// Device fast forms (same values, fewer instructions):
// x = 1 - n*2^-32 exactly as (2^20 + m*2^-32) - 2^20 with m = 2^32 - n: in [2^20, 2^21) the
// ulp is 2^-32, so the bit pattern (0x413 exponent, mantissa m) is built directly and one
// exact subtraction normalises it.
__device__ __forceinline__ double one_minus_u32_dev(uint32_t n) {
    const int hi = 0x41300000 + (n == 0u ? 1 : 0);
    return __dsub_rn(__hiloint2double(hi, static_cast<int>(0u - n)), 0x1p20);
}

// The same for n != 0 without the n == 0 bump (callers route n == 0 to the near path).
__device__ __forceinline__ double one_minus_u32_nz(uint32_t n) {
    return __dsub_rn(__hiloint2double(0x41300000, static_cast<int>(0u - n)), 0x1p20);
}

// For x = 1 - n*2^-32 the near-one window (x >= 1 - 2^-4) is exactly n <= 2^28, so callers
// test the draw itself. OFF has a zero low word, so the table-path decomposition only
// touches the high word of x.
__device__ __forceinline__ double log_table_dev(double x, const double* tab) {
    const uint32_t hx = static_cast<uint32_t>(__double2hiint(x));
    const uint32_t thi = hx - 0x3fe60000u;  // high word of ix - OFF
    const int i = static_cast<int>((thi >> 13) & 127u);
    const int k = static_cast<int>(thi) >> 20;
    const double z = __hiloint2double(static_cast<int>(hx - (thi & 0xfff00000u)), __double2loint(x));
    const double2 c = reinterpret_cast<const double2*>(tab)[i];  // {invc, logc}
    const double kd = static_cast<double>(k);
    constexpr double A[5] = WLP_LOG_POLY_INIT;
    const double r = __fma_rn(z, c.x, -1.0);
    const double w = __fma_rn(kd, WLP_LOG_LN2HI, c.y);
    const double hi = __dadd_rn(r, w);
    const double lo = __fma_rn(kd, WLP_LOG_LN2LO, __dadd_rn(__dsub_rn(w, hi), r));
    const double r2 = __dmul_rn(r, r);
    const double q = __fma_rn(__fma_rn(r, A[4], A[3]), r2, __fma_rn(r, A[2], A[1]));
    const double y = __fma_rn(__dmul_rn(r, r2), q, __fma_rn(r2, A[0], lo));
    return __dadd_rn(y, hi);
}

// -log(1 - n*2^-32) on the table path (n > 2^28; for n = 0 the value is garbage and the
// caller replaces it), the form the mm1 kernels use. Same arithmetic as
// -log_table_dev(one_minus_u32_nz(n)) with two instructions fewer:
// * x = m*2^-32 for m = 2^32 - n, and m converts to double exactly (I2F, off the FP64
//   pipe), so hi(x) = hi(m) - (32 << 20): thi is the same value against a shifted OFF, and
//   z's high word takes the shift in the same integer subtraction;
// * the result is negated in the final add (-(y + hi) == (-y) + (-hi) in round-to-nearest;
//   y + hi is never an exact zero here since x != 1).
// tools/log_check.cu compares it with the two-step form for every n.
// The polynomial and ln2 constants as constant-bank operands: a DFMA takes one c[][]
// operand directly, where immediates would be rebuilt in registers (two moves per
// double) wherever the compiler does not keep them live across a loop.
__constant__ double kLogTabConstDev[7] = {WLP_LOG_LN2HI, WLP_LOG_LN2LO, -0x1.0000000000001p-1, 0x1.555555551305bp-2,
                                          -0x1.fffffffeb4590p-3, 0x1.999b324f10111p-3, -0x1.55575e506c89fp-3};

constexpr double kLogPolyCheck[5] = WLP_LOG_POLY_INIT;
static_assert(kLogPolyCheck[0] == -0x1.0000000000001p-1 && kLogPolyCheck[1] == 0x1.555555551305bp-2 &&
                  kLogPolyCheck[2] == -0x1.fffffffeb4590p-3 && kLogPolyCheck[3] == 0x1.999b324f10111p-3 &&
                  kLogPolyCheck[4] == -0x1.55575e506c89fp-3,
              "kLogTabConstDev follows WLP_LOG_POLY_INIT");

#ifndef WLP_LOG_NOI2F
#define WLP_LOG_NOI2F 0
#endif
__device__ __forceinline__ double neg_log1m_table_dev(uint32_t n, const double* tab) {
#if WLP_LOG_NOI2F & 1
    const double dm = __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(0u - n)), 0x1p52);
#else
    const double dm = __uint2double_rn(0u - n);
#endif
    const uint32_t hm = static_cast<uint32_t>(__double2hiint(dm));
    const uint32_t thi = hm - (0x3fe60000u + (32u << 20));  // == hi(x) - hi(OFF)
    const int i = static_cast<int>((thi >> 13) & 127u);
    const int k = static_cast<int>(thi) >> 20;
    const double z = __hiloint2double(static_cast<int>(hm - (thi & 0xfff00000u) - (32u << 20)), __double2loint(dm));
    const double2 c = reinterpret_cast<const double2*>(tab)[i];  // {invc, logc}
#if WLP_LOG_NOI2F & 2
    const double kd = __dsub_rn(__hiloint2double(0x43380000 + (k >> 31), k), 0x1.8p52);
#else
    const double kd = static_cast<double>(k);
#endif
    const double* K = kLogTabConstDev;  // ln2hi, ln2lo, A[0..4] (WLP_LOG_POLY_INIT)
    const double r = __fma_rn(z, c.x, -1.0);
    const double w = __fma_rn(kd, K[0], c.y);
    const double hi = __dadd_rn(r, w);
    const double lo = __fma_rn(kd, K[1], __dadd_rn(__dsub_rn(w, hi), r));
    const double r2 = __dmul_rn(r, r);
    const double q = __fma_rn(__fma_rn(r, K[6], K[5]), r2, __fma_rn(r, K[4], K[3]));
    const double y = __fma_rn(__dmul_rn(r, r2), q, __fma_rn(r2, K[2], lo));
    return __dadd_rn(-y, -hi);
}
#endif

// -log(1 - n*2^-32) for a taus88 output n: the exponential numerator of mm1
// (models.hpp:67,75). Scalar form (host reference of the batched device routine).
WLP_HD double neg_log1m_u32_tab(uint32_t n, const double* tab) {
    const uint64_t ix = one_minus_u32_bits(n);
    if (log_is_near_one(ix)) return ix == kOneBits ? -0.0 : -log_near_one(wlp_as_f64(ix));
    return -log_table(ix, tab);
}

}  // namespace wlp
