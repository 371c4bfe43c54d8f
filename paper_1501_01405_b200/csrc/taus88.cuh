// taus88 on the device (and host): state, step, stream seeding, GF(2) jump-ahead.
//
// Reference semantics (all in /root/reference/proj):
//   RngState {s1,s2,s3}            include/warpsim/rng.hpp:11-17
//   make_rng_state (re-map by OR)  src/rng.cpp:29-34
//   rng_state_from_seed/splitmix64 src/rng.cpp:19-25, 36-40
//   taus_next                      src/rng.cpp:42-51
//   uniform01 = out * 2^-32        src/rng.cpp:53-55
//   random_spacing                 src/rng.cpp:67-87
//
// Each taus88 component is a linear map over GF(2)^32 of its 32-bit word (the masks and
// shifts are linear), so n steps of a component are one 32x32 bit-matrix M_c^n applied
// to the word. That turns the reference's strictly sequential stream consumption into
// something a warp can split: lane l of a replication warp starts at draw 2*l*K by one
// matrix application (a "jump"), and the seeding kernel starts thread t at master draw
// 3*t*C the same way.
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define TAUS_HD __host__ __device__ __forceinline__
#else
#define TAUS_HD static inline
#endif

namespace wlp {

// Component parameters (k, q, s) = (31,13,12), (29,2,4), (28,3,17); the word keeps the
// top k bits live, the low 32-k bits are dead (never reach an output).
constexpr uint32_t kMin1 = 2u, kMin2 = 8u, kMin3 = 16u;

struct Taus {
    uint32_t s1, s2, s3;
};

// High word of (hi:lo) << n (SHF.L.HI on the device).
TAUS_HD uint32_t funnel_hi(uint32_t lo, uint32_t hi, int n) {
#if defined(__CUDA_ARCH__)
    return __funnelshift_l(lo, hi, n);
#else
    return static_cast<uint32_t>(((static_cast<uint64_t>(hi) << 32 | lo) << n) >> 32);
#endif
}

// One step of a component (rng.cpp:44-50), ((s & M) << s_) ^ (((s << q) ^ s) >> (k - s_)).
// The two terms occupy disjoint bits, and (s & M) << s_ == (s >> (32-k)) << (32-k+s_), so
// the step is one funnel shift of (s >> (32-k) : (s << q) ^ s) by 32-k+s_: SHR, SHL, LOP3,
// SHF — one instruction fewer than mask, two shifts, xor and merge (pi 12.49 -> 11.37 ms
// at config 2, mm1 TLP 50.0 -> 47.5 ms at config 4). Moving the SHR to the FMA pipe as
// IMAD.HI (quarter rate) measured slower (12.27 / 51.4 ms).
TAUS_HD uint32_t taus_c1(uint32_t s) { return funnel_hi((s << 13) ^ s, s >> 1, 13); }
TAUS_HD uint32_t taus_c2(uint32_t s) { return funnel_hi((s << 2) ^ s, s >> 3, 7); }
TAUS_HD uint32_t taus_c3(uint32_t s) { return funnel_hi((s << 3) ^ s, s >> 4, 21); }

// Two steps of component 2 at once: its step s = 4 satisfies 2s <= k - q (8 <= 27), so
// advancing the underlying LFSR by 8 bits is one shift/xor round with s' = 8.
TAUS_HD uint32_t taus_c2x2(uint32_t s) { return funnel_hi((s << 2) ^ s, s >> 3, 11); }

// One draw: advance all three components, output their xor (rng.cpp:42-51).
TAUS_HD uint32_t taus_next(Taus& t) {
    t.s1 = taus_c1(t.s1);
    t.s2 = taus_c2(t.s2);
    t.s3 = taus_c3(t.s3);
    return t.s1 ^ t.s2 ^ t.s3;
}

// Two consecutive draws (o1 then o2). Component 2's two steps share v = (s<<2)^s and
// the masked word: s' = (m<<4) | v>>25, s'' = (m<<8) | v>>21 (the double-step form of
// taus_c2x2), which saves two ALU-pipe ops per pair of draws.
TAUS_HD void taus_next2(Taus& t, uint32_t& o1, uint32_t& o2) {
    const uint32_t a1 = taus_c1(t.s1), c1 = taus_c3(t.s3);
    const uint32_t h = t.s2 >> 3, v = (t.s2 << 2) ^ t.s2;
    const uint32_t b1 = funnel_hi(v, h, 7);
    o1 = a1 ^ b1 ^ c1;
    t.s1 = taus_c1(a1);
    t.s2 = funnel_hi(v, h, 11);
    t.s3 = taus_c3(c1);
    o2 = t.s1 ^ t.s2 ^ t.s3;
}

// Advance two draws, returning only the first output (the walk discards the second
// draw of every step, models.hpp:94).
TAUS_HD uint32_t taus_next_skip1(Taus& t) {
    uint32_t o1, o2;
    taus_next2(t, o1, o2);
    return o1;  // o2 is dead code for the compiler
}

// make_rng_state: components below their minimum get the minimum OR-ed in.
TAUS_HD Taus make_state(uint32_t a, uint32_t b, uint32_t c) {
    if (a < kMin1) a |= kMin1;
    if (b < kMin2) b |= kMin2;
    if (c < kMin3) c |= kMin3;
    return Taus{a, b, c};
}

// A stream key that could equal another candidate's key although their raw master
// triples differ: some component below twice its minimum.
TAUS_HD bool is_special_key(const Taus& t) {
    return t.s1 < 2u * kMin1 || t.s2 < 2u * kMin2 || t.s3 < 2u * kMin3;
}

// Exact u32 -> [0,1) double: n * 2^-32 (rng.cpp:53-55).
#if defined(__CUDA_ARCH__)
__device__ __forceinline__ double u01(uint32_t n) { return __dmul_rn(__uint2double_rn(n), 0x1p-32); }
#else
TAUS_HD double u01(uint32_t n) { return static_cast<double>(n) * 0x1p-32; }
#endif

// ---- host-side GF(2) algebra (jump matrices) --------------------------------------

// 32x32 bit matrix as 32 columns: col[j] = image of bit j.
struct Mat32 {
    uint32_t col[32];
};

}  // namespace wlp
