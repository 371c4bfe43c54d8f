// Bitsliced taus88: one thread advances 32 streams at once.
//
// taus88 is linear over GF(2) (taus88.cuh), and the random walk (models.hpp:86-108) only
// looks at the top two bits of every other draw (d = out >> 30). So instead of one
// stream per 32-bit register, a thread keeps each state bit of 32 streams in one word:
// B_c[i] bit j = bit i of component c of stream j. One draw of all 32 streams is then
//   component 1: B[i] = B[i+6] ^ B[i+19] (i = 1..12),  B[i] = B[i-12] (i = 13..31)
//   component 2: B[i] = B[i+23] ^ B[i+25] (i = 3..6),  B[i] = B[i-4]  (i = 7..31)
//   component 3: B[i] = B[i+8] ^ B[i+11] (i = 4..20),  B[i] = B[i-17] (i = 21..31)
// (the shift/mask/xor of taus_next bit by bit; the low 32-k bits are dead and never read)
// = 33 XORs for 32 draws, and the moves are register renames in the unrolled loop. The
// top two output bits of a draw are bits 31/30 of the new state, i.e. plain bits of the
// old one: o31 = B1[19]^B2[27]^B3[14], o30 = B1[18]^B2[26]^B3[13].
#pragma once

#include <stdint.h>

#include "taus88.cuh"

namespace wlp {

// In-place 32x32 bit-matrix transpose: a[r] bit c -> a[c] bit r. Five stages of swapping
// the off-diagonal S x S blocks of every 2S x 2S diagonal block.
template <int S, uint32_t M>
TAUS_HD void transpose32_stage(uint32_t (&a)[32]) {
#pragma unroll
    for (int r = 0; r < 32; ++r) {
        if (r & S) continue;
        const uint32_t t = ((a[r] >> S) ^ a[r + S]) & M;
        a[r + S] ^= t;
        a[r] ^= t << S;
    }
}

#if defined(__CUDA_ARCH__)
// The 16- and 8-bit stages move whole bytes: two PRMTs per row pair instead of the
// shift/mask/xor swap (five instructions).
__device__ __forceinline__ void transpose32_bytes(uint32_t (&a)[32]) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {  // (a[r], a[r+16]): low halves to a[r], high halves to a[r+16]
        const uint32_t x = a[r], y = a[r + 16];
        a[r] = __byte_perm(x, y, 0x5410);
        a[r + 16] = __byte_perm(x, y, 0x7632);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) {  // (a[r], a[r+8]): even bytes to a[r], odd bytes to a[r+8]
        if (r & 8) continue;
        const uint32_t x = a[r], y = a[r + 8];
        a[r] = __byte_perm(x, y, 0x6240);
        a[r + 8] = __byte_perm(x, y, 0x7351);
    }
}
#endif

TAUS_HD void transpose32(uint32_t (&a)[32]) {
#if defined(__CUDA_ARCH__)
    transpose32_bytes(a);
#else
    transpose32_stage<16, 0x0000FFFFu>(a);
    transpose32_stage<8, 0x00FF00FFu>(a);
#endif
    transpose32_stage<4, 0x0F0F0F0Fu>(a);
    transpose32_stage<2, 0x33333333u>(a);
    transpose32_stage<1, 0x55555555u>(a);
}

struct BsTaus {
    uint32_t b1[32], b2[32], b3[32];
};

// One taus88 draw of all 32 streams. Only the live bits are formed (c1 1..31, c2 3..31,
// c3 4..31): the others never reach a later state, so output bits 0..3 are not available.
TAUS_HD void bs_step(BsTaus& t) {
    uint32_t n[32];
#pragma unroll
    for (int i = 1; i <= 12; ++i) n[i] = t.b1[i + 6] ^ t.b1[i + 19];
#pragma unroll
    for (int i = 13; i <= 31; ++i) n[i] = t.b1[i - 12];
#pragma unroll
    for (int i = 1; i <= 31; ++i) t.b1[i] = n[i];
#pragma unroll
    for (int i = 3; i <= 6; ++i) n[i] = t.b2[i + 23] ^ t.b2[i + 25];
#pragma unroll
    for (int i = 7; i <= 31; ++i) n[i] = t.b2[i - 4];
#pragma unroll
    for (int i = 3; i <= 31; ++i) t.b2[i] = n[i];
#pragma unroll
    for (int i = 4; i <= 20; ++i) n[i] = t.b3[i + 8] ^ t.b3[i + 11];
#pragma unroll
    for (int i = 21; i <= 31; ++i) n[i] = t.b3[i - 17];
#pragma unroll
    for (int i = 4; i <= 31; ++i) t.b3[i] = n[i];
}

// One walk step of all 32 streams (models.hpp:93-104: d = first draw >> 30, the second
// draw discarded): masks of the streams moving +x (d == 0) and -x (d == 1).
TAUS_HD void bs_walk_step(BsTaus& t, uint32_t& plus, uint32_t& minus) {
    const uint32_t o31 = t.b1[19] ^ t.b2[27] ^ t.b3[14];
    const uint32_t o30 = t.b1[18] ^ t.b2[26] ^ t.b3[13];
    plus = ~(o31 | o30);
    minus = ~o31 & o30;
    bs_step(t);
    bs_step(t);
}

// The live bit planes of a group (b1[1..31], b2[3..31], b3[4..31]): the layout the
// bitsliced walk pipeline feeds from.
constexpr int kBsLive = 88;

// Transposes 32 streams' words (t.bc[j] = component c of stream j) into bit planes and
// stores the 88 live planes at out (16-byte aligned on the device).
TAUS_HD void bs_store_planes(BsTaus& t, uint32_t* out) {
    transpose32(t.b1);
    transpose32(t.b2);
    transpose32(t.b3);
    uint32_t w[kBsLive];
#pragma unroll
    for (int i = 1; i < 32; ++i) w[i - 1] = t.b1[i];
#pragma unroll
    for (int i = 3; i < 32; ++i) w[31 + i - 3] = t.b2[i];
#pragma unroll
    for (int i = 4; i < 32; ++i) w[60 + i - 4] = t.b3[i];
#if defined(__CUDA_ARCH__)
    uint4* o = reinterpret_cast<uint4*>(out);
#pragma unroll
    for (int k = 0; k < kBsLive / 4; ++k) o[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
#else
    for (int k = 0; k < kBsLive; ++k) out[k] = w[k];
#endif
}

// Carry-save adder over bitsliced words: (hi, lo) = a + b + c, per bit position.
TAUS_HD void bs_csa(uint32_t& hi, uint32_t& lo, uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t u = a ^ b;
    hi = (a & b) | (u & c);
    lo = u ^ c;
}

// 32 per-stream counters in bitsliced binary: bit w of stream j's count is bit j of
// c[w]. Masks are added 16 at a time through a Harley-Seal carry-save tree whose
// partial sums are the low four digits (weights 1, 2, 4, 8) and whose weight-16 carry
// ripples into digits 4..15; so c[] is always an exact binary count below 2^16.
struct BsCount {
    uint32_t c[16];
};

TAUS_HD void bs_count_init(BsCount& k) {
#pragma unroll
    for (int w = 0; w < 16; ++w) k.c[w] = 0u;
}

// Adds one mask (a single count per set bit): ripple from digit 0.
TAUS_HD void bs_count_add1(BsCount& k, uint32_t m) {
#pragma unroll
    for (int w = 0; w < 16; ++w) {
        const uint32_t carry = k.c[w] & m;
        k.c[w] ^= m;
        m = carry;
    }
}

// Per-stream values: v[j] = count of stream j (transposes the digits).
TAUS_HD void bs_count_values(const BsCount& k, uint32_t (&v)[32]) {
#pragma unroll
    for (int w = 0; w < 32; ++w) v[w] = w < 16 ? k.c[w] : 0u;
    transpose32(v);
}

// Per-stream P - Q of two 16-digit counters with one transpose: row w < 16 holds P's
// digit w, row 16 + w Q's digit w, so column j is stream j's P count in bits 0..15 and
// its Q count in bits 16..31.
TAUS_HD void bs_count_diff(const BsCount& P, const BsCount& Q, int32_t (&dx)[32]) {
    uint32_t v[32];
#pragma unroll
    for (int w = 0; w < 16; ++w) {
        v[w] = P.c[w];
        v[16 + w] = Q.c[w];
    }
    transpose32(v);
#pragma unroll
    for (int j = 0; j < 32; ++j) dx[j] = static_cast<int32_t>(v[j] & 0xFFFFu) - static_cast<int32_t>(v[j] >> 16);
}

}  // namespace wlp
