// Host-side GF(2) jump-ahead algebra for taus88 (see taus88.cuh for the why).
//
// A component word x advances by x' = M_c x over GF(2)^32. n draws = M_c^n. We keep
// M_c^(2^k) for k < 64 (binary powers, uploaded once per device for the seeding
// kernel) and build, per launch, the lane-start tables the replication kernels use:
// lane l of a replication warp starts at draw 2*l*K, i.e. at J_l = M^(2 l K).
//
// Device application uses "nibble tables": T[c][p][v] = M_c^n (v << 4p) for the 8 nibble
// positions p and the 16 nibble values v, so M_c^n x = xor_p T[c][p][(x >> 4p) & 15]
// (8 table reads instead of 32 conditional column xors).
#pragma once

#include <stdint.h>

#include <array>
#include <vector>

#include "taus88.cuh"

namespace wlp {

inline uint32_t mat_apply(const Mat32& m, uint32_t x) {
    uint32_t y = 0;
    for (int j = 0; j < 32; ++j)
        if ((x >> j) & 1u) y ^= m.col[j];
    return y;
}

// (a*b) x = a(b(x))
inline Mat32 mat_mul(const Mat32& a, const Mat32& b) {
    Mat32 r;
    for (int j = 0; j < 32; ++j) r.col[j] = mat_apply(a, b.col[j]);
    return r;
}

inline Mat32 mat_identity() {
    Mat32 r;
    for (int j = 0; j < 32; ++j) r.col[j] = 1u << j;
    return r;
}

inline Mat32 step_matrix(int comp) {
    Mat32 r;
    for (int j = 0; j < 32; ++j) {
        const uint32_t e = 1u << j;
        r.col[j] = comp == 0 ? taus_c1(e) : comp == 1 ? taus_c2(e) : taus_c3(e);
    }
    return r;
}

struct Jump3 {
    Mat32 m[3];
};

// M^(2^k) for k = 0..63, per component (computed once).
inline const std::vector<Jump3>& binary_powers() {
    static const std::vector<Jump3> pw = [] {
        std::vector<Jump3> v(64);
        for (int c = 0; c < 3; ++c) v[0].m[c] = step_matrix(c);
        for (int k = 1; k < 64; ++k)
            for (int c = 0; c < 3; ++c) v[k].m[c] = mat_mul(v[k - 1].m[c], v[k - 1].m[c]);
        return v;
    }();
    return pw;
}

// M^n for each component.
inline Jump3 jump_matrix(uint64_t n) {
    Jump3 r;
    for (int c = 0; c < 3; ++c) r.m[c] = mat_identity();
    const auto& pw = binary_powers();
    for (int k = 0; k < 64; ++k)
        if ((n >> k) & 1u)
            for (int c = 0; c < 3; ++c) r.m[c] = mat_mul(pw[k].m[c], r.m[c]);
    return r;
}

inline Taus jump_state(const Taus& t, uint64_t n) {
    const Jump3 j = jump_matrix(n);
    return Taus{mat_apply(j.m[0], t.s1), mat_apply(j.m[1], t.s2), mat_apply(j.m[2], t.s3)};
}

// Nibble table entry for matrix m, nibble position p, value v.
inline uint32_t nibble_entry(const Mat32& m, int p, uint32_t v) {
    uint32_t y = 0;
    for (int b = 0; b < 4; ++b)
        if ((v >> b) & 1u) y ^= m.col[4 * p + b];
    return y;
}

constexpr int kLaneTabWords = 3 * 8 * 16 * 32;  // [comp][p][v][lane], 48 KB
constexpr int kUniTabWords = 3 * 8 * 16;         // [comp][p][v], 1.5 KB

inline void put_lane(std::vector<uint32_t>& out, int l, const Jump3& j) {
    for (int c = 0; c < 3; ++c)
        for (int p = 0; p < 8; ++p)
            for (uint32_t v = 0; v < 16; ++v) out[((c * 8 + p) * 16 + v) * 32 + l] = nibble_entry(j.m[c], p, v);
}

// Lane-start tables: lane l jumps by l * stride draws.
inline std::vector<uint32_t> lane_tables(uint64_t stride) {
    std::vector<uint32_t> out(kLaneTabWords);
    Jump3 step = jump_matrix(stride), cur;
    for (int c = 0; c < 3; ++c) cur.m[c] = mat_identity();
    for (int l = 0; l < 32; ++l) {
        put_lane(out, l, cur);
        for (int c = 0; c < 3; ++c) cur.m[c] = mat_mul(step.m[c], cur.m[c]);
    }
    return out;
}

// Lane tables for arbitrary per-lane distances: lane l jumps dist[l] draws (the wrapped
// warp pipelines start lane l of their first step at a replication's chunk l).
inline std::vector<uint32_t> lane_tables_dist(const std::array<uint64_t, 32>& dist) {
    std::vector<uint32_t> out(kLaneTabWords);
    for (int l = 0; l < 32; ++l) put_lane(out, l, jump_matrix(dist[l]));
    return out;
}

// Lane-uniform table for a single jump of n draws.
inline std::vector<uint32_t> uniform_table(uint64_t n) {
    std::vector<uint32_t> out(kUniTabWords);
    const Jump3 j = jump_matrix(n);
    for (int c = 0; c < 3; ++c)
        for (int p = 0; p < 8; ++p)
            for (uint32_t v = 0; v < 16; ++v) out[(c * 8 + p) * 16 + v] = nibble_entry(j.m[c], p, v);
    return out;
}

// Binary powers as nibble tables [k][comp][p][v] (96 KB) for the device jumps: applying
// M^(2^k) to a word is 8 independent lookups and an XOR tree, not 32 masked columns in a
// dependent chain (jump-ahead latency is what bounds the seeding of small runs).
inline std::vector<uint32_t> flat_nibble_powers() {
    std::vector<uint32_t> out(64 * kUniTabWords);
    const auto& pw = binary_powers();
    for (int k = 0; k < 64; ++k)
        for (int c = 0; c < 3; ++c)
            for (int p = 0; p < 8; ++p)
                for (uint32_t v = 0; v < 16; ++v)
                    out[k * kUniTabWords + (c * 8 + p) * 16 + v] = nibble_entry(pw[k].m[c], p, v);
    return out;
}

// Binary powers flattened as [k][comp][col] for the device seeding kernel.
inline std::vector<uint32_t> flat_binary_powers() {
    std::vector<uint32_t> out(64 * 3 * 32);
    const auto& pw = binary_powers();
    for (int k = 0; k < 64; ++k)
        for (int c = 0; c < 3; ++c)
            for (int j = 0; j < 32; ++j) out[(k * 3 + c) * 32 + j] = pw[k].m[c].col[j];
    return out;
}

}  // namespace wlp
