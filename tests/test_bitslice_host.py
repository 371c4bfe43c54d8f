"""Bitsliced taus88 / walk algebra (csrc/bitslice.cuh) on the host: the 32x32 transpose,
32 streams stepped bit-plane-wise against taus_next, and the carry-save walk counters
against the scalar walk (models.hpp:86-108), also read out through the one-transpose
difference the kernels use. Compiled with g++ from the same header the
kernel uses; no GPU."""
import subprocess

import pytest

from conftest import ROOT

SRC = r'''
#include <cstdio>
#include "paper_1501_01405_b200/csrc/bitslice.cuh"
using namespace wlp;
int main() {
    uint64_t x = 88172645463325252ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (uint32_t)(x >> 32); };
    for (int rep = 0; rep < 20; ++rep) {
        uint32_t a[32], b[32];
        for (int r = 0; r < 32; ++r) a[r] = b[r] = rnd();
        transpose32(b);
        for (int r = 0; r < 32; ++r)
            for (int c = 0; c < 32; ++c)
                if (((a[r] >> c) & 1) != ((b[c] >> r) & 1)) return 1;
        transpose32(b);
        for (int r = 0; r < 32; ++r) if (a[r] != b[r]) return 2;
    }
    for (int rep = 0; rep < 8; ++rep) {
        Taus s[32];
        for (int j = 0; j < 32; ++j) s[j] = make_state(rnd(), rnd(), rnd());
        BsTaus t;
        for (int j = 0; j < 32; ++j) { t.b1[j] = s[j].s1; t.b2[j] = s[j].s2; t.b3[j] = s[j].s3; }
        transpose32(t.b1); transpose32(t.b2); transpose32(t.b3);
        BsCount P, Q; bs_count_init(P); bs_count_init(Q);
        long dx[32] = {0};
        const int steps = 1000 + 977 * rep;
        for (int st = 0; st < steps; ++st) {
            uint32_t pl, mi;
            bs_walk_step(t, pl, mi);
            bs_count_add1(P, pl); bs_count_add1(Q, mi);
            for (int j = 0; j < 32; ++j) {
                const uint32_t d = taus_next_skip1(s[j]) >> 30;
                dx[j] += d == 0 ? 1 : (d == 1 ? -1 : 0);
            }
        }
        uint32_t pv[32], qv[32];
        bs_count_values(P, pv); bs_count_values(Q, qv);
        for (int j = 0; j < 32; ++j) if ((long)pv[j] - (long)qv[j] != dx[j]) return 3;
        int32_t dd[32];  // both counters through one transpose (the kernels' form)
        bs_count_diff(P, Q, dd);
        for (int j = 0; j < 32; ++j) if (dd[j] != dx[j]) return 6;
        transpose32(t.b1); transpose32(t.b2); transpose32(t.b3);
        for (int j = 0; j < 32; ++j)  // live bits (the top k of each component)
            if ((t.b1[j] ^ s[j].s1) & ~1u || (t.b2[j] ^ s[j].s2) & ~7u || (t.b3[j] ^ s[j].s3) & ~15u) return 4;
        // one more draw: output bits 4..31 (where every component's new bits are formed;
        // bs_step skips the bits that never reach a later state) equal taus_next's
        uint32_t o[32];
        BsTaus u = t;
        transpose32(u.b1); transpose32(u.b2); transpose32(u.b3);
        bs_step(u);
        for (int i = 0; i < 32; ++i) o[i] = u.b1[i] ^ u.b2[i] ^ u.b3[i];
        transpose32(o);
        for (int j = 0; j < 32; ++j) if ((o[j] ^ taus_next(s[j])) & ~15u) return 5;
    }
    std::puts("ok");
    return 0;
}
'''


def test_bitsliced_taus_and_walk_counts(tmp_path):
    src = tmp_path / "bs.cpp"
    src.write_text(SRC)
    exe = tmp_path / "bs"
    subprocess.run(["g++", "-std=c++17", "-O2", f"-I{ROOT}", "-o", str(exe), str(src)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", (r.returncode, r.stdout)
