// Pins the glibc-log port (paper_1501_01405_b200/csrc/glibc_log.cuh) against this
// host's libm `log`.
//
//   g++ -std=c++17 -O2 -ffp-contract=off -mfma -pthread tools/check_glibc_log.cpp -o /tmp/chk -lm
//   /tmp/chk [--exhaustive]
//
// Default: 2^26 evenly spaced model inputs x = 1 - k*2^-32 plus special/subnormal
// samples (a few seconds). --exhaustive: all 2^32 model inputs (the complete domain of
// -log(1-u) for a taus88 draw u), split over hardware threads.
// Prints one line per class and exits non-zero on any bit mismatch.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "../paper_1501_01405_b200/csrc/glibc_log.cuh"

static std::uint64_t bits(double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}

int main(int argc, char** argv) {
    const bool exhaustive = argc > 1 && std::strcmp(argv[1], "--exhaustive") == 0;
    const std::uint64_t total = 1ull << 32;
    const std::uint64_t stride = exhaustive ? 1 : 64;
    unsigned nt = std::thread::hardware_concurrency();
    if (nt == 0) nt = 1;
    std::vector<std::uint64_t> bad(nt, 0), near(nt, 0), first_bad(nt, ~0ull);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < nt; ++t) {
        pool.emplace_back([&, t] {
            const std::uint64_t lo = total / nt * t, hi = (t + 1 == nt) ? total : total / nt * (t + 1);
            for (std::uint64_t k = lo - (lo % stride); k < hi; k += stride) {
                if (k < lo) continue;
                const double u = static_cast<double>(static_cast<std::uint32_t>(k)) * 0x1p-32;
                const double x = 1.0 - u;
                const double a = wlp::glibc_log(x), b = std::log(x);
                // the integer construction of 1-u and the split near-one/table paths the
                // device kernels use
                const double c = wlp::neg_log1m_u32_tab(static_cast<std::uint32_t>(k), wlp::kLogTabHost);
                if (x >= 1.0 - 0x1p-4) ++near[t];
                if (bits(a) != bits(b) || bits(c) != bits(-b) || wlp::one_minus_u32_bits(static_cast<std::uint32_t>(k)) != bits(x)) {
                    if (!bad[t]) first_bad[t] = k;
                    ++bad[t];
                }
            }
        });
    }
    for (auto& th : pool) th.join();
    std::uint64_t nbad = 0, nnear = 0;
    for (unsigned t = 0; t < nt; ++t) {
        nbad += bad[t];
        nnear += near[t];
        if (bad[t]) std::printf("  first mismatch k=%llu\n", (unsigned long long)first_bad[t]);
    }
    std::printf("model inputs 1-k*2^-32: checked %llu (stride %llu, %llu near-one), mismatches %llu\n",
                (unsigned long long)(total / stride), (unsigned long long)stride,
                (unsigned long long)nnear, (unsigned long long)nbad);

    // generic inputs: wide range, subnormals, specials
    std::uint64_t gbad = 0, gn = 0;
    std::uint64_t s = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < 4000000; ++i) {
        s ^= s << 13;
        s ^= s >> 7;
        s ^= s << 17;
        double x;
        std::uint64_t b = s & 0x7FFFFFFFFFFFFFFFull;
        std::memcpy(&x, &b, 8);
        if (!(x == x)) continue;
        const double a = wlp::glibc_log(x), c = std::log(x);
        ++gn;
        if (bits(a) != bits(c) && !(a != a && c != c)) ++gbad;
    }
    const double specials[] = {0.0, -0.0, 1.0, -1.0, INFINITY, 0x1p-1074, 0x1p-1022, 0x1.fffffffffffffp-1023, 2.0, 0.5, 0x1p-32};
    for (double x : specials) {
        const double a = wlp::glibc_log(x), c = std::log(x);
        ++gn;
        if (bits(a) != bits(c) && !(a != a && c != c)) {
            ++gbad;
            std::printf("  special mismatch x=%a port=%a libm=%a\n", x, a, c);
        }
    }
    std::printf("generic inputs: checked %llu, mismatches %llu\n", (unsigned long long)gn,
                (unsigned long long)gbad);
    return (nbad || gbad) ? 1 : 0;
}
