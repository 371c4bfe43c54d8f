// Exhaustive check of the mm1 rate division by reciprocal + one correction (Markstein):
//   y = RN(1/b);  q = RN(e*y);  r = RN(b*q - e) (exact);  q' = RN(q - r*y) == RN(e/b)
// against IEEE division (__ddiv_rn) for EVERY numerator the mm1 model can produce
// (e = -log(1 - n*2^-32), n in [0, 2^32): models.hpp:67,75 through the glibc-log port) and
// a set of rates b (edge significands, powers of two, random); plus random (a, b) pairs
// over whole binades. Prints mismatch counts; exit status 1 on any mismatch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -o tools/div_check tools/div_check.cu && tools/div_check [random_rates] [pairs_e9]
// (-DDIV_CHECK_NO_CORRECTION: the negative control, expected to report mismatches)
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_1501_01405_b200/csrc/glibc_log.cuh"

#ifndef DIV_CHECK_NO_CORRECTION
__device__ __forceinline__ double div_rcp(double e, double b, double y) {
    const double q = __dmul_rn(e, y);
    const double r = __fma_rn(b, q, -e);
    return __fma_rn(-r, y, q);
}
#else  // negative control: the product alone is not correctly rounded; the check must see it
__device__ __forceinline__ double div_rcp(double e, double, double y) { return __dmul_rn(e, y); }
#endif

__device__ __forceinline__ bool same(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}

__global__ void k_numerators(const double* rates, const double* rcps, int nrates, unsigned long long* bad,
                             unsigned long long* first) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long nbad = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < (1ull << 32); i += stride) {
        const uint32_t n = static_cast<uint32_t>(i);
        const double e = n <= 0x10000000u ? (n == 0u ? -0.0 : -wlp::log_near_one(wlp::one_minus_u32_dev(n)))
                                          : -wlp::log_table_dev(wlp::one_minus_u32_nz(n), wlp::kLogTabDev);
        for (int k = 0; k < nrates; ++k) {
            const double b = rates[k];
            if (!same(div_rcp(e, b, rcps[k]), __ddiv_rn(e, b))) {
                ++nbad;
                atomicMin(first, static_cast<unsigned long long>(k) << 32 | n);
            }
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// a, b with random significands in [1, 2) (the check is scale-invariant away from
// over/underflow); y = RN(1/b) by IEEE division.
__global__ void k_pairs(uint64_t count, uint64_t seed, unsigned long long* bad) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long nbad = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
        const uint64_t h = mix(seed ^ i), g = mix(h);
        const double a = __longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | (h >> 12)));
        const double b = __longlong_as_double(static_cast<long long>(0x3FF0000000000000ull | (g >> 12)));
        const double y = __ddiv_rn(1.0, b);
        if (!same(div_rcp(a, b, y), __ddiv_rn(a, b))) ++nbad;
    }
    if (nbad) atomicAdd(bad, nbad);
}

int main(int argc, char** argv) {
    const int nrand = argc > 1 ? std::atoi(argv[1]) : 64;
    const double pairs = (argc > 2 ? std::atof(argv[2]) : 100.0) * 1e9;
    std::vector<double> rates = {0.5, 1.0, 0.3, 0.9, 0.1, 0.7, 1.1, 3.0, 7.0, 1e-3, 1e3, 1e-250, 1e250,
                                 0x1.fffffffffffffp0, 0x1.0000000000001p0, 0x1.fffffffffffffp-1,
                                 0x1.0000000000001p-1, 0x1.5555555555555p0, 0x1.999999999999ap-4};
    for (int k = 0; k < 64; ++k) rates.push_back(0.1 + 0.8 * k / 63.0);  // BASELINE config-5 lambdas
    std::mt19937_64 rng(20260201);
    for (int k = 0; k < nrand; ++k)
        rates.push_back(std::ldexp(1.0 + static_cast<double>(rng() >> 11) * 0x1p-53, static_cast<int>(rng() % 41) - 20));
    std::vector<double> rcps(rates.size());
    for (size_t k = 0; k < rates.size(); ++k) rcps[k] = 1.0 / rates[k];
    double *dr, *dy;
    unsigned long long *bad, *first;
    cudaMalloc(&dr, rates.size() * 8);
    cudaMalloc(&dy, rates.size() * 8);
    cudaMalloc(&bad, 16);
    first = bad + 1;
    cudaMemcpy(dr, rates.data(), rates.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, rcps.data(), rates.size() * 8, cudaMemcpyHostToDevice);
    unsigned long long h[2] = {0, ~0ull};
    cudaMemcpy(bad, h, 16, cudaMemcpyHostToDevice);
    k_numerators<<<148 * 8, 256>>>(dr, dy, static_cast<int>(rates.size()), bad, first);
    cudaMemcpy(h, bad, 16, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) return std::printf("cuda error\n"), 2;
    std::printf("numerators: 2^32 x %zu rates, mismatches %llu", rates.size(), h[0]);
    if (h[0]) std::printf(" (first rate %.17g n %llu)", rates[h[1] >> 32], h[1] & 0xffffffffull);
    std::printf("\n");
    unsigned long long pb = 0;
    cudaMemcpy(bad, &pb, 8, cudaMemcpyHostToDevice);
    k_pairs<<<148 * 8, 256>>>(static_cast<uint64_t>(pairs), 42, bad);
    cudaMemcpy(&pb, bad, 8, cudaMemcpyDeviceToHost);
    std::printf("random pairs: %.3g, mismatches %llu\n", pairs, pb);
    return h[0] || pb ? 1 : 0;
}
