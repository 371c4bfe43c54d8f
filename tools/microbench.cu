// Pipe-throughput microbenchmarks on the GPU box (the roofline denominators for an
// ALU-bound path; MEASURED_PEAKS.json only carries HBM and bf16 tensor peaks).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
//
// Each kernel runs 8 independent dependency chains per thread (enough ILP with 32
// warps/SM to saturate a pipe) of one instruction class; prints warp-instructions per
// cycle per SM (4.0 = one per SMSP per clock = the issue limit) using the measured SM clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_lop3(uint32_t* out, uint32_t seed) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[i]) : "r"(a[(i + 1) & 7]), "r"(a[(i + 2) & 7]));
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_shl_imad(uint32_t* out, uint32_t seed) {  // IMAD.SHL (fma pipe)
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("mad.lo.u32 %0, %0, 8192, %1;" : "+r"(a[i]) : "r"(a[(i + 3) & 7]));
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_mixed_taus(uint32_t* out, uint32_t seed) {  // the real taus88 step, 4 streams
    uint32_t s1[4], s2[4], s3[4], acc = 0;
    for (int i = 0; i < 4; ++i) {
        s1[i] = seed * (i + 3) + threadIdx.x;
        s2[i] = seed * (i + 7) ^ threadIdx.x;
        s3[i] = seed + i * 977 + threadIdx.x * 31;
    }
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            s1[i] = ((s1[i] & 0xFFFFFFFEu) << 12) ^ (((s1[i] << 13) ^ s1[i]) >> 19);
            s2[i] = ((s2[i] & 0xFFFFFFF8u) << 4) ^ (((s2[i] << 2) ^ s2[i]) >> 25);
            s3[i] = ((s3[i] & 0xFFFFFFF0u) << 17) ^ (((s3[i] << 3) ^ s3[i]) >> 11);
            acc += s1[i] ^ s2[i] ^ s3[i];
        }
    if (acc == 0x12345) out[0] = acc;
}

// taus88 with some components rebalanced onto the FMA pipe: the right shift as
// mul.hi by 2^(32-r) and the final merge as mad (operands from kernel params so ptxas
// cannot turn them back into SHF/LEA). variant bit c set = component c rebalanced.
struct Mul {
    uint32_t hi[3], sh[3];
};
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
__device__ __forceinline__ uint32_t mad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
    return r;
}
template <int V>
__global__ void k_taus_rebal(uint32_t* out, uint32_t seed, Mul mm) {
    uint32_t s1[4], s2[4], s3[4], acc = 0;
    for (int i = 0; i < 4; ++i) {
        s1[i] = seed * (i + 3) + threadIdx.x;
        s2[i] = seed * (i + 7) ^ threadIdx.x;
        s3[i] = seed + i * 977 + threadIdx.x * 31;
    }
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (V & 1)
                s1[i] = mad(s1[i] & 0xFFFFFFFEu, mm.sh[0], mulhi((s1[i] << 13) ^ s1[i], mm.hi[0]));
            else
                s1[i] = ((s1[i] & 0xFFFFFFFEu) << 12) ^ (((s1[i] << 13) ^ s1[i]) >> 19);
            if (V & 2)
                s2[i] = mad(s2[i] & 0xFFFFFFF8u, mm.sh[1], mulhi((s2[i] << 2) ^ s2[i], mm.hi[1]));
            else
                s2[i] = ((s2[i] & 0xFFFFFFF8u) << 4) ^ (((s2[i] << 2) ^ s2[i]) >> 25);
            if (V & 4)
                s3[i] = mad(s3[i] & 0xFFFFFFF0u, mm.sh[2], mulhi((s3[i] << 3) ^ s3[i], mm.hi[2]));
            else
                s3[i] = ((s3[i] & 0xFFFFFFF0u) << 17) ^ (((s3[i] << 3) ^ s3[i]) >> 11);
            acc += s1[i] ^ s2[i] ^ s3[i];
        }
    if (acc == 0x12345) out[0] = acc;
}

__global__ void k_dadd(double* out, double seed) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __dadd_rn(a[i], 1e-300);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_dfma(double* out, double seed) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __fma_rn(a[i], 0.999999, 1e-300);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}

// Eight independent conversion chains: each conversion's input is the high word of the
// previous result (a register half, no extra instruction), so no conversion is loop
// invariant. (The round-1 version converted the same v + i every iteration; the compiler
// hoisted it out of the loop and the row reported an impossible 124 warp-instr/clk/SM.)
template <bool SIGNED>
__global__ void k_i2f64(double* out, uint32_t seed) {
    uint32_t v[8];
    for (int i = 0; i < 8; ++i) v[i] = seed + threadIdx.x * 8 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double d;
            if (SIGNED)
                asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(d) : "r"(v[i]));
            else
                asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(d) : "r"(v[i]));
            v[i] = static_cast<uint32_t>(__double2hiint(d));
        }
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s += v[i];
    if (s == 12345u) out[0] = s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t seed) {
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(a[(i + 5) & 7] | 0x80000001u));
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x12345) out[0] = s;
}

// DFMA interleaved with R independent IMAD chains per DFMA (FMA pipe, full rate): if an
// FP64 warp-instruction held the SMSP's dispatch for two cycles, R = 1 would reach 2
// instructions per 3 cycles (2.67 warp-instr/clk/SM) instead of 1 per cycle (4.0).
template <int R>
__global__ void k_dfma_mix(double* out, double seed) {
    double a[4];
    uint32_t b[4 * R];
    for (int i = 0; i < 4; ++i) a[i] = seed + threadIdx.x + i;
    for (int i = 0; i < 4 * R; ++i) b[i] = threadIdx.x * 7 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            a[i] = __fma_rn(a[i], 0.999999, 1e-300);
#pragma unroll
            for (int k = 0; k < R; ++k) asm volatile("mad.lo.u32 %0, %0, 8193, %1;" : "+r"(b[i * R + k]) : "r"(b[(i * R + k + 1) % (4 * R)]));
        }
    double s = 0;
    for (int i = 0; i < 4; ++i) s += a[i];
    uint32_t t = 0;
    for (int i = 0; i < 4 * R; ++i) t ^= b[i];
    if (s == 1.2345 || t == 12345u) out[0] = s + t;
}

__global__ void k_shfl(uint32_t* out, uint32_t seed) {  // SHFL.UP (the pipelines' hand-over)
    uint32_t a[8];
    for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 8 + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __shfl_up_sync(0xffffffffu, a[i], 1);
    uint32_t s = 0;
    for (int i = 0; i < 8; ++i) s ^= a[i];
    if (s == 0x12345) out[0] = s;
}

__global__ void k_clock(long long* t) {
    long long c0 = clock64();
    long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    long long c = c0;
    while (c - c0 < 200000000LL) c = clock64();
    long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    t[0] = c - c0;
    t[1] = g1 - g0;
}

template <class F>
float time_it(F f) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    long long* dt;
    cudaMalloc(&dt, 16);
    // warm the clocks up, then measure the SM clock
    uint32_t* du;
    double* dd;
    cudaMalloc(&du, 64);
    cudaMalloc(&dd, 64);
    const int blocks = sms * 4, threads = 256;  // 32 warps / SM
    for (int i = 0; i < 20; ++i) k_lop3<<<blocks, threads>>>(du, i);
    k_clock<<<1, 1>>>(dt);
    long long h[2];
    cudaMemcpy(h, dt, 16, cudaMemcpyDeviceToHost);
    const double mhz = double(h[0]) / double(h[1]) * 1e3;
    std::printf("sms=%d sm_clock=%.0f MHz (clock64 vs globaltimer)\n", sms, mhz);
    const double warp_instr = double(blocks) * threads / 32 * ITERS * 8;
    auto report = [&](const char* name, float ms, double per_iter_instr) {
        const double wi = double(blocks) * threads / 32 * ITERS * per_iter_instr;
        const double cyc = ms * 1e-3 * mhz * 1e6;
        std::printf("%-28s %8.3f ms  %6.3f warp-instr/clk/SM\n", name, ms, wi / cyc / sms);
    };
    report("LOP3 (alu pipe)", time_it([&] { k_lop3<<<blocks, threads>>>(du, 1); }), 8);
    report("IMAD.SHL (fma pipe)", time_it([&] { k_shl_imad<<<blocks, threads>>>(du, 1); }), 8);
    report("IMAD.HI", time_it([&] { k_imadhi<<<blocks, threads>>>(du, 1); }), 8);
    report("DADD", time_it([&] { k_dadd<<<blocks, threads>>>(dd, 1.0); }), 8);
    report("DFMA", time_it([&] { k_dfma<<<blocks, threads>>>(dd, 1.0); }), 8);
    report("I2F.F64.U32 (chained)", time_it([&] { k_i2f64<false><<<blocks, threads>>>(dd, 1); }), 8);
    report("DFMA + 1 IMAD (mixed)", time_it([&] { k_dfma_mix<1><<<blocks, threads>>>(dd, 1.0); }), 8);
    report("DFMA + 2 IMAD (mixed)", time_it([&] { k_dfma_mix<2><<<blocks, threads>>>(dd, 1.0); }), 12);
    report("DFMA + 3 IMAD (mixed)", time_it([&] { k_dfma_mix<3><<<blocks, threads>>>(dd, 1.0); }), 16);
    report("SHFL.UP", time_it([&] { k_shfl<<<blocks, threads>>>(du, 1); }), 8);
    report("I2F.F64.S32 (chained)", time_it([&] { k_i2f64<true><<<blocks, threads>>>(dd, 1); }), 8);
    // taus88: 4 streams x (16 SASS per draw) + acc add per draw
    report("taus88 draw (16 SASS+1)", time_it([&] { k_mixed_taus<<<blocks, threads>>>(du, 7); }), 4 * 17);
    Mul mm{{1u << 13, 1u << 7, 1u << 21}, {1u << 12, 1u << 4, 1u << 17}};
    // same draws per launch as above: report as draws/clk relative (warp-instr count of the
    // reference form, 17 per draw, so the numbers compare directly)
    report("taus rebal comp1", time_it([&] { k_taus_rebal<1><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal comp2", time_it([&] { k_taus_rebal<2><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal comp3", time_it([&] { k_taus_rebal<4><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal comp2+3", time_it([&] { k_taus_rebal<6><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal comp1+2", time_it([&] { k_taus_rebal<3><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal all", time_it([&] { k_taus_rebal<7><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    report("taus rebal none", time_it([&] { k_taus_rebal<0><<<blocks, threads>>>(du, 7, mm); }), 4 * 17);
    (void)warp_instr;
    return 0;
}
