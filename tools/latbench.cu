// Dependent-chain latencies (cycles from issue to a dependent issue) of the ops on the
// WLP mm1 critical paths: one warp, one chain, clock64 around N dependent instructions.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lb tools/latbench.cu && /tmp/lb
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

#define CHAIN(name, decl, body, sink)                                              \
    __global__ void name(long long* t, double* out, double seed) {                 \
        decl;                                                                      \
        long long t0 = clock64();                                                  \
        _Pragma("unroll 64") for (int i = 0; i < N; ++i) { body; }                 \
        long long t1 = clock64();                                                  \
        if (threadIdx.x == 0) { t[0] = t1 - t0; out[0] = sink; }                   \
    }

CHAIN(k_dadd, double x = seed, asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x) : "d"(seed)), x)
CHAIN(k_dfma, double x = seed, asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(x) : "d"(seed)), x)
CHAIN(k_dmax, double x = seed, asm volatile("max.f64 %0, %0, %1;" : "+d"(x) : "d"(seed)), x)
CHAIN(k_fadd, float x = (float)seed, asm volatile("add.rn.f32 %0, %0, %1;" : "+f"(x) : "f"((float)seed)), x)
CHAIN(k_iadd, unsigned x = (unsigned)seed, asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"((unsigned)seed)), x)
CHAIN(k_lop, unsigned x = (unsigned)seed, asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"((unsigned)seed)), x)
CHAIN(k_shfl, unsigned x = (unsigned)seed, x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31), x)

__global__ void k_lds(long long* t, double* out, double seed) {
    __shared__ unsigned buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
    __syncthreads();
    unsigned x = (unsigned)seed & 1023;
    long long t0 = clock64();
#pragma unroll 64
    for (int i = 0; i < N; ++i) x = buf[x];
    long long t1 = clock64();
    if (threadIdx.x == 0) { t[0] = t1 - t0; out[0] = x; }
}

template <class K>
void run(const char* name, K k) {
    long long* t;
    double* o;
    cudaMalloc(&t, 8);
    cudaMalloc(&o, 8);
    k<<<1, 32>>>(t, o, 1.0000001);
    k<<<1, 32>>>(t, o, 1.0000001);
    long long h = 0;
    cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    std::printf("%-8s %6.2f cycles\n", name, double(h) / N);
    cudaFree(t);
    cudaFree(o);
}

int main() {
    run("DADD", k_dadd);
    run("DFMA", k_dfma);
    run("DMNMX", k_dmax);
    run("FADD", k_fadd);
    run("IADD", k_iadd);
    run("LOP3", k_lop);
    run("SHFL", k_shfl);
    run("LDS", k_lds);
    return 0;
}
