// Exhaustive check of the mm1 kernels' table-path exponential numerator
// (neg_log1m_table_dev, glibc_log.cuh) against the two-step form it replaced,
// -log_table_dev(one_minus_u32_nz(n)), itself pinned to host glibc by
// tests/test_parity_gpu.py::test_device_log_port_vs_host_libm_dense: every n in
// (2^28, 2^32), bit for bit. Exit status 1 on any mismatch.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -o tools/log_check tools/log_check.cu && tools/log_check
#include <cuda_runtime.h>

#include <cstdio>

#include "../paper_1501_01405_b200/csrc/glibc_log.cuh"

__global__ void k_check(unsigned long long* bad, unsigned long long* first) {
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    unsigned long long nbad = 0;
    for (uint64_t i = 0x10000001ull + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
         i < (1ull << 32); i += stride) {
        const uint32_t n = static_cast<uint32_t>(i);
        const double a = wlp::neg_log1m_table_dev(n, wlp::kLogTabDev);
        const double b = -wlp::log_table_dev(wlp::one_minus_u32_nz(n), wlp::kLogTabDev);
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
            ++nbad;
            atomicMin(first, static_cast<unsigned long long>(n));
        }
    }
    if (nbad) atomicAdd(bad, nbad);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    unsigned long long h[2] = {0, ~0ull};
    cudaMemcpy(d, h, 16, cudaMemcpyHostToDevice);
    k_check<<<148 * 8, 256>>>(d, d + 1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) return std::printf("cuda error\n"), 2;
    std::printf("table-path numerators n in (2^28, 2^32): mismatches %llu", h[0]);
    if (h[0]) std::printf(" (first n %llu)", h[1]);
    std::printf("\n");
    return h[0] ? 1 : 0;
}
