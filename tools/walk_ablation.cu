// Ablation of the walk's divergence (BASELINE config 3 / 4): the same thread-per-replication
// mapping with the reference's 4-way branch (what k_tlp<2> runs, models.hpp:96-104) and
// with the branch-free count (the cubic the WLP kernels use). Separates the two effects
// behind "WLP beats TLP on the walk": the mapping (divergence confined to one warp) and
// the arithmetic (no branch at all).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -o tools/walk_ablation tools/walk_ablation.cu && tools/walk_ablation [R] [steps]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1501_01405_b200/csrc/taus88.cuh"

using wlp::Taus;

__global__ void k_branchy(const uint32_t* s, int64_t R, int steps, int* dx_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= R) return;
    Taus st{s[r], s[R + r], s[2 * R + r]};
    double px = 0.0, py = 0.0;
    for (int i = 0; i < steps; ++i) {
        const uint32_t d = wlp::taus_next(st) >> 30;
        (void)wlp::taus_next(st);
        if (d == 0u)
            px = __dadd_rn(px, 1.0);
        else if (d == 1u)
            px = __dsub_rn(px, 1.0);
        else if (d == 2u)
            py = __dadd_rn(py, 1.0);
        else
            py = __dsub_rn(py, 1.0);
    }
    dx_out[r] = static_cast<int>(px);
}

__global__ void k_branch_free(const uint32_t* s, int64_t R, int steps, int* dx_out) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= R) return;
    Taus st{s[r], s[R + r], s[2 * R + r]};
    int acc = 0;
    for (int i = 0; i < steps; ++i) {
        const int d = static_cast<int>(wlp::taus_next_skip1(st) >> 30);
        acc += (((21 - 4 * d) * d) - 29) * d;  // 6*([d==0]-[d==1]) - 6
    }
    dx_out[r] = (acc + 6 * steps) / 6;
}

template <class K>
float time_kernel(K k, const uint32_t* s, int64_t R, int steps, int* out) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int block = 256;
    const int grid = static_cast<int>((R + block - 1) / block);
    k<<<grid, block>>>(s, R, steps, out);  // warm-up
    float best = 1e30f;
    for (int i = 0; i < 5; ++i) {
        cudaEventRecord(a);
        k<<<grid, block>>>(s, R, steps, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    return best;
}

int main(int argc, char** argv) {
    const int64_t R = argc > 1 ? std::atoll(argv[1]) : 10000000;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 1000;
    std::vector<uint32_t> h(3 * R);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (auto& v : h) {  // any valid taus88 states (components above their minimums)
        x ^= x << 13, x ^= x >> 7, x ^= x << 17;
        v = static_cast<uint32_t>(x >> 32) | 16u;
    }
    uint32_t* s;
    int *o1, *o2;
    cudaMalloc(&s, h.size() * 4);
    cudaMalloc(&o1, R * 4);
    cudaMalloc(&o2, R * 4);
    cudaMemcpy(s, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    const float t1 = time_kernel(k_branchy, s, R, steps, o1);
    const float t2 = time_kernel(k_branch_free, s, R, steps, o2);
    std::vector<int> a(R), b(R);
    cudaMemcpy(a.data(), o1, R * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), o2, R * 4, cudaMemcpyDeviceToHost);
    const bool same = a == b;
    std::printf("walk TLP R=%lld steps=%d: 4-way branch %.3f ms, branch-free %.3f ms, outputs %s\n",
                static_cast<long long>(R), steps, t1, t2, same ? "identical" : "DIFFER");
    return same ? 0 : 1;
}
