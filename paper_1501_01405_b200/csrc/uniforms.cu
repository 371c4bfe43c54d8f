// The reference's replication bodies over caller-given uniform sequences, on the device.
//
// The reference writes each model once as a template over a uniform source
// (pi_replication_u / mm1_replication_u / walk_replication_u, models.hpp:49-108) and its
// unit tests drive them with scripted sequences (test_models.cpp:36-43 the (0.6, 0.8)
// boundary point, :58-65 the mm1 hand trace, :123-137 the walk cut points). These kernels
// are those bodies with the source replaced by an array: replication r reads
// u[r*2n .. r*2n + 2n) in the reference's order, one thread per replication, every
// operation the reference's (unfused: --fmad=false; log = the glibc port, exact for every
// double; IEEE division). Any double is accepted, as in the templates.
//
// Also here: exponential_from_u (rng.cpp:58-61) over an array.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "glibc_log.cuh"
#include "kernels.cuh"

namespace wlp {
namespace {

__device__ double pi_u(const double* __restrict__ u, int64_t draws) {
    double c = 0.0;
    for (int64_t i = 0; i < draws; ++i) {
        const double x = u[2 * i], y = u[2 * i + 1];
        c = __dadd_rn(c, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)) <= 1.0 ? 1.0 : 0.0);
    }
    return __ddiv_rn(__dmul_rn(4.0, c), static_cast<double>(draws));
}

__device__ double expo_u(double u, double rate, const double* tab) {
    return __ddiv_rn(-glibc_log_tab(__dsub_rn(1.0, u), tab), rate);
}

__device__ void mm1_u(const double* __restrict__ u, int64_t clients, double lambda, double mu, const double* tab,
                      double& o_idle, double& o_wait, double& o_sys) {
    double w = 0.0, s = 0.0, idle = 0.0, sumw = 0.0, sums = 0.0;
    for (int64_t i = 0; i < clients; ++i) {
        const double a = expo_u(u[2 * i], lambda, tab);
        const double t = __dsub_rn(__dadd_rn(w, s), a);
        if (t < 0.0) {
            idle = __dsub_rn(idle, t);
            w = 0.0;
        } else {
            w = t;
        }
        s = expo_u(u[2 * i + 1], mu, tab);
        sumw = __dadd_rn(sumw, w);
        sums = __dadd_rn(sums, __dadd_rn(w, s));
    }
    const double n = static_cast<double>(clients);
    o_idle = __ddiv_rn(idle, n);
    o_wait = __ddiv_rn(sumw, n);
    o_sys = __ddiv_rn(sums, n);
}

__device__ double walk_u(const double* __restrict__ u, int64_t steps, int64_t chunks) {
    double px = 0.0, py = 0.0;
    for (int64_t i = 0; i < steps; ++i) {
        const int64_t d = static_cast<int64_t>(floor(__dmul_rn(4.0, u[2 * i])));
        if (d == 0)
            px = __dadd_rn(px, 1.0);
        else if (d == 1)
            px = __dsub_rn(px, 1.0);
        else if (d == 2)
            py = __dadd_rn(py, 1.0);
        else
            py = __dsub_rn(py, 1.0);
    }
    const double c = static_cast<double>(chunks);
    return fmod(__dadd_rn(fmod(px, c), c), c);
}

__global__ void k_uniform_reps(UniArgs a) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.count) return;
    const double* u = a.u + r * 2 * a.n;
    if (a.model == 0) {
        a.out0[r] = pi_u(u, a.n);
    } else if (a.model == 1) {
        mm1_u(u, a.n, a.lambda, a.mu, kLogTabDev, a.out0[r], a.out1[r], a.out2[r]);
    } else {
        a.out0[r] = walk_u(u, a.n, a.chunks);
    }
}

// exponential_from_u: rate > 0 is checked on the host; u outside [0, 1) sets *bad (the
// reference throws DomainError, rng.cpp:59-60) and the lowest such index wins.
__global__ void k_exponentials(const double* __restrict__ u, int64_t n, double rate, double* __restrict__ out,
                               unsigned long long* bad) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double x = u[i];
        if (!(x >= 0.0 && x < 1.0)) {
            atomicMin(bad, static_cast<unsigned long long>(i));
            continue;
        }
        out[i] = expo_u(x, rate, kLogTabDev);
    }
}

}  // namespace

cudaError_t launch_uniform_reps(const UniArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int block = 128;
    k_uniform_reps<<<static_cast<unsigned>((a.count + block - 1) / block), block, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_exponentials(const double* u, int64_t n, double rate, double* out, unsigned long long* bad,
                                cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int block = 256;
    const int64_t blocks = std::min<int64_t>((n + block - 1) / block, 148 * 16);
    k_exponentials<<<static_cast<unsigned>(blocks), block, 0, st>>>(u, n, rate, out, bad);
    return cudaGetLastError();
}

}  // namespace wlp
