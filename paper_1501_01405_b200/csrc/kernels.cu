// sm_100a kernels of the WLP replication engine. No tensor cores: every kernel here is
// integer / FP64 ALU work bounded by instruction issue.
//
//   k_seed       random_spacing (rng.cpp:67-87) by jump-ahead: thread t fills 32 stream
//                slots from master draw 3*c(t) on, flags "special" candidates.
//   k_taus       raw taus88 stream (taus88.golden format) by jump-ahead.
//   k_wlp_lanes  pi / walk, one replication per warp; lane l consumes the replication's
//                units [l*K, (l+1)*K) after one nibble-table jump; exact integer
//                warp reduction (__reduce_add_sync) of hits / x-displacement.
//   k_wlp_mm1    mm1, one replication per warp; lanes produce the exponentials of a
//                32*T-client panel into shared memory, lane 0 runs the order-preserving
//                Lindley recursion (models.hpp:61-84) on them.
//   k_tlp        the thread-per-replication comparison mapping (plan_launch TLP
//                geometry, wlp.cpp:88-92).
//   k_stats      sums / centred sums of squares for the confidence interval.
//
// Compiled with --fmad=false: the reference is built with -ffp-contract=off
// (CMakeLists.txt:12-13), so no a*b+c may fuse; the only FMAs are the explicit ones in
// the glibc log port.
#include <cuda_runtime.h>
#include <stdint.h>

#include "glibc_log.cuh"
#include "jump.hpp"
#include "kernels.cuh"

namespace wlp {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// x -> M x for a matrix given by 32 columns in global memory.
__device__ __forceinline__ uint32_t mat_apply_g(const uint32_t* __restrict__ col, uint32_t x) {
    uint32_t y = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) y ^= (0u - ((x >> j) & 1u)) & __ldg(col + j);
    return y;
}

// Jump n draws with the binary powers M^(2^k) ([k][comp][32]).
__device__ Taus jump_pow(const uint32_t* __restrict__ pw, Taus t, uint64_t n) {
    while (n) {
        const int k = __ffsll(static_cast<long long>(n)) - 1;
        n &= n - 1;
        const uint32_t* m = pw + k * 96;
        t.s1 = mat_apply_g(m, t.s1);
        t.s2 = mat_apply_g(m + 32, t.s2);
        t.s3 = mat_apply_g(m + 64, t.s3);
    }
    return t;
}

// Nibble-table application; `t` points at [p][v] rows with row stride `S` words.
template <int S>
__device__ __forceinline__ uint32_t nib_apply(const uint32_t* t, uint32_t x) {
    uint32_t y = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p) y ^= t[(p * 16 + ((x >> (4 * p)) & 15u)) * S];
    return y;
}

// Lane-specific jump: tables laid out [comp][p][v][lane] (conflict-free: lane = bank).
__device__ __forceinline__ Taus lane_jump(const uint32_t* tab, int lane, Taus t) {
    t.s1 = nib_apply<32>(tab + lane, t.s1);
    t.s2 = nib_apply<32>(tab + 4096 + lane, t.s2);
    t.s3 = nib_apply<32>(tab + 8192 + lane, t.s3);
    return t;
}

// Lane-uniform jump: tables [comp][p][v] (16-word rows: distinct v = distinct banks,
// equal v = broadcast).
__device__ __forceinline__ Taus uni_jump(const uint32_t* tab, Taus t) {
    t.s1 = nib_apply<1>(tab, t.s1);
    t.s2 = nib_apply<1>(tab + 128, t.s2);
    t.s3 = nib_apply<1>(tab + 256, t.s3);
    return t;
}

__device__ __forceinline__ Taus load_seed(const RepArgs& a, int64_t r) {
    return Taus{__ldg(a.seeds + r), __ldg(a.seeds + a.count + r), __ldg(a.seeds + 2 * a.count + r)};
}

// Inside test of one pi point, x*x + y*y <= 1.0 in unfused fp64 (models.hpp:54-56),
// evaluated on the unscaled draws: with x = a*2^-32 every product and sum is the
// reference's value times 2^64 exactly (power-of-two scaling commutes with rounding
// in the normal range), so the test is fl(fl(a*a) + fl(b*b)) <= 2^64.
__device__ __forceinline__ bool pi_inside(uint32_t a, uint32_t b) {
    const double x = __uint2double_rn(a), y = __uint2double_rn(b);
    return __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)) <= 0x1p64;
}

// Hits among `units` consecutive points of a stream (main loop unrolled by 4).
__device__ __forceinline__ uint32_t pi_hits(Taus& st, uint32_t units) {
    uint32_t hits = 0, u = 0;
    for (; u + 4 <= units; u += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t x = taus_next(st);
            const uint32_t y = taus_next(st);
            if (pi_inside(x, y)) ++hits;
        }
    }
    for (; u < units; ++u) {
        const uint32_t x = taus_next(st);
        const uint32_t y = taus_next(st);
        if (pi_inside(x, y)) ++hits;
    }
    return hits;
}

// x displacement of `units` consecutive walk steps (direction = floor(4u) = out >> 30,
// second draw of each step discarded, models.hpp:93-104).
__device__ __forceinline__ int walk_dx(Taus& st, uint32_t units) {
    int dx = 0;
    uint32_t u = 0;
    for (; u + 4 <= units; u += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t d = taus_next_skip1(st) >> 30;
            dx += static_cast<int>(d == 0u) - static_cast<int>(d == 1u);
        }
    }
    for (; u < units; ++u) {
        const uint32_t d = taus_next_skip1(st) >> 30;
        dx += static_cast<int>(d == 0u) - static_cast<int>(d == 1u);
    }
    return dx;
}

// -log(1-u)/rate (models.hpp:67,75); exact reciprocal product when rate = 2^k.
template <bool INV>
__device__ __forceinline__ double expo(uint32_t n, double rate, double inv) {
    const double e = neg_log1m_u32(n);
    return INV ? __dmul_rn(e, inv) : __ddiv_rn(e, rate);
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// fold of the walk's final x (models.hpp:106-107): fmod(fmod(px,c)+c,c) on an integral
// px is exact and equals ((px % c) + c) % c (C remainder, sign of the dividend).
__device__ __forceinline__ double walk_fold(int64_t px, int64_t c) {
    return static_cast<double>(((px % c) + c) % c);
}

// ---------------------------------------------------------------------------------
// Seeding
// ---------------------------------------------------------------------------------

__global__ void __launch_bounds__(kSeedBlock) k_seed(SeedArgs a) {
    extern __shared__ uint32_t sh[];  // 3 x [kSeedBlock][33] (padded: conflict-free)
    constexpr int kRow = kSeedPerThread + 1;
    constexpr int kPlane = kSeedBlock * kRow;
    const int tid = threadIdx.x;
    const int64_t blk0 = static_cast<int64_t>(blockIdx.x) * kSeedBlock * kSeedPerThread;
    const int64_t my0 = blk0 + static_cast<int64_t>(tid) * kSeedPerThread;
    int64_t left = a.count - my0;
    const int nmine = left <= 0 ? 0 : (left < kSeedPerThread ? static_cast<int>(left) : kSeedPerThread);
    if (nmine > 0) {
        int64_t c = a.slot_begin + my0;  // candidate index of my first slot
        int64_t ri = 0;
        while (ri < a.n_rejected && a.rejected[ri] <= c) {
            ++c;
            ++ri;
        }
        Taus m = jump_pow(a.powers, a.master, 3ull * static_cast<uint64_t>(c));
        for (int j = 0; j < nmine; ++j) {
            Taus key;
            for (;;) {
                const uint32_t x = taus_next(m), y = taus_next(m), z = taus_next(m);
                key = make_state(x, y, z);
                if (ri < a.n_rejected && a.rejected[ri] == c) {  // a redrawn candidate
                    ++ri;
                    ++c;
                    continue;
                }
                break;
            }
            if (is_special_key(key)) {
                const unsigned long long pos = atomicAdd(a.n_special, 1ull);
                if (static_cast<int64_t>(pos) < a.special_cap) {
                    SpecialRec* sp = static_cast<SpecialRec*>(a.specials) + pos;
                    sp->index = c;
                    sp->s1 = key.s1;
                    sp->s2 = key.s2;
                    sp->s3 = key.s3;
                    sp->pad = 0;
                }
            }
            ++c;
            sh[tid * kRow + j] = key.s1;
            sh[kPlane + tid * kRow + j] = key.s2;
            sh[2 * kPlane + tid * kRow + j] = key.s3;
        }
    }
    __syncthreads();
    int64_t nblk = a.count - blk0;
    if (nblk > kSeedBlock * kSeedPerThread) nblk = kSeedBlock * kSeedPerThread;
    for (int i = tid; i < nblk; i += kSeedBlock) {
        const int si = (i / kSeedPerThread) * kRow + (i % kSeedPerThread);
        a.out[blk0 + i] = sh[si];
        a.out[a.count + blk0 + i] = sh[kPlane + si];
        a.out[2 * a.count + blk0 + i] = sh[2 * kPlane + si];
    }
}

// -log(1 - k*2^-32) for a batch of k (pins the device glibc-log port directly).
__global__ void k_neg_log1m(const uint32_t* __restrict__ k, int64_t n, double* __restrict__ out) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = neg_log1m_u32(k[i]);
}

constexpr int kTausPerThread = 64;

__global__ void k_taus(const uint32_t* __restrict__ pw, Taus seed, int64_t n, uint32_t* out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t i0 = t * kTausPerThread;
    if (i0 >= n) return;
    Taus s = jump_pow(pw, seed, static_cast<uint64_t>(i0));
    const int64_t i1 = i0 + kTausPerThread < n ? i0 + kTausPerThread : n;
    for (int64_t i = i0; i < i1; ++i) out[i] = taus_next(s);
}

// ---------------------------------------------------------------------------------
// WLP: one replication per warp
// ---------------------------------------------------------------------------------

// Warp w of the persistent grid owns replications [w*R/W, (w+1)*R/W) (every replication
// costs the same, so a static split is balanced). Results are parked in lane
// (r - lo) % 32 and stored 32 at a time (coalesced 256 B).
template <int MODEL>
__global__ void __launch_bounds__(kWlpBlock) k_wlp_lanes(RepArgs a, const uint32_t* __restrict__ gtab,
                                                          int64_t K) {
    extern __shared__ uint32_t tab[];  // kLaneTabWords
    {
        const uint4* src = reinterpret_cast<const uint4*>(gtab);
        uint4* dst = reinterpret_cast<uint4*>(tab);
        for (int i = threadIdx.x; i < kLaneTabWords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t lo = warp * a.count / nwarps, hi = (warp + 1) * a.count / nwarps;
    int64_t mine = a.n - static_cast<int64_t>(lane) * K;
    mine = mine < 0 ? 0 : (mine > K ? K : mine);
    const uint32_t units = static_cast<uint32_t>(mine);
    const bool wide = a.n >= (int64_t(1) << 31);
    double keep = 0.0;
    for (int64_t r = lo; r < hi; ++r) {
        Taus st = lane_jump(tab, lane, load_seed(a, r));
        double val;
        if (MODEL == 0) {  // pi: count points inside the quarter circle
            const uint32_t hits = pi_hits(st, units);
            const int64_t total = wide ? warp_sum_i64(hits) : static_cast<int64_t>(__reduce_add_sync(kFull, hits));
            // c counts exactly in a double, so (4.0*c)/draws is the reference's value.
            val = __ddiv_rn(__dmul_rn(4.0, static_cast<double>(total)), static_cast<double>(a.n));
        } else {  // walk: only the x displacement reaches the output
            const int dx = walk_dx(st, units);
            const int64_t total = wide ? warp_sum_i64(dx) : static_cast<int64_t>(__reduce_add_sync(kFull, dx));
            val = walk_fold(total, a.chunks);
        }
        const int slot = static_cast<int>((r - lo) & 31);
        if (lane == slot) keep = val;
        if (slot == 31 || r == hi - 1) {
            if (lane <= slot) a.out0[r - slot + lane] = keep;
        }
    }
}

// mm1: lanes generate, lane 0 recurses. Panel p covers clients [p*32T, (p+1)*32T); lane l
// produces clients p*32T + l*T + j (j < T) from draws 2*(that index) and 2*(...)+1, so
// each lane steps its own contiguous draw range and hops 62T draws between panels.
template <bool INV>
__global__ void __launch_bounds__(kMm1Block) k_wlp_mm1(RepArgs a, const uint32_t* __restrict__ gtab,
                                                        const uint32_t* __restrict__ gskip) {
    constexpr int T = kMm1PanelT;
    constexpr int P = 32 * T;
    extern __shared__ uint32_t sm[];
    uint32_t* tab = sm;
    uint32_t* skip = sm + kLaneTabWords;
    {
        const uint4* src = reinterpret_cast<const uint4*>(gtab);
        uint4* dst = reinterpret_cast<uint4*>(tab);
        for (int i = threadIdx.x; i < kLaneTabWords / 4; i += blockDim.x) dst[i] = __ldg(src + i);
        for (int i = threadIdx.x; i < kUniTabWords; i += blockDim.x) skip[i] = __ldg(gskip + i);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double* buf = reinterpret_cast<double*>(sm + kLaneTabWords + kUniTabWords) + (threadIdx.x >> 5) * (2 * P);
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    const int64_t lo = warp * a.count / nwarps, hi = (warp + 1) * a.count / nwarps;
    double k0 = 0.0, k1 = 0.0, k2 = 0.0;
    for (int64_t r = lo; r < hi; ++r) {
        Taus st = lane_jump(tab, lane, load_seed(a, r));
        double w = 0.0, s = 0.0, idle = 0.0, sumw = 0.0, sums = 0.0;
        for (int64_t base = 0; base < a.n; base += P) {
#pragma unroll
            for (int j = 0; j < T; ++j) {
                const uint32_t ua = taus_next(st);
                const uint32_t us = taus_next(st);
                buf[j * 32 + lane] = expo<INV>(ua, a.lambda, a.inv_lambda);
                buf[P + j * 32 + lane] = expo<INV>(us, a.mu, a.inv_mu);
            }
            __syncwarp();
            if (lane == 0) {
                const int64_t left = a.n - base;
                const int cnt = left < P ? static_cast<int>(left) : P;
                for (int c = 0; c < cnt; ++c) {
                    const int idx = (c % T) * 32 + c / T;
                    const double av = buf[idx];
                    const double t = __dsub_rn(__dadd_rn(w, s), av);
                    if (t < 0.0) {  // server idle before this arrival
                        idle = __dsub_rn(idle, t);
                        w = 0.0;
                    } else {
                        w = t;
                    }
                    s = buf[P + idx];
                    sumw = __dadd_rn(sumw, w);
                    sums = __dadd_rn(sums, __dadd_rn(w, s));
                }
            }
            __syncwarp();
            st = uni_jump(skip, st);
        }
        const double nd = static_cast<double>(a.n);
        const double v0 = __shfl_sync(kFull, __ddiv_rn(idle, nd), 0);
        const double v1 = __shfl_sync(kFull, __ddiv_rn(sumw, nd), 0);
        const double v2 = __shfl_sync(kFull, __ddiv_rn(sums, nd), 0);
        const int slot = static_cast<int>((r - lo) & 31);
        if (lane == slot) {
            k0 = v0;
            k1 = v1;
            k2 = v2;
        }
        if (slot == 31 || r == hi - 1) {
            if (lane <= slot) {
                a.out0[r - slot + lane] = k0;
                a.out1[r - slot + lane] = k1;
                a.out2[r - slot + lane] = k2;
            }
        }
    }
}

// ---------------------------------------------------------------------------------
// TLP: one replication per thread (the comparison mapping)
// ---------------------------------------------------------------------------------

template <int MODEL, bool INV>
__global__ void k_tlp(RepArgs a) {
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.count) return;  // tail threads of the last block stay inert (wlp.cpp:125-138)
    Taus st = load_seed(a, r);
    if (MODEL == 0) {
        // c counts exactly (the reference accumulates 0.0/1.0 in a double, exact < 2^53)
        uint64_t c = 0;
        for (int64_t done = 0; done < a.n;) {
            const int64_t left = a.n - done;
            const uint32_t part = left > 0x40000000 ? 0x40000000u : static_cast<uint32_t>(left);
            c += pi_hits(st, part);
            done += part;
        }
        a.out0[r] = __ddiv_rn(__dmul_rn(4.0, static_cast<double>(c)), static_cast<double>(a.n));
    } else if (MODEL == 1) {
        double w = 0.0, s = 0.0, idle = 0.0, sumw = 0.0, sums = 0.0;
        for (int64_t i = 0; i < a.n; ++i) {
            const double av = expo<INV>(taus_next(st), a.lambda, a.inv_lambda);
            const double t = __dsub_rn(__dadd_rn(w, s), av);
            if (t < 0.0) {
                idle = __dsub_rn(idle, t);
                w = 0.0;
            } else {
                w = t;
            }
            s = expo<INV>(taus_next(st), a.mu, a.inv_mu);
            sumw = __dadd_rn(sumw, w);
            sums = __dadd_rn(sums, __dadd_rn(w, s));
        }
        const double nd = static_cast<double>(a.n);
        a.out0[r] = __ddiv_rn(idle, nd);
        a.out1[r] = __ddiv_rn(sumw, nd);
        a.out2[r] = __ddiv_rn(sums, nd);
    } else {
        // models.hpp:92-105 as written: a 4-way branch per step on d = floor(4u).
        double px = 0.0, py = 0.0;
        for (int64_t i = 0; i < a.n; ++i) {
            const uint32_t d = taus_next(st) >> 30;
            (void)taus_next(st);
            if (d == 0u)
                px = __dadd_rn(px, 1.0);
            else if (d == 1u)
                px = __dsub_rn(px, 1.0);
            else if (d == 2u)
                py = __dadd_rn(py, 1.0);
            else
                py = __dsub_rn(py, 1.0);
        }
        a.out0[r] = walk_fold(static_cast<int64_t>(px), a.chunks);
    }
}

// ---------------------------------------------------------------------------------
// Statistics
// ---------------------------------------------------------------------------------

__device__ __forceinline__ void two_sum(double& hi, double& lo, double v) {
    const double s = __dadd_rn(hi, v);
    const double bb = __dsub_rn(s, hi);
    const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(s, bb)), __dsub_rn(v, bb));
    hi = s;
    lo = __dadd_rn(lo, err);
}

__device__ __forceinline__ double stat_term(double x, int pass, double center) {
    if (pass == 1) return x;
    const double d = __dsub_rn(x, center);
    return __dmul_rn(d, d);
}

constexpr int kStatsBlock = 256;
constexpr int64_t kStatsSeqMax = 256;

__global__ void __launch_bounds__(kStatsBlock) k_stats(const double* __restrict__ x, int64_t n, int pass,
                                                       double center, double* __restrict__ partials) {
    if (n <= kStatsSeqMax) {  // the reference's naive sequential loop, bit for bit
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            double s = 0.0;
            for (int64_t i = 0; i < n; ++i) s = __dadd_rn(s, stat_term(x[i], pass, center));
            partials[0] = s;
            partials[1] = 0.0;
        }
        return;
    }
    double hi = 0.0, lo = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        two_sum(hi, lo, stat_term(__ldg(x + i), pass, center));
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double oh = __shfl_xor_sync(kFull, hi, o), ol = __shfl_xor_sync(kFull, lo, o);
        two_sum(hi, lo, oh);
        lo = __dadd_rn(lo, ol);
    }
    __shared__ double sh[2][kStatsBlock / 32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sh[0][w] = hi;
        sh[1][w] = lo;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double h = 0.0, l = 0.0;
        for (int i = 0; i < kStatsBlock / 32; ++i) {
            two_sum(h, l, sh[0][i]);
            l = __dadd_rn(l, sh[1][i]);
        }
        partials[2 * blockIdx.x] = h;
        partials[2 * blockIdx.x + 1] = l;
    }
}

}  // namespace

// ---------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------

int wlp_blocks_per_sm(int model) {
    int nb = 0;
    if (model == 1) {
        const size_t smem = (kLaneTabWords + kUniTabWords) * 4 + (kMm1Block / 32) * 2 * 32 * kMm1PanelT * 8;
        cudaFuncSetAttribute(k_wlp_mm1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaFuncSetAttribute(k_wlp_mm1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_mm1<false>, kMm1Block, smem);
    } else {
        const size_t smem = kLaneTabWords * 4;
        if (model == 0) {
            cudaFuncSetAttribute(k_wlp_lanes<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_lanes<0>, kWlpBlock, smem);
        } else {
            cudaFuncSetAttribute(k_wlp_lanes<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_lanes<2>, kWlpBlock, smem);
        }
    }
    return nb < 1 ? 1 : nb;
}

int tlp_blocks_per_sm(int model, int block) {
    int nb = 0;
    switch (model) {
        case 0: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp<0, false>, block, 0); break;
        case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp<1, false>, block, 0); break;
        default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp<2, false>, block, 0); break;
    }
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_seed(const SeedArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int64_t per_block = static_cast<int64_t>(kSeedBlock) * kSeedPerThread;
    const int64_t grid = (a.count + per_block - 1) / per_block;
    const size_t smem = 3 * kSeedBlock * (kSeedPerThread + 1) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        attr = true;
    }
    k_seed<<<static_cast<unsigned>(grid), kSeedBlock, smem, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_neg_log1m(const uint32_t* k, int64_t n, double* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_neg_log1m<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(k, n, out);
    return cudaGetLastError();
}

cudaError_t launch_taus_stream(const uint32_t* powers, Taus seed, int64_t n, uint32_t* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t threads = (n + kTausPerThread - 1) / kTausPerThread;
    const int block = 128;
    k_taus<<<static_cast<unsigned>((threads + block - 1) / block), block, 0, st>>>(powers, seed, n, out);
    return cudaGetLastError();
}

cudaError_t launch_wlp(int model, const RepArgs& a, const uint32_t* lane_tab, const uint32_t* uni_tab,
                       int64_t lane_units, int grid, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (model == 1) {
        const size_t smem = (kLaneTabWords + kUniTabWords) * 4 + (kMm1Block / 32) * 2 * 32 * kMm1PanelT * 8;
        if (a.inv_lambda != 0.0 && a.inv_mu != 0.0)
            k_wlp_mm1<true><<<grid, kMm1Block, smem, st>>>(a, lane_tab, uni_tab);
        else
            k_wlp_mm1<false><<<grid, kMm1Block, smem, st>>>(a, lane_tab, uni_tab);
    } else if (model == 0) {
        k_wlp_lanes<0><<<grid, kWlpBlock, kLaneTabWords * 4, st>>>(a, lane_tab, lane_units);
    } else {
        k_wlp_lanes<2><<<grid, kWlpBlock, kLaneTabWords * 4, st>>>(a, lane_tab, lane_units);
    }
    return cudaGetLastError();
}

cudaError_t launch_tlp(int model, const RepArgs& a, int tlp_block, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int64_t block = a.count < tlp_block ? a.count : tlp_block;
    const int64_t grid = (a.count + block - 1) / block;
    const bool inv = a.inv_lambda != 0.0 && a.inv_mu != 0.0;
    const dim3 g(static_cast<unsigned>(grid)), b(static_cast<unsigned>(block));
    switch (model) {
        case 0: k_tlp<0, false><<<g, b, 0, st>>>(a); break;
        case 1:
            if (inv)
                k_tlp<1, true><<<g, b, 0, st>>>(a);
            else
                k_tlp<1, false><<<g, b, 0, st>>>(a);
            break;
        default: k_tlp<2, false><<<g, b, 0, st>>>(a); break;
    }
    return cudaGetLastError();
}

cudaError_t launch_stats(const double* x, int64_t n, int pass, double center, double* partials, int grid,
                         cudaStream_t st) {
    if (n <= kStatsSeqMax) grid = 1;
    k_stats<<<grid, kStatsBlock, 0, st>>>(x, n, pass, center, partials);
    return cudaGetLastError();
}

}  // namespace wlp
