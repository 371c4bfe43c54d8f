// sm_100a kernels of the WLP replication engine. No tensor cores: every kernel here is
// integer / FP64 ALU work bounded by instruction issue and the ALU / FP64 pipes (see
// DESIGN.md §roofline).
//
//   k_seed       random_spacing (rng.cpp:67-87) by jump-ahead: thread t fills 32 stream
//                slots from master draw 3*c(t) on, flags "special" candidates.
//   k_taus       raw taus88 stream (taus88.golden format) by jump-ahead.
//   k_wlp_lanes  pi / walk, one replication per warp; lane l consumes the replication's
//                units [l*K, (l+1)*K) after one nibble-table jump; exact integer
//                warp reduction (__reduce_add_sync) of hits / x-displacement.
//   k_wlp_mm1    mm1, one replication per warp; lanes produce the exponentials of a
//                32*T-client panel, chain the Lindley recursion (models.hpp:61-84) across
//                their segments by exact fixed-point rounds, and lanes 0-2 run the three
//                order-dependent sums.
//   k_tlp        the thread-per-replication comparison mapping (plan_launch TLP
//                geometry, wlp.cpp:88-92); mm1 shares the batched exponential routine.
//   k_stats      sums / centred sums of squares for the confidence interval.
//
// Compiled with --fmad=false: the reference is built with -ffp-contract=off
// (CMakeLists.txt:12-13), so no a*b+c may fuse; the only FMAs are the explicit ones in
// the glibc log port.
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

#include "bitslice.cuh"
#include "glibc_log.cuh"
#include "jump.hpp"
#include "kernels.cuh"

namespace wlp {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;

// Programmatic dependent launch (sm_90+): a model kernel launched with the programmatic
// stream-serialization attribute right after the seeding kernel may start while the
// seeding drains; pdl_wait() (griddepcontrol.wait) then holds it until the seeding grid
// has completed and its writes are visible. Each model kernel waits after its own
// prologue (shared-memory table staging) and before its first read of the seeds or the
// work counter; launched without the attribute, the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


// Nibble-table application from global memory (L1-resident tables): 8 independent loads
// and an XOR tree.
__device__ __forceinline__ uint32_t nib_apply_g(const uint32_t* __restrict__ t, uint32_t x) {
    uint32_t y[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) y[p] = __ldg(t + p * 16 + ((x >> (4 * p)) & 15u));
    return ((y[0] ^ y[1]) ^ (y[2] ^ y[3])) ^ ((y[4] ^ y[5]) ^ (y[6] ^ y[7]));
}

// The same for a lane-major table ([p][v][lane], row stride 32 words) in global memory.
__device__ __forceinline__ uint32_t nib_apply_g32(const uint32_t* __restrict__ t, uint32_t x) {
    uint32_t y[8];
#pragma unroll
    for (int p = 0; p < 8; ++p) y[p] = __ldg(t + (p * 16 + ((x >> (4 * p)) & 15u)) * 32);
    return ((y[0] ^ y[1]) ^ (y[2] ^ y[3])) ^ ((y[4] ^ y[5]) ^ (y[6] ^ y[7]));
}

// Jump n draws with the binary powers M^(2^k) as nibble tables ([k][comp][p][v], jump.hpp
// flat_nibble_powers): per set bit of n one nibble application per component.
__device__ Taus jump_pow(const uint32_t* __restrict__ pn, Taus t, uint64_t n) {
    while (n) {
        const int k = __ffsll(static_cast<long long>(n)) - 1;
        n &= n - 1;
        const uint32_t* m = pn + k * kUniTabWords;
        t.s1 = nib_apply_g(m, t.s1);
        t.s2 = nib_apply_g(m + 128, t.s2);
        t.s3 = nib_apply_g(m + 256, t.s3);
    }
    return t;
}

// jump_pow with the binary-power tables staged in shared memory (k powers, k >= bits of n).
__device__ Taus jump_pow_s(const uint32_t* pn, Taus t, uint64_t n) {
    while (n) {
        const int k = __ffsll(static_cast<long long>(n)) - 1;
        n &= n - 1;
        const uint32_t* m = pn + k * kUniTabWords;
        uint32_t y1[8], y2[8], y3[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            y1[p] = m[p * 16 + ((t.s1 >> (4 * p)) & 15u)];
            y2[p] = m[128 + p * 16 + ((t.s2 >> (4 * p)) & 15u)];
            y3[p] = m[256 + p * 16 + ((t.s3 >> (4 * p)) & 15u)];
        }
        t.s1 = ((y1[0] ^ y1[1]) ^ (y1[2] ^ y1[3])) ^ ((y1[4] ^ y1[5]) ^ (y1[6] ^ y1[7]));
        t.s2 = ((y2[0] ^ y2[1]) ^ (y2[2] ^ y2[3])) ^ ((y2[4] ^ y2[5]) ^ (y2[6] ^ y2[7]));
        t.s3 = ((y3[0] ^ y3[1]) ^ (y3[2] ^ y3[3])) ^ ((y3[4] ^ y3[5]) ^ (y3[6] ^ y3[7]));
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

// Output stores: the device arrays, and the host mirrors when the run writes the host's
// pinned buffers directly (RepArgs::h0..h2).
__device__ __forceinline__ void put1(const RepArgs& a, int64_t r, double v) {
    a.out0[r] = v;
    if (a.h0) a.h0[r] = v;
}
__device__ __forceinline__ void put3(const RepArgs& a, int64_t r, double v0, double v1, double v2) {
    a.out0[r] = v0;
    a.out1[r] = v1;
    a.out2[r] = v2;
    if (a.h0) {
        a.h0[r] = v0;
        a.h1[r] = v1;
        a.h2[r] = v2;
    }
}

__device__ __forceinline__ Taus load_seed(const RepArgs& a, int64_t r) {
    return Taus{__ldg(a.seeds + r), __ldg(a.seeds + a.count + r), __ldg(a.seeds + 2 * a.count + r)};
}

template <int WORDS>
__device__ __forceinline__ void stage_u32(uint32_t* dst, const uint32_t* __restrict__ src) {
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    for (int i = threadIdx.x; i < WORDS / 4; i += blockDim.x) d[i] = __ldg(s + i);
}

__device__ __forceinline__ void stage_log_table(double* dst) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) dst[i] = kLogTabDev[i];
}

// Warp-level load instructions of a `for (i = tid; i < total; i += blockDim)` staging
// loop: the iterations of the warp's first lane.
__device__ __forceinline__ unsigned staged_loads(int total) {
    const int first = static_cast<int>(threadIdx.x) & ~31;
    return first < total ? static_cast<unsigned>((total - first + blockDim.x - 1) / blockDim.x) : 0u;
}

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

__device__ __forceinline__ long long hw_clock() { return clock64(); }

__device__ __forceinline__ void flush_tally(const HwTally& h, unsigned long long* hw) {
    const unsigned act = __activemask();
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(act) - 1)) {
        if (h.div) atomicAdd(hw, static_cast<unsigned long long>(h.div));
        if (h.ld) atomicAdd(hw + 1, static_cast<unsigned long long>(h.ld));
        if (h.st) atomicAdd(hw + 2, static_cast<unsigned long long>(h.st));
        if (h.splits) atomicAdd(hw + 3, static_cast<unsigned long long>(h.splits));
        const unsigned sm = smid();
        if (sm < static_cast<unsigned>(kHwMaxSms)) {
            atomicMin(hw + kHwClk + sm, static_cast<unsigned long long>(h.t0));
            atomicMax(hw + kHwClk + kHwMaxSms + sm, static_cast<unsigned long long>(hw_clock()));
        }
    }
}

// Divergence events of one execution of a loop whose trip count `trips` differs per lane
// (the reference's While event, warp_exec.cpp:286-293: an evaluation of the condition
// where some active lanes enter and some skip). The lanes leave in groups of equal trip
// count, and every group but the last leaves while others stay: events = the number of
// distinct trip counts among the `mask` lanes, minus one. (All lanes call it.)
__device__ __forceinline__ unsigned loop_split_events(unsigned mask, unsigned trips) {
    const unsigned same = __match_any_sync(mask, trips);
    const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
    const unsigned firsts = __ballot_sync(mask, (same & lt & mask) == 0u);
    return static_cast<unsigned>(__popc(firsts)) - 1u;
}

// Inside test of one pi point, x*x + y*y <= 1.0 in unfused fp64 (models.hpp:54-56),
// evaluated on the unscaled draws: with x = a*2^-32 every product and sum is the
// reference's value times 2^64 exactly (power-of-two scaling commutes with rounding
// in the normal range), so the test is fl(fl(a*a) + fl(b*b)) <= 2^64.
// hits += inside as one compare and one predicated add (from C++ the compiler adds
// unconditionally and then undoes the add under the opposite predicate).
__device__ __forceinline__ void pi_count(uint32_t& hits, uint32_t a, uint32_t b) {
    const double x = __uint2double_rn(a), y = __uint2double_rn(b);
    const double s = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
    asm("{\n\t.reg .pred p;\n\tsetp.le.f64 p, %1, 0d43F0000000000000;\n\t@p add.u32 %0, %0, 1;\n\t}"
        : "+r"(hits)
        : "d"(s));
}


// Hits among `units` consecutive points of a stream (main loop unrolled by 8).
__device__ __forceinline__ uint32_t pi_hits(Taus& st, uint32_t units) {
    uint32_t hits = 0;
    for (uint32_t it = units >> 3; it; --it) {  // (a count-down: one counter, no bound)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t x, y;
            taus_next2(st, x, y);
            pi_count(hits, x, y);
        }
    }
    for (uint32_t u = units & 7u; u; --u) {
        uint32_t x, y;
        taus_next2(st, x, y);
        pi_count(hits, x, y);
    }
    return hits;
}

// x displacement of `units` consecutive walk steps (direction d = floor(4u) = out >> 30,
// second draw of each step discarded, models.hpp:93-104): dx = #(d==0) - #(d==1). Per
// step we add the cubic q(d) = -4d^3 + 21d^2 - 29d (= 6*([d==0]-[d==1]) - 6 on {0..3}) by
// Horner in three IMADs (FMA pipe) instead of compares and selects (ALU pipe); then
// dx = (sum q + 6*units) / 6 exactly. |sum| <= 12*units < 2^31 for units < 2^27.
// The raw sum of q over `units` steps (units < 2^27); dx = (sum + 6*units) / 6.
__device__ __forceinline__ int walk_q(Taus& st, uint32_t units) {
    int acc = 0;
    for (uint32_t it = units >> 3; it; --it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int d = static_cast<int>(taus_next_skip1(st) >> 30);
            acc += (((21 - 4 * d) * d) - 29) * d;
        }
    }
    for (uint32_t u = units & 7u; u; --u) {
        const int d = static_cast<int>(taus_next_skip1(st) >> 30);
        acc += (((21 - 4 * d) * d) - 29) * d;
    }
    return acc;
}

__device__ __forceinline__ int walk_dx_block(Taus& st, uint32_t units) {
    int acc = 0;
    uint32_t u = 0;
    for (; u + 4 <= units; u += 4) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int d = static_cast<int>(taus_next_skip1(st) >> 30);
            acc += (((21 - 4 * d) * d) - 29) * d;
        }
    }
    for (; u < units; ++u) {
        const int d = static_cast<int>(taus_next_skip1(st) >> 30);
        acc += (((21 - 4 * d) * d) - 29) * d;
    }
    return (acc + 6 * static_cast<int>(units)) / 6;
}

__device__ __forceinline__ int walk_dx(Taus& st, uint32_t units) {
    int dx = 0;
    while (units > (1u << 24)) {
        dx += walk_dx_block(st, 1u << 24);
        units -= 1u << 24;
    }
    return dx + walk_dx_block(st, units);
}

__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// fold of the walk's final x (models.hpp:106-107), in the reference's own arithmetic:
// c = (double)chunks (rounded above 2^53, as there), fmod(fmod(px, c) + c, c). fmod is
// exact in IEEE arithmetic on both sides; px is an exact integer (|px| <= steps).
__device__ __forceinline__ double walk_fold(int64_t px, int64_t chunks) {
    // For integers below 2^31 both fmods are exact integer remainders (fmod is exact, the
    // operands are exact doubles, r + c is exact), and the result is never -0 (r + c > 0),
    // so 32-bit remainders give the same value at a fraction of fmod's cost.
    if (chunks > 0 && chunks <= 0x7FFFFFFF && px >= -0x7FFFFFFF && px <= 0x7FFFFFFF) {
        const int32_t c = static_cast<int32_t>(chunks);
        const int32_t r = static_cast<int32_t>(px) % c;  // sign of px, as fmod; |r| < c
        return static_cast<double>(r < 0 ? r + c : r);    // (r + c) mod c
    }
    const double c = static_cast<double>(chunks);
    return fmod(__dadd_rn(fmod(static_cast<double>(px), c), c), c);
}

// ---------------------------------------------------------------------------------
// mm1 exponentials: -log(1 - u)/rate for a batch of draws per lane, warp-cooperative.
//
// glibc's log has two algorithms: the table path and, for 1 - 2^-4 <= x < 1 + ..., a
// longer polynomial (1 in 16 model draws). Per lane the branch is data dependent, so a
// warp that evaluates draws lane by lane runs both paths almost always (1-(15/16)^32 =
// 87%). Instead every input goes through the table path (branch-free), and the
// near-one inputs of the whole warp are compacted (ballot/popc) and evaluated once, spread
// over the lanes; their results replace the table-path values.
// ---------------------------------------------------------------------------------

constexpr int kExpoB = 8;  // log inputs per lane per batch

struct NearList {  // per-warp compaction scratch
    uint32_t n[32 * kExpoB];
};

// -log(1 - n*2^-32) for every lane's B inputs. Each lane flags its near-one inputs in a
// B-bit mask; an exclusive prefix sum of the flag counts over the lanes (five shuffles per
// batch, instead of a ballot and popcounts per input) places them in nl, each is
// evaluated by one lane into res[pos], and picked up by its owner. FULL: all 32 lanes take
// part; else `mask_` names the (contiguous, low) lanes of a partial warp.
// ev (instrumented kernels): add the near-one loop's divergence events (its lanes run
// different trip counts whenever the list is not a multiple of the warp width).
template <int B, bool FULL>
__device__ __forceinline__ void neg_log1m_batch(const uint32_t (&n)[B], double (&e)[B], const double* tab,
                                                NearList& nl, double* res, unsigned mask_, int lane,
                                                unsigned* ev = nullptr) {
    static_assert(B <= 32, "near flags fit one word");
    const unsigned mask = FULL ? kFull : mask_;
    unsigned near = 0;
    bool nr[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
        // 1 - u >= 1 - 2^-4 (glibc's near-one window) exactly when n <= 2^28; n = 0 (1 - u
        // = 1) is near too, so the table path may see the wrapped x = 0 there: its value is
        // replaced below
        e[j] = neg_log1m_table_dev(n[j], tab);
        nr[j] = n[j] <= 0x10000000u;
        if (nr[j]) near |= 1u << j;
    }
    const int c = __popc(near);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(mask, incl, o);
        if (lane >= o) incl += v;
    }
    const int width = FULL ? 32 : __popc(mask);
    const int total = __shfl_sync(mask, incl, width - 1);
    if (total == 0) return;  // warp-uniform
    // predicated store then pointer bump, in this order (as C++ the compiler bumps into a
    // temporary first and copies it back: one instruction more per input)
    uint32_t sp = static_cast<uint32_t>(__cvta_generic_to_shared(nl.n + (incl - c)));
#pragma unroll
    for (int j = 0; j < B; ++j)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p st.shared.u32 [%0], %1;\n\t"
                     "@p add.u32 %0, %0, 4;\n\t}"
                     : "+r"(sp)
                     : "r"(n[j]), "r"(static_cast<uint32_t>(nr[j]))
                     : "memory");
    __syncwarp(mask);
    if (ev) *ev += loop_split_events(mask, lane < total ? static_cast<unsigned>((total - lane + width - 1) / width) : 0u);
    for (int p = lane; p < total; p += width) {
        const uint32_t v = nl.n[p];
        res[p] = v == 0u ? -0.0 : -log_near_one_dev(one_minus_u32_dev(v));
    }
    __syncwarp(mask);
    uint32_t rp = static_cast<uint32_t>(__cvta_generic_to_shared(res + (incl - c)));
#pragma unroll
    for (int j = 0; j < B; ++j)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.f64 %1, [%0];\n\t"
                     "@p add.u32 %0, %0, 8;\n\t}"
                     : "+r"(rp), "+d"(e[j])
                     : "r"(static_cast<uint32_t>(nr[j]))
                     : "memory");
    __syncwarp(mask);
}

// e / rate in IEEE double (models.hpp:67,75 divide -log(1 - u) by lambda or mu).
// kDivRcp: inv = RN(1/rate), q = RN(e * inv) is within an ulp of e / rate, the residual
// rate * q - e is exact in one FMA, and q - residual * inv rounds to RN(e / rate)
// (Markstein's correction); the residual's sign convention keeps -0 / rate = -0. Checked
// against __ddiv_rn for every numerator the model can produce (2^32 draws) at 1083
// rates plus 2e12 random pairs (tools/div_check.cu). Valid away from over/underflow:
// the host picks kDivIeee for rates outside [2^-900, 2^900].
template <int DIV>
__device__ __forceinline__ double scale(double e, double rate, double inv) {
    if constexpr (DIV == kDivPow2 || DIV == kDivPow2One) {  // (kDivPow2One: arrivals; services below)
        return __dmul_rn(e, inv);
    } else if constexpr (DIV == kDivRcp) {
        const double q = __dmul_rn(e, inv);
        return __fma_rn(-__fma_rn(rate, q, -e), inv, q);
    } else {
        return __ddiv_rn(e, rate);
    }
}

// One client of the Lindley recursion (models.hpp:67-78) in the reference's rounding:
//   t = (w + s) - a;  if (t < 0) { idle -= t; w = 0 } else w = t;  s = s';
//   sumw += w;  sums += (w + s)
// * u = fl(w + s) is carried: the next client's (w + s) has the same operands as this
//   client's sums term.
// * The branch clears t's two words when its sign bit is set. t is never -0 or NaN here
//   (u >= +0, a finite), so this is w = t < 0 ? +0 : t.
// * idle - t == idle + fl(w - t) exactly: -t when dry, and idle + (+0) == idle otherwise
//   (idle >= +0).
struct Queue {
    double u = 0.0, idle = 0.0, sumw = 0.0, sums = 0.0;
    // returns whether the `t < 0` branch (server idle) was taken
    __device__ __forceinline__ bool client(double a, double s_next) {
        const double t = __dsub_rn(u, a);
        const int hi = __double2hiint(t), keep = ~(hi >> 31);
        const double w = __hiloint2double(hi & keep, __double2loint(t) & keep);
        idle = __dadd_rn(idle, __dsub_rn(w, t));
        u = __dadd_rn(w, s_next);
        sumw = __dadd_rn(sumw, w);
        sums = __dadd_rn(sums, u);
        return hi < 0;
    }
};

// ---------------------------------------------------------------------------------
// Seeding
// ---------------------------------------------------------------------------------

// Shared-memory staging of the seeding: slots are produced and written out in batches of
// kB = min(PER, 32) slots per thread, 3 x [kSeedBlock][kRow] words. A batch of 32 uses
// an XOR swizzle (word j of row r at r*32 + (j ^ r)) instead of a padded row: 12 KB per
// block, so a whole 1e7-stream run (2,442 blocks of 32 threads at 128 slots) is resident
// in one wave (17 blocks per SM) where the 128-slot padded staging (49.5 KB) allowed 4.
__host__ __device__ constexpr int seed_batch(int per) { return per < 32 ? per : 32; }
__host__ __device__ constexpr int seed_row(int per) { return seed_batch(per) == 32 ? 32 : seed_batch(per) + 1; }
__host__ __device__ constexpr int seed_stage_words(int per) { return 3 * kSeedBlock * seed_row(per); }
template <int PER>
__device__ __forceinline__ int seed_sidx(int r, int j) {
    return r * seed_row(PER) + (seed_batch(PER) == 32 ? (j ^ r) : j);
}

// One block of stream slots of one random_spacing run: slots [blk*B, (blk+1)*B) of
// `count` (B = kSeedBlock * PER), slot i = candidate c(slot_begin + i) after
// the sorted rejection list; keys land SoA at out[plane*stride + out_off + i]. Thread t
// walks the master stream over slots [t*PER, (t+1)*PER) of the block (one jump-ahead),
// staging kB slots at a time; each batch is written out as kSeedBlock runs of kB
// consecutive slots (coalesced), and for the walk as one bit-plane group per thread.
template <int PER, bool STAGED = false>
__device__ __forceinline__ void seed_block(const uint32_t* __restrict__ pw, Taus master, int64_t slot_begin,
                                           int64_t count, int64_t blk, const int64_t* __restrict__ rejected,
                                           int64_t n_rejected, uint32_t* __restrict__ out, int64_t out_off,
                                           int64_t stride, SpecialRec* specials, int64_t special_cap,
                                           unsigned long long* n_special, uint32_t job,
                                           uint32_t* __restrict__ planes = nullptr, const uint32_t* spw = nullptr) {
    extern __shared__ uint32_t sh[];  // 3 x [kSeedBlock][kRow] (padded or swizzled: conflict-free)
    constexpr int kB = seed_batch(PER);
    constexpr int kPlane = kSeedBlock * seed_row(PER);
    static_assert(PER % kB == 0, "whole batches");
    const int tid = threadIdx.x;
    const int64_t blk0 = blk * kSeedBlock * PER;
    const int64_t my0 = blk0 + static_cast<int64_t>(tid) * PER;
    const int64_t left = count - my0;
    const int nmine = left <= 0 ? 0 : (left < PER ? static_cast<int>(left) : PER);
    int64_t c = slot_begin + my0;  // candidate index of my next slot
    int64_t ri = 0;
    Taus m{};
    if (nmine > 0) {
        while (ri < n_rejected && rejected[ri] <= c) {
            ++c;
            ++ri;
        }
        m = STAGED ? jump_pow_s(spw, master, 3ull * static_cast<uint64_t>(c))
                   : jump_pow(pw, master, 3ull * static_cast<uint64_t>(c));
    }
    int64_t nblk = count - blk0;
    if (nblk > kSeedBlock * PER) nblk = kSeedBlock * PER;
    // no redrawn candidate among my slots (the rule: rejections are rare collisions), so
    // the slot loop needs no rejection test
    const bool clean = ri >= n_rejected || rejected[ri] >= c + nmine;
    const bool full_blk = nblk == kSeedBlock * PER;
    auto special = [&](const Taus& key) {
        if (is_special_key(key)) {
            const unsigned long long pos = atomicAdd(n_special, 1ull);
            if (static_cast<int64_t>(pos) < special_cap) {
                SpecialRec* sp = specials + pos;
                sp->index = c;
                sp->s1 = key.s1;
                sp->s2 = key.s2;
                sp->s3 = key.s3;
                sp->pad = job;
            }
        }
    };
    auto stage = [&](int j, const Taus& key) {
        const int si = seed_sidx<PER>(tid, j);
        sh[si] = key.s1;
        sh[kPlane + si] = key.s2;
        sh[2 * kPlane + si] = key.s3;
    };
#pragma unroll 1
    for (int b0 = 0; b0 < PER && b0 < nblk; b0 += kB) {
        const int nb = nmine - b0 < 0 ? 0 : (nmine - b0 < kB ? nmine - b0 : kB);
        if (clean) {
            for (int j = 0; j < nb; ++j) {
                uint32_t x, y;
                taus_next2(m, x, y);
                const uint32_t z = taus_next(m);
                const Taus key = make_state(x, y, z);
                special(key);
                ++c;
                stage(j, key);
            }
        } else {
            for (int j = 0; j < nb; ++j) {
                Taus key;
                for (;;) {
                    const uint32_t x = taus_next(m), y = taus_next(m), z = taus_next(m);
                    key = make_state(x, y, z);
                    if (ri < n_rejected && rejected[ri] == c) {  // a redrawn candidate
                        ++ri;
                        ++c;
                        continue;
                    }
                    break;
                }
                special(key);
                ++c;
                stage(j, key);
            }
        }
        __syncthreads();
        if (kB == 32 && planes != nullptr) {  // the walk's bit planes: this batch is one group
            const int64_t s0 = my0 + b0;
            if (s0 < count) {
                BsTaus t;
                if (s0 + 32 <= count) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int si = seed_sidx<PER>(tid, j);
                        t.b1[j] = sh[si];
                        t.b2[j] = sh[kPlane + si];
                        t.b3[j] = sh[2 * kPlane + si];
                    }
                } else {  // a ragged last group: idle streams at the minimum state
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const bool in = s0 + j < count;
                        const int si = seed_sidx<PER>(tid, j);
                        t.b1[j] = in ? sh[si] : kMin1;
                        t.b2[j] = in ? sh[kPlane + si] : kMin2;
                        t.b3[j] = in ? sh[2 * kPlane + si] : kMin3;
                    }
                }
                bs_store_planes(t, planes + (s0 / 32) * kBsLive);
            }
        }
        if (kB == 32 && planes != nullptr) {
            // the bitsliced walk pipeline reads the planes alone (its wrap groups' seeds too)
        } else if (kB == 32 && full_blk) {  // row r's batch is 32 consecutive slots: lane k stores slot k
            uint32_t* o = out + out_off + blk0 + b0 + tid;
#pragma unroll 8
            for (int r = 0; r < kSeedBlock; ++r) {
                const int si = seed_sidx<PER>(r, tid);
                o[r * PER] = sh[si];
                o[stride + r * PER] = sh[kPlane + si];
                o[2 * stride + r * PER] = sh[2 * kPlane + si];
            }
        } else {
            for (int i = tid; i < kSeedBlock * kB; i += kSeedBlock) {
                const int r = i / kB, k = i % kB;
                const int64_t g = blk0 + static_cast<int64_t>(r) * PER + b0 + k;  // (row r's slots are consecutive)
                if (g < count) {
                    const int si = seed_sidx<PER>(r, k);
                    out[out_off + g] = sh[si];
                    out[stride + out_off + g] = sh[kPlane + si];
                    out[2 * stride + out_off + g] = sh[2 * kPlane + si];
                }
            }
        }
        __syncthreads();  // (the next batch overwrites the staging)
    }
}

// The last block of a seeding grid to finish stores the final specials count to `report`
// (mapped pinned host memory: the host polls it, no copy launch) and rearms `done`;
// `rearm_count` also clears the count (all other blocks' atomics are done by then).
__device__ __forceinline__ void seed_report(unsigned int* done, unsigned long long* report,
                                            unsigned long long* n_special, bool rearm_count) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(done, 1u) == gridDim.x - 1) {
            __threadfence_system();  // the specials list before the count the host polls
            *done = 0u;
            const unsigned long long n = atomicAdd(n_special, 0ull);
            if (rearm_count) *n_special = 0ull;
            *reinterpret_cast<volatile unsigned long long*>(report) = n;
        }
    }
}

// (at most 120 registers: 17 blocks of a 1e7-stream run per SM, its 2,442 blocks in one wave)
template <int PER>
__global__ void __maxnreg__(120) k_seed(SeedArgs a) {
    pdl_wait();     // (launched early behind the previous run's kernels: they read what this writes)
    pdl_trigger();  // the model kernel may launch now; it waits for this grid to complete
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (a.zero_a) *a.zero_a = 0ull;
        if (a.zero_b) *a.zero_b = 0ull;
    }
    if constexpr (PER == 8) {
        // small runs: a thread's jump is a chain of ~10 dependent table steps, each an L2
        // round trip from global memory; staged in shared memory (the powers up to the
        // run's largest candidate, 29 KB at R = 1e5), the chain runs at shared-memory latency.
        // The copy is one TMA bulk transfer (cp.async.bulk, completion counted on an
        // mbarrier): a plain load/store loop kept one L2 round trip per iteration in
        // flight and cost ~10 us of this ~10 us kernel.
        extern __shared__ __align__(16) uint32_t sh[];
        __shared__ __align__(8) uint64_t bar;
        uint32_t* spw = sh + seed_stage_words(PER);
        const uint32_t bytes = static_cast<uint32_t>(a.stage_powers) * kUniTabWords * 4;
        const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             static_cast<uint32_t>(__cvta_generic_to_shared(spw))),
                         "l"(a.powers), "r"(bytes), "r"(b)
                         : "memory");
        }
        __syncthreads();  // (the barrier is initialised before anyone waits on it)
        asm volatile(
            "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(b)
            : "memory");
        seed_block<PER, true>(a.powers, a.master, a.slot_begin, a.count, blockIdx.x, a.rejected, a.n_rejected, a.out,
                              a.out_off, a.stride ? a.stride : a.count, static_cast<SpecialRec*>(a.specials),
                              a.special_cap, a.n_special, 0u, a.planes, spw);
    } else {
        seed_block<PER>(a.powers, a.master, a.slot_begin, a.count, blockIdx.x, a.rejected, a.n_rejected, a.out,
                        a.out_off, a.stride ? a.stride : a.count, static_cast<SpecialRec*>(a.specials),
                        a.special_cap, a.n_special, 0u, a.planes);
    }
    if (a.report) seed_report(a.done, a.report, a.n_special, false);
}

// Many independent runs (one per plan set) in one launch; block -> job by binary search.
__global__ void __launch_bounds__(kSeedBlock) k_seed_jobs(const uint32_t* __restrict__ pw,
                                                          const SeedJob* __restrict__ jobs, int n_jobs,
                                                          uint32_t* __restrict__ out, int64_t total,
                                                          SpecialRec* specials, int64_t special_cap,
                                                          unsigned long long* n_special,
                                                          unsigned long long* zero_a, unsigned int* done,
                                                          unsigned long long* report) {
    pdl_wait();     // (may launch behind the previous plan's model, which reads the seeds)
    pdl_trigger();  // the plan's model may launch now; it waits for this grid to complete
    if (zero_a && blockIdx.x == 0 && threadIdx.x == 0) *zero_a = 0ull;  // the model's grab counter
    int lo = 0, hi = n_jobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (jobs[mid].block0 <= static_cast<int64_t>(blockIdx.x))
            lo = mid;
        else
            hi = mid - 1;
    }
    const SeedJob& J = jobs[lo];
    seed_block<kSeedJobPer>(pw, J.master, 0, J.count, blockIdx.x - J.block0, nullptr, 0, out, J.out_off, total, specials,
               special_cap, n_special, static_cast<uint32_t>(lo));
    if (report) seed_report(done, report, n_special, true);
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

// -log(1 - k*2^-32) through the production batch routine (pins the device log port).
constexpr int kLogHookBlock = 256;
__global__ void __launch_bounds__(kLogHookBlock) k_neg_log1m(const uint32_t* __restrict__ k, int64_t n,
                                                             double* __restrict__ out) {
    __shared__ double tab[256];
    __shared__ NearList nl[kLogHookBlock / 32];
    __shared__ double res[kLogHookBlock / 32][32 * kExpoB];
    stage_log_table(tab);
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * kExpoB;
    uint32_t in[kExpoB];
    double e[kExpoB];
#pragma unroll
    for (int j = 0; j < kExpoB; ++j) in[j] = base + j < n ? k[base + j] : 0u;
    neg_log1m_batch<kExpoB, true>(in, e, tab, nl[w], res[w], kFull, lane);
#pragma unroll
    for (int j = 0; j < kExpoB; ++j)
        if (base + j < n) out[base + j] = e[j];
}

// ---------------------------------------------------------------------------------
// WLP: one replication per warp
// ---------------------------------------------------------------------------------

// Work distribution of the persistent WLP grids: a warp takes a.grab consecutive
// replications from a global counter (lane 0's atomic is issued one group ahead, so its
// latency hides behind the current group). Static splits left a tail: the issue arbiter
// favours some warps, which then finish long before the others. Results of a group are
// parked in lanes 0..grab-1 and stored together (coalesced).
__device__ __forceinline__ unsigned long long grab_issue(const RepArgs& a, int lane) {
    return lane == 0 ? atomicAdd(a.next, static_cast<unsigned long long>(a.grab)) : 0ull;
}

__device__ __forceinline__ int64_t grab_take(unsigned long long ticket) {
    return static_cast<int64_t>(__shfl_sync(kFull, ticket, 0));
}

template <int MODEL, bool COUNT>
__global__ void __launch_bounds__(kWlpBlock, 4) k_wlp_lanes(RepArgs a, const uint32_t* __restrict__ gtab,
                                                             int64_t K) {
    extern __shared__ uint32_t tab[];  // kLaneTabWords
    stage_u32<kLaneTabWords>(tab, gtab);
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    HwTally hw;
    if (COUNT) {
        hw.t0 = hw_clock();
        hw.ld = staged_loads(kLaneTabWords / 4);
    }
    int64_t mine = a.n - static_cast<int64_t>(lane) * K;
    mine = mine < 0 ? 0 : (mine > K ? K : mine);
    const uint32_t units = static_cast<uint32_t>(mine);
    const bool wide = a.n >= (int64_t(1) << 31);
    // The model's branches are arithmetic here (pi's count is a predicated add, the walk's
    // direction a polynomial), so a warp splits only where its lanes' unit loops end at
    // different trips (pi_hits: 8-point main loop and tail; walk_dx: 2^24-step blocks, 4-step
    // main loop, tail). The lanes' units are fixed for the launch, so every replication
    // splits the same way: count it once per warp.
    unsigned ev_rep = 0;
    if (COUNT) {
        if (MODEL == 0) {
            ev_rep = loop_split_events(kFull, units / 8) + loop_split_events(kFull, units % 8);
        } else {
            const unsigned blocks = units > (1u << 24) ? (units - 1u) >> 24 : 0u;  // walk_dx's while
            const unsigned last = units - (blocks << 24);
            ev_rep = loop_split_events(kFull, blocks) + loop_split_events(kFull, last / 4) +
                     loop_split_events(kFull, last % 4);
        }
    }
    for (int64_t base = grab_take(grab_issue(a, lane)); base < a.count;) {
        const unsigned long long ticket = grab_issue(a, lane);  // next group, in flight
        const int64_t end = base + a.grab < a.count ? base + a.grab : a.count;
        double keep = 0.0;
        for (int64_t r = base; r < end; ++r) {
            Taus st = lane_jump(tab, lane, load_seed(a, r));
            double val;
            if (MODEL == 0) {  // pi: count points inside the quarter circle
                const uint32_t hits = pi_hits(st, units);
                const int64_t total =
                    wide ? warp_sum_i64(hits) : static_cast<int64_t>(__reduce_add_sync(kFull, hits));
                // c counts exactly in a double, so (4.0*c)/draws is the reference's value.
                val = __ddiv_rn(__dmul_rn(4.0, static_cast<double>(total)), static_cast<double>(a.n));
            } else {  // walk: only the x displacement reaches the output
                const int dx = walk_dx(st, units);
                const int64_t total = wide ? warp_sum_i64(dx) : static_cast<int64_t>(__reduce_add_sync(kFull, dx));
                val = walk_fold(total, a.chunks);
            }
            if (lane == static_cast<int>(r - base)) keep = val;
        }
        if (lane < end - base) put1(a, base + lane, keep);
        if (COUNT) {
            hw.ld += 3 * static_cast<unsigned>(end - base);
            hw.st += 1;
            hw.splits += ev_rep * static_cast<unsigned>(end - base);
        }
        base = grab_take(ticket);
    }
    if (COUNT) flush_tally(hw, a.hw);
}

// WLP as a systolic warp pipeline (pi / walk, many short replications per warp). Lane l
// owns chunk l of every replication, but instead of each lane jumping its stream ahead
// (lane_jump: ~24 table reads per lane per replication), replication r enters at lane 0
// and moves one lane per step: at step t lane l runs its chunk of the replication that
// entered at step t - l, starting from the stream state lane l-1 ended with (chunk l-1
// ends exactly where chunk l begins), and passes (state, partial sum, index) up with
// __shfl_up_sync. The last lane completes a replication every step; finished sums collect
// in shared memory and 32 of them are finalised and stored by the 32 lanes at once.
//
// * Rotating schedule (PipeSched): every lane runs L(t) units at step t, and any S
//   consecutive L sum to n, so no lane idles behind a longer chunk.
// * S lanes per replication: S = 32 is the whole warp; S = 16 or 8 runs 32/S such
//   pipelines side by side in the warp (every replication still passes through lanes of
//   one warp only, split into S chunks), so a step carries 32/S times the units per
//   lane for the same hand-over and bookkeeping instructions (config 4, 1,000 points:
//   31 units per step at S = 32, 125 at S = 8).
// * Wrap (WRAP): a straight pipeline idles a triangle of (S-1) x S lane-steps per
//   pipeline (lanes p > t while it fills, lanes p < s while it drains). Each S-lane
//   pipeline owns S - 1 "wrap" replications besides the ones its warp grabs: at step 0
//   its lane p >= 1 starts wrap replication p at chunk p (the seed jumped by the units of
//   chunks 0..p-1: one lane-table jump per lane and warp), and these late chunks fill the
//   fill triangle; once the grabbed replications run out, its lane 0 is fed the wrap
//   replications S-1, .., 1, whose early chunks 0..k-1 fill the drain triangle exactly
//   and all end at the pipeline's last step. Late and early partial sums are integers,
//   added exactly. A pipeline fed N grabbed replications runs N + S - 1 steps for
//   N + S - 1 replications.
// WIDE: 64-bit sums and indices (n >= 2^27 or count >= 2^31); else 32-bit, fewer shuffles.
__device__ __forceinline__ Taus lane_jump_g(const uint32_t* __restrict__ tab, int lane, Taus t) {
    t.s1 = nib_apply_g32(tab + lane, t.s1);
    t.s2 = nib_apply_g32(tab + 4096 + lane, t.s2);
    t.s3 = nib_apply_g32(tab + 8192 + lane, t.s3);
    return t;
}

#ifndef WLP_PIPE_MINB
#define WLP_PIPE_MINB 3
#endif
// The pipeline's bookkeeping lives in shared memory (volatile: re-read each step), so
// none of it is live across the unit loop; the loop then runs in 32 registers and the
// kernel fits 4 blocks (64 warps) per SM like the thread-per-replication kernel.
struct PipeCtl {
    long long cur, cend;  // the warp's current group of replications
    int more;             // the warp still grabs
    int nemit;            // finished replications waiting in the result buffer
    int drain[16];        // per pipeline: takes no more grabbed replications
    int wraps[16];        // per pipeline: wrap replications still to feed
};

template <int MODEL, bool WIDE, int S, bool WRAP>
__global__ void __launch_bounds__(kWlpBlock, WLP_PIPE_MINB) k_wlp_pipe(RepArgs a, PipeSched ps,
                                                           const uint32_t* __restrict__ wtab) {
    static_assert(S == 32 || WRAP, "S < 32 pipelines always wrap");
    pdl_wait();
    using I = typename std::conditional<WIDE, long long, int>::type;
    constexpr int kW = kWlpBlock / 32, P = 32 / S, kWr = S - 1;
    __shared__ I emit_rep[kW][32];
    __shared__ I emit_sum[kW][32];
    __shared__ I late_sum[kW][32];
    __shared__ PipeCtl ctl[kW];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane / S, pos = lane % S;  // pipeline of the lane, stage in it
    volatile PipeCtl& C = ctl[wid];
    // wrap replication k (1..S-1) of pipeline g: wrap_first() + k - 1
    auto wrap_first = [&]() {
        return (static_cast<int64_t>(blockIdx.x) * kW + wid) * (P * kWr) + g * kWr;
    };
    // item codes: r >= 0 a grabbed replication, -1 idle, -1-k the late chunks of wrap k,
    // -33-k its early chunks
    Taus st{kMin1, kMin2, kMin3};
    I sum = 0, rep = -1, left = 0;
    if (WRAP && pos > 0) {
        st = lane_jump_g(wtab, lane, load_seed(a, wrap_first() + pos - 1));
        rep = static_cast<I>(-1 - pos);
    }
    if (lane == 0) {
        C.cur = 0;
        C.cend = 0;
        C.more = 1;
        C.nemit = 0;
    }
    if (pos == 0) {
        C.drain[g] = 0;
        C.wraps[g] = kWr;
    }
    __syncwarp();
    int phase = 0;
    auto value = [&](I c) {  // pi: hits; walk: the raw q sum, dx = (sum + 6n) / 6
        return MODEL == 0 ? __ddiv_rn(__dmul_rn(4.0, static_cast<double>(c)), static_cast<double>(a.n))
                          : walk_fold((static_cast<int64_t>(c) + 6 * a.n) / 6, a.chunks);
    };
    auto flush = [&](int cnt) {
        __syncwarp();
        if (lane < cnt) put1(a, emit_rep[wid][lane], value(emit_sum[wid][lane]));
        __syncwarp();
    };
    for (;;) {
        int64_t cur = C.cur, cend = C.cend;
        bool more = C.more != 0, drain = C.drain[g] != 0;
        int wraps = C.wraps[g];
        if (more && cur >= cend) {  // next group (a multiple of P replications)
            const int64_t base = (WRAP ? static_cast<int64_t>(gridDim.x) * kW * (P * kWr) : 0) +
                                 grab_take(grab_issue(a, lane));
            if (base >= a.count) {
                more = false;
            } else {
                cur = base;
                cend = base + a.grab < a.count ? base + a.grab : a.count;
            }
        }
        bool last = false;  // this lane's pipeline runs its last step
        if (!drain) {
            const int64_t r = cur + g;
            if (more && r < cend) {  // feed a grabbed replication
                if (pos == 0) {
                    rep = static_cast<I>(r);
                    st = load_seed(a, r);
                    sum = 0;
                }
            } else {
                drain = true;
            }
        }
        if (more) cur += P;
        if (drain) {
            if (WRAP && wraps > 0) {  // the early chunks of wrap replication `wraps`
                if (pos == 0) {
                    rep = static_cast<I>(-33 - wraps);
                    st = load_seed(a, wrap_first() + wraps - 1);
                    sum = 0;
                    left = static_cast<I>(pipe_wrap_units(ps, wraps));
                }
                last = wraps == 1;
                --wraps;
            } else if (!WRAP) {
                if (pos == 0) rep = -1;
            } else {
                rep = -1;  // finished pipeline
            }
        }
        __syncwarp();
        if (lane == 0) {
            C.cur = cur;
            C.cend = cend;
            C.more = more ? 1 : 0;
        }
        if (pos == 0) {
            C.drain[g] = drain ? 1 : 0;
            C.wraps[g] = wraps;
        }
        if (!more && !__any_sync(kFull, rep != -1)) break;
        uint32_t units = static_cast<uint32_t>(pipe_units(ps, phase));
        if (WRAP && rep <= -34) {  // early chunk pos of wrap k: stop exactly at its late part
            const I k = -33 - rep;
            const I u = pos == k - 1 ? left : (left < static_cast<I>(units) ? left : static_cast<I>(units));
            left -= u;
            units = static_cast<uint32_t>(u);
        }
        if (rep != -1) sum += MODEL == 0 ? static_cast<I>(pi_hits(st, units)) : static_cast<I>(walk_q(st, units));
        int nemit = C.nemit;
        if (S == 32) {
            const I r31 = __shfl_sync(kFull, rep, 31);
            if (r31 >= 0) {  // lane 31 finished a replication
                if (lane == 31) {
                    emit_rep[wid][nemit] = rep;
                    emit_sum[wid][nemit] = sum;
                }
                if (++nemit == 32) {
                    flush(32);
                    nemit = 0;
                }
            } else if (WRAP && r31 < -1 && lane == 31) {  // the late chunks of a wrap replication
                late_sum[wid][-1 - r31] = sum;
            }
        } else {
            const bool fin = pos == S - 1 && rep >= 0;
            const unsigned m = __ballot_sync(kFull, fin);
            if (fin) {
                const int slot = nemit + __popc(m & ((1u << lane) - 1u));
                emit_rep[wid][slot] = rep;
                emit_sum[wid][slot] = sum;
            } else if (pos == S - 1 && rep < -1 && rep >= -32) {
                late_sum[wid][g * S - 1 - static_cast<int>(rep)] = sum;
            }
            nemit += __popc(m);
            if (nemit > 32 - P) {
                flush(nemit);
                nemit = 0;
            }
        }
        __syncwarp();
        if (lane == 0) C.nemit = nemit;
        if (WRAP && __any_sync(kFull, last)) {  // early chunks of wraps 1..S-1 end here
            __syncwarp();
            if (last && pos < S - 1) put1(a, wrap_first() + pos, value(sum + late_sum[wid][g * S + pos + 1]));
            if (last) rep = -1;
            if (S == 32) break;
        }
        st.s1 = __shfl_up_sync(kFull, st.s1, 1, S);
        st.s2 = __shfl_up_sync(kFull, st.s2, 1, S);
        st.s3 = __shfl_up_sync(kFull, st.s3, 1, S);
        sum = __shfl_up_sync(kFull, sum, 1, S);
        rep = __shfl_up_sync(kFull, rep, 1, S);
        if (WRAP) left = __shfl_up_sync(kFull, left, 1, S);
        phase = phase == S - 1 ? 0 : phase + 1;
        __syncwarp();
    }
    __syncwarp();
    flush(C.nemit);
}

// mm1 WLP shared memory: lane-start tables, panel-skip table, log table, then per warp
// the panel's per-client terms of the three ordered sums and the near-one compaction list.
constexpr int kMm1P = 32 * kMm1PanelT;
constexpr int kMm1Seg = kMm1PanelT + 2;  // lane segment stride (doubles): STS.128 rows spread over banks
constexpr int kMm1Arr = 32 * kMm1Seg + 2;  // array stride: the three sum lanes read different banks
struct Mm1Warp {
    // [k][l*kMm1Seg + c] = term k of client l*T + c of the panel: k = 0 w (-> sumw),
    // 1 w + s (-> sums), 2 the idle increment -t or +0 (-> idle). Also the near-one
    // scratch of the exponential batches before the terms are written.
    double term[3 * kMm1Arr];
    NearList nl;
};
static_assert(kMm1Arr >= 32 * kExpoB, "near-one results alias the term arrays");
constexpr size_t kMm1Smem = kUniTabWords * 4 + 256 * 8 + (kMm1Block / 32) * sizeof(Mm1Warp);

// One client of the Lindley recursion, models.hpp:67-78 in the reference's rounding:
// t = (w + s_prev) - a with u = fl(w + s_prev) carried from the previous client (it is
// the previous client's sums term, the same fl(w + s)); w = t < 0 ? 0 : t; u = fl(w + s).
// * The branch is w = t < 0 ? +0 : t. t is never -0 or NaN here (u >= +0, a finite), so
//   clearing both words when the sign bit is set is the same; it is two integer ops
//   (DMNMX / DSETP would put 8-25 cycles of FP64 latency on the recursion's chain).
// * d is the idle increment, d = fl(w - t): -t when dry, +0 otherwise, exactly. idle - t
//   == idle + (-t), and idle + (+0) == idle (idle >= +0), so the reference's conditional
//   `idle = idle - t` becomes a plain ordered sum of d like the other two.
__device__ __forceinline__ void lindley(double& w, double& u, double a, double s, double& d) {
    const double t = __dsub_rn(u, a);
    const int hi = __double2hiint(t), keep = ~(hi >> 31);
    w = __hiloint2double(hi & keep, __double2loint(t) & keep);
    d = __dsub_rn(w, t);
    u = __dadd_rn(w, s);
}

// mm1, one replication per warp. Panel p covers clients [p*32T, (p+1)*32T); lane l owns
// clients p*32T + l*T + c (c < T), drawn from draws 2*(that index) and 2*(...)+1, so each
// lane steps its own contiguous draw range and hops 62T draws between panels.
//
// Per panel: (1) lanes compute their clients' exponentials (a, s). (2) The Lindley
// recursion is chained across the 32 lane segments. Round 1: every lane runs its segment
// from an input waiting time (lane 0 the true carry, the others 0) and stores its clients'
// sum terms. Then, while some lane's input (its predecessor's segment end) changed, those
// lanes re-run from the new input, storing terms, until their waiting time is 0: there
// the new trajectory has met the old one (the recursion is monotone in w and inputs only
// grow from round to round, so new w = 0 forces old w = 0) and everything after is
// unchanged; a lane that never meets it passes a new end on. Lane 0 is exact in round 1
// and lane l by round l+1, so the fixed point is the sequential trajectory bit for bit;
// at rho = 1/2 the server runs dry at about every other arrival, so the re-runs are
// short. (3) Lanes 0-2 run the three ordered sums over the panel's terms: sumw, sums and
// idle are order-dependent fp64 and stay sequential, one lane each, in one instruction.
template <int DIV>
__device__ __forceinline__ double mm1_warp_rep(Taus st, int64_t n, double lambda, double mu, double inv_l,
                                               double inv_m, const double* logtab, const uint32_t* skip, Mm1Warp& W,
                                               int lane, unsigned* ev = nullptr) {
    constexpr int T = kMm1PanelT;
    constexpr int P = kMm1P;
    static_assert(2 * T % kExpoB == 0 && T % 2 == 0, "panel draws per lane must be whole batches");
    double wc = 0.0, sc = 0.0;  // carry (warp-uniform): w and s of the panel's predecessor client
    double acc = 0.0;           // lane k < 3: ordered sum of term k
    double* const term = W.term + lane * kMm1Seg;
    for (int64_t base = 0; base < n; base += P) {
        double ea[T], es[T];
#pragma unroll
        for (int h = 0; h < 2 * T; h += kExpoB) {
            uint32_t d[kExpoB];
            double e[kExpoB];
#pragma unroll
            for (int j = 0; j < kExpoB; j += 2) taus_next2(st, d[j], d[j + 1]);
            neg_log1m_batch<kExpoB, true>(d, e, logtab, W.nl, W.term, kFull, lane, ev);
#pragma unroll
            for (int j = 0; j < kExpoB; j += 2) {
                ea[(h + j) / 2] = scale<DIV>(e[j], lambda, inv_l);
                es[(h + j) / 2] = scale<DIV>(e[j + 1], mu, inv_m);
            }
        }
        const int64_t left = n - base;
        const bool has = left > static_cast<int64_t>(lane) * T;  // my segment holds clients
        double sp = __shfl_up_sync(kFull, es[T - 1], 1);       // s of my segment's predecessor
        if (lane == 0) sp = sc;
        double in = lane == 0 ? wc : 0.0;
        double end;
        {  // round 1: the whole segment (clients past n are computed too, never summed)
            double w = in, u = __dadd_rn(in, sp);
#pragma unroll
            for (int c = 0; c < T; c += 2) {
                double w0, d0, w1, d1;
                lindley(w0, u, ea[c], es[c], d0);
                const double u0 = u;
                lindley(w1, u, ea[c + 1], es[c + 1], d1);
                *reinterpret_cast<double2*>(term + c) = make_double2(w0, w1);
                *reinterpret_cast<double2*>(term + kMm1Arr + c) = make_double2(u0, u);
                *reinterpret_cast<double2*>(term + 2 * kMm1Arr + c) = make_double2(d0, d1);
                w = w1;
            }
            end = w;
        }
        for (;;) {  // ripple rounds (warp-uniform loop)
            double nin = __shfl_up_sync(kFull, end, 1);
            if (lane == 0) nin = wc;
            bool run = has && __double_as_longlong(nin) != __double_as_longlong(in);
            if (!__any_sync(kFull, run)) break;
            if (run) in = nin;
            double w = in, u = __dadd_rn(in, sp);
#pragma unroll
            for (int c = 0; c < T; ++c) {
                if (c % 2 == 0 && !__any_sync(kFull, run)) break;  // (checked every other client)
                if (run) {
                    double d;
                    lindley(w, u, ea[c], es[c], d);
                    term[c] = w;
                    term[kMm1Arr + c] = u;
                    term[2 * kMm1Arr + c] = d;
                    run = (__double2hiint(w) | __double2loint(w)) != 0;  // w == +0: met the old trajectory
                    if (c == T - 1 && run) end = w;
                }
            }
        }
        wc = __shfl_sync(kFull, end, 31);
        sc = __shfl_sync(kFull, es[T - 1], 31);
        __syncwarp();
        if (lane < 3) {  // the ordered sums, one lane per sum
            const double* x = W.term + lane * kMm1Arr;
            const int cnt = left >= P ? P : static_cast<int>(left);
            const int nseg = cnt / T;
            // segment loads run one segment ahead of the adds (the last prefetch reads past
            // the array into the next one or the near-one list: in bounds, unused)
            double2 v[T / 2];
#pragma unroll
            for (int j = 0; j < T / 2; ++j) v[j] = reinterpret_cast<const double2*>(x)[j];
            for (int seg = 0; seg < nseg; ++seg) {
                x += kMm1Seg;
                double2 nv[T / 2];
#pragma unroll
                for (int j = 0; j < T / 2; ++j) nv[j] = reinterpret_cast<const double2*>(x)[j];
#pragma unroll
                for (int j = 0; j < T / 2; ++j) {
                    acc = __dadd_rn(acc, v[j].x);
                    acc = __dadd_rn(acc, v[j].y);
                }
#pragma unroll
                for (int j = 0; j < T / 2; ++j) v[j] = nv[j];
            }
            for (int c = 0; c < cnt - nseg * T; ++c) acc = __dadd_rn(acc, x[c]);
        }
        __syncwarp();
        st = uni_jump(skip, st);
    }
    return acc;
}

// Heavy traffic: the segment chain barely regenerates, ripple rounds go one lane at a
// time, and the separate sum phase adds its own chain. Then lane 0 runs the recursion and
// the three sums of the panel in one ordered loop (the four chains overlap), reading the
// client-ordered (a, s) pairs the lanes staged in shared memory. Same result bits;
// returns the same per-lane layout as mm1_warp_rep (lanes 0/1/2: sumw/sums/idle).
template <int DIV>
__device__ __forceinline__ double mm1_warp_rep_serial(Taus st, int64_t n, double lambda, double mu, double inv_l,
                                                      double inv_m, const double* logtab, const uint32_t* skip,
                                                      Mm1Warp& W, int lane, unsigned* ev = nullptr) {
    constexpr int T = kMm1PanelT;
    constexpr int P = kMm1P;
    static_assert(sizeof(double2) * 32 * (T + 1) <= sizeof(W.term), "pair panel fits the term arrays");
    double2* const pair = reinterpret_cast<double2*>(W.term);
    Queue q;
    for (int64_t base = 0; base < n; base += P) {
        double ea[T], es[T];
#pragma unroll
        for (int h = 0; h < 2 * T; h += kExpoB) {
            uint32_t d[kExpoB];
            double e[kExpoB];
#pragma unroll
            for (int j = 0; j < kExpoB; j += 2) taus_next2(st, d[j], d[j + 1]);
            neg_log1m_batch<kExpoB, true>(d, e, logtab, W.nl, W.term, kFull, lane, ev);
#pragma unroll
            for (int j = 0; j < kExpoB; j += 2) {
                ea[(h + j) / 2] = scale<DIV>(e[j], lambda, inv_l);
                es[(h + j) / 2] = scale<DIV>(e[j + 1], mu, inv_m);
            }
        }
#pragma unroll
        for (int c = 0; c < T; ++c) pair[lane * (T + 1) + c] = make_double2(ea[c], es[c]);
        __syncwarp();
        if (lane == 0) {
            const int64_t left = n - base;
            if (left >= P) {
                const double2* p = pair;
                for (int seg = 0; seg < 32; ++seg, p += T + 1) {
                    double2 v[T];
#pragma unroll
                    for (int j = 0; j < T; ++j) v[j] = p[j];
#pragma unroll
                    for (int j = 0; j < T; ++j) q.client(v[j].x, v[j].y);
                }
            } else {
                for (int c = 0; c < static_cast<int>(left); ++c) {
                    const double2 v = pair[(c / T) * (T + 1) + c % T];
                    q.client(v.x, v.y);
                }
            }
        }
        __syncwarp();
        st = uni_jump(skip, st);
    }
    const double sumw = __shfl_sync(kFull, q.sumw, 0), sums = __shfl_sync(kFull, q.sums, 0),
                 idle = __shfl_sync(kFull, q.idle, 0);
    return lane == 0 ? sumw : (lane == 1 ? sums : idle);
}

// The lane-start tables stay in global memory (L1/L2 resident): one 24-load jump per
// replication of ~10^3 clients is noise, and the 48 KB are better spent on term arrays.
struct Mm1Smem {
    const uint32_t* tab;
    uint32_t* skip;
    double* logtab;
    Mm1Warp* W;
};

__device__ __forceinline__ Mm1Smem mm1_stage(const uint32_t* gtab, const uint32_t* gskip) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Mm1Smem m;
    m.tab = gtab;
    m.skip = reinterpret_cast<uint32_t*>(smraw);
    m.logtab = reinterpret_cast<double*>(m.skip + kUniTabWords);
    m.W = reinterpret_cast<Mm1Warp*>(m.logtab + 256) + (threadIdx.x >> 5);
    for (int i = threadIdx.x; i < kUniTabWords; i += blockDim.x) m.skip[i] = __ldg(gskip + i);
    stage_log_table(m.logtab);
    __syncthreads();
    return m;
}

template <int DIV, bool COUNT>
__global__ void __launch_bounds__(kMm1Block, 3) k_wlp_mm1(RepArgs a, const uint32_t* __restrict__ gtab,
                                                        const uint32_t* __restrict__ gskip) {
    const Mm1Smem m = mm1_stage(gtab, gskip);
    pdl_wait();
    const int lane = threadIdx.x & 31;
    // the `t < 0` decision is a per-lane select, never a warp branch; the warp splits in
    // the near-one loops of the exponential batches (counted there)
    HwTally hw;
    if (COUNT) {
        hw.t0 = hw_clock();
        hw.ld = staged_loads(kUniTabWords) + staged_loads(256);
    }
    unsigned* const ev = COUNT ? &hw.splits : nullptr;
    for (int64_t base = grab_take(grab_issue(a, lane)); base < a.count;) {
        const unsigned long long ticket = grab_issue(a, lane);
        const int64_t end = base + a.grab < a.count ? base + a.grab : a.count;
        double k0 = 0.0, k1 = 0.0, k2 = 0.0;
        for (int64_t r = base; r < end; ++r) {
            const Taus st = lane_jump(m.tab, lane, load_seed(a, r));
            const double acc =
                a.lambda >= a.serial_rho * a.mu
                    ? mm1_warp_rep_serial<DIV>(st, a.n, a.lambda, a.mu, a.inv_lambda, a.inv_mu, m.logtab, m.skip,
                                               *m.W, lane, ev)
                    : mm1_warp_rep<DIV>(st, a.n, a.lambda, a.mu, a.inv_lambda, a.inv_mu, m.logtab, m.skip, *m.W, lane,
                                        ev);
            const double avg = __ddiv_rn(acc, static_cast<double>(a.n));  // lanes 0/1/2: wait/sys/idle
            const double v0 = __shfl_sync(kFull, avg, 2);
            const double v1 = __shfl_sync(kFull, avg, 0);
            const double v2 = __shfl_sync(kFull, avg, 1);
            if (lane == static_cast<int>(r - base)) {
                k0 = v0;
                k1 = v1;
                k2 = v2;
            }
        }
        if (lane < end - base) {
            put3(a, base + lane, k0, k1, k2);
        }
        if (COUNT) {
            hw.ld += (3 + 24) * static_cast<unsigned>(end - base);  // seed words, lane-jump table reads
            hw.st += 3;
        }
        base = grab_take(ticket);
    }
    if (COUNT) flush_tally(hw, a.hw);
}

// ---------------------------------------------------------------------------------
// TLP: one replication per thread (the comparison mapping)
// ---------------------------------------------------------------------------------

__device__ __forceinline__ double pi_rep_tlp(Taus st, int64_t n) {
    // c counts exactly (the reference accumulates 0.0/1.0 in a double, exact < 2^53)
    uint64_t c = 0;
    for (int64_t done = 0; done < n;) {
        const int64_t left = n - done;
        const uint32_t part = left > 0x40000000 ? 0x40000000u : static_cast<uint32_t>(left);
        c += pi_hits(st, part);
        done += part;
    }
    return __ddiv_rn(__dmul_rn(4.0, static_cast<double>(c)), static_cast<double>(n));
}

// models.hpp:92-105 as written: a 4-way branch per step on d = floor(4u).
__device__ __forceinline__ double walk_rep_tlp(Taus st, int64_t n, int64_t chunks) {
    double px = 0.0, py = 0.0;
    for (int64_t i = 0; i < n; ++i) {
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
    return walk_fold(static_cast<int64_t>(px), chunks);
}

// One warp-level `if` of the reference's event definition (warp_exec.cpp:272-284): with
// active lanes `act`, the branch diverges when some take it and some do not. Returns the
// lanes that did not take it (the else side's active mask).
__device__ __forceinline__ unsigned split_if(unsigned act, bool cond, unsigned& events, unsigned sync = 0u) {
    const unsigned taken = __ballot_sync(sync ? sync : act, cond) & act;
    if (taken != 0u && taken != act) ++events;
    return act & ~taken;
}

// The walk with its 4-way branch (models.cpp:216-253 nests three ifs) and event counting.
__device__ __forceinline__ double walk_rep_tlp_counted(Taus st, int64_t n, int64_t chunks, unsigned& events) {
    const unsigned act = __activemask();
    double px = 0.0, py = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        const uint32_t d = taus_next(st) >> 30;
        (void)taus_next(st);
        const unsigned a1 = split_if(act, d == 0u, events);
        const unsigned a2 = a1 ? split_if(a1, d == 1u, events) : 0u;
        if (a2) split_if(a2, d == 2u, events);
        if (d == 0u)
            px = __dadd_rn(px, 1.0);
        else if (d == 1u)
            px = __dsub_rn(px, 1.0);
        else if (d == 2u)
            py = __dadd_rn(py, 1.0);
        else
            py = __dsub_rn(py, 1.0);
    }
    return walk_fold(static_cast<int64_t>(px), chunks);
}

template <int MODEL, bool COUNT>
__global__ void k_tlp(RepArgs a) {
    pdl_wait();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.count) return;  // tail threads of the last block stay inert (wlp.cpp:125-138)
    const Taus st = load_seed(a, r);
    HwTally hw;
    if (COUNT) hw.t0 = hw_clock();
    if (MODEL == 0) {
        put1(a, r, pi_rep_tlp(st, a.n));  // no data-dependent branch: no events
    } else if (COUNT) {
        put1(a, r, walk_rep_tlp_counted(st, a.n, a.chunks, hw.div));
    } else {
        put1(a, r, walk_rep_tlp(st, a.n, a.chunks));
    }
    if (COUNT) {
        hw.ld = 3;  // the seed words
        hw.st = 1;
        flush_tally(hw, a.hw);
    }
}

// ---------------------------------------------------------------------------------
// Walk, bitsliced thread per 32 replications (TLP variant; bitslice.cuh). Thread t owns
// replications 32t .. 32t+31: their seeds are transposed into bit planes, every step
// costs ~33 XORs per draw for all 32, and the +x / -x step masks are counted per stream
// by a Harley-Seal carry-save tree (16 steps per tree, weight-16 carries rippled into
// the higher digits). Counts stay exact below 2^16; longer walks flush every 65520 steps
// into per-stream int32 sums in shared memory. Same draws, same d, same dx as
// walk_replication: the outputs are the reference's bit for bit.
// ---------------------------------------------------------------------------------
constexpr int kBsBlock = 128;
constexpr int64_t kBsFlushBlocks = 4095;  // 4095 * 16 steps keep every count below 2^16

// Thread t of the block gets its group's 32 seeds (replications 32(g0 + t) ..) of
// component `comp` in w[]: the block reads its 32 * blockDim consecutive words coalesced
// into shared memory (rows padded to 33 words: conflict-free both ways) and each thread
// takes its row. Past the end: the component's minimum (a valid state). Every thread of
// the block must call it.
__device__ __forceinline__ void bs_load_component(const RepArgs& a, int comp, int64_t g0, uint32_t* sm,
                                                  uint32_t (&w)[32]) {
    const uint32_t fill = comp == 0 ? kMin1 : (comp == 1 ? kMin2 : kMin3);
    const uint32_t* src = a.seeds + comp * a.count;
    const int64_t r0 = g0 * 32;
    for (int k = threadIdx.x; k < 32 * static_cast<int>(blockDim.x); k += blockDim.x) {
        const int64_t r = r0 + k;
        sm[(k >> 5) * 33 + (k & 31)] = r < a.count ? __ldg(src + r) : fill;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 32; ++j) w[j] = sm[threadIdx.x * 33 + j];
    __syncthreads();
}


// Steps k of a 16-step block count only while k < valid (MASK; the masks fold into the
// LOP3s that form them). Without MASK every step counts.
template <bool MASK>
__device__ __forceinline__ void bs_step_m(BsTaus& t, uint32_t& pl, uint32_t& mi, int k, int valid) {
    bs_walk_step(t, pl, mi);
    if (MASK) {
        const uint32_t keep = k < valid ? ~0u : 0u;
        pl &= keep;
        mi &= keep;
    }
}

template <bool MASK>
__device__ __forceinline__ void bs_pair(BsTaus& t, BsCount& P, BsCount& Q, uint32_t& p2, uint32_t& q2, int k,
                                        int valid) {
    uint32_t pa, ma, pb, mb;
    bs_step_m<MASK>(t, pa, ma, k, valid);
    bs_step_m<MASK>(t, pb, mb, k + 1, valid);
    bs_csa(p2, P.c[0], P.c[0], pa, pb);
    bs_csa(q2, Q.c[0], Q.c[0], ma, mb);
}

template <bool MASK>
__device__ __forceinline__ void bs_quad(BsTaus& t, BsCount& P, BsCount& Q, uint32_t& p4, uint32_t& q4, int k,
                                        int valid) {
    uint32_t pa, qa, pb, qb;
    bs_pair<MASK>(t, P, Q, pa, qa, k, valid);
    bs_pair<MASK>(t, P, Q, pb, qb, k + 2, valid);
    bs_csa(p4, P.c[1], P.c[1], pa, pb);
    bs_csa(q4, Q.c[1], Q.c[1], qa, qb);
}

template <bool MASK>
__device__ __forceinline__ void bs_oct(BsTaus& t, BsCount& P, BsCount& Q, uint32_t& p8, uint32_t& q8, int k,
                                       int valid) {
    uint32_t pa, qa, pb, qb;
    bs_quad<MASK>(t, P, Q, pa, qa, k, valid);
    bs_quad<MASK>(t, P, Q, pb, qb, k + 4, valid);
    bs_csa(p8, P.c[2], P.c[2], pa, pb);
    bs_csa(q8, Q.c[2], Q.c[2], qa, qb);
}

__device__ __forceinline__ void bs_ripple16(BsCount& k, uint32_t m) {  // add m at weight 16
#pragma unroll
    for (int w = 4; w < 16; ++w) {
        const uint32_t carry = k.c[w] & m;
        k.c[w] ^= m;
        m = carry;
    }
}

__global__ void __launch_bounds__(kBsBlock) k_tlp_walk_bs(RepArgs a) {
    extern __shared__ int32_t bs_acc[];  // [kBsBlock][33] when n > 65520 steps
    const int64_t r0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 32;
    if (r0 >= a.count) return;
    pdl_wait();
    // (direct loads: staging them through shared memory as k_bs_seeds does measured
    // 0.899 vs 0.884 ms here, where the seeds are read once per 1,000 steps)
    BsTaus t;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const Taus st = r0 + j < a.count ? load_seed(a, r0 + j) : Taus{kMin1, kMin2, kMin3};
        t.b1[j] = st.s1;
        t.b2[j] = st.s2;
        t.b3[j] = st.s3;
    }
    transpose32(t.b1);
    transpose32(t.b2);
    transpose32(t.b3);
    BsCount P, Q;
    bs_count_init(P);
    bs_count_init(Q);
    const bool flushing = a.n > kBsFlushBlocks * 16;
    int32_t* acc = bs_acc + threadIdx.x * 33;
    if (flushing)
        for (int j = 0; j < 32; ++j) acc[j] = 0;
    auto flush = [&]() {
        int32_t d[32];
        bs_count_diff(P, Q, d);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] += d[j];
        bs_count_init(P);
        bs_count_init(Q);
    };
    const int64_t blocks = a.n / 16;
    for (int64_t b = 0; b < blocks; ++b) {
        uint32_t pa, qa, pb, qb, p16, q16;
        bs_oct<false>(t, P, Q, pa, qa, 0, 16);
        bs_oct<false>(t, P, Q, pb, qb, 8, 16);
        bs_csa(p16, P.c[3], P.c[3], pa, pb);
        bs_csa(q16, Q.c[3], Q.c[3], qa, qb);
        bs_ripple16(P, p16);
        bs_ripple16(Q, q16);
        if (flushing && (b + 1) % kBsFlushBlocks == 0) flush();
    }
    for (int64_t s = blocks * 16; s < a.n; ++s) {
        uint32_t pl, mi;
        bs_walk_step(t, pl, mi);
        bs_count_add1(P, pl);
        bs_count_add1(Q, mi);
    }
    int32_t d[32];
    bs_count_diff(P, Q, d);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        if (r0 + j >= a.count) break;
        const int64_t dx = static_cast<int64_t>(d[j]) + (flushing ? acc[j] : 0);
        put1(a, r0 + j, walk_fold(dx, a.chunks));
    }
}

// ---------------------------------------------------------------------------------
// Walk WLP, bitsliced warp pipeline. The warp pipeline of k_wlp_pipe (a replication
// enters at lane 0, lane l runs steps [l*K, (l+1)*K) of it from the state lane l-1 hands
// over, lane 31 completes one every pipeline step) with 32 replications per slot held as
// bit planes (bitslice.cuh): each lane advances a group of 32 replications, so a warp
// still owns every replication it runs and its lanes split each one's steps. Per step a
// lane hands over 88 live state words and the 32 counter digits. Group seeds are
// transposed once by k_bs_seeds; lane 31's finished counters collect in shared memory and
// 32 groups are finalised at once (one per lane). Counts must stay below 2^16 (n < 65536).
// ---------------------------------------------------------------------------------

__global__ void __launch_bounds__(kBsBlock) k_bs_seeds(RepArgs a, int64_t groups, uint32_t* __restrict__ out) {
    __shared__ uint32_t stage[kBsBlock * 33];
    pdl_wait();
    const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    BsTaus t;
    const int64_t g0 = static_cast<int64_t>(blockIdx.x) * blockDim.x;
    bs_load_component(a, 0, g0, stage, t.b1);
    bs_load_component(a, 1, g0, stage, t.b2);
    bs_load_component(a, 2, g0, stage, t.b3);
    if (g >= groups) return;
    bs_store_planes(t, out + g * kBsLive);
}

// A lane's chunk of its group: `blocks` 16-step carry-save blocks for every lane of the
// warp alike (no lane runs a tail the others wait for); steps past the lane's `units`
// do not count. Only a group's last chunk is partial (the lane chunk is a multiple of
// 16), and the state it ends with is never used. (The bitsliced lane-chunk kernel.)
__device__ __forceinline__ void bs_walk_units(BsTaus& t, BsCount& P, BsCount& Q, uint32_t units, uint32_t blocks) {
    for (uint32_t b = 0; b < blocks; ++b) {
        const int valid = static_cast<int>(units > 16 * b ? (units - 16 * b < 16 ? units - 16 * b : 16) : 0);
        uint32_t pa, qa, pb, qb, p16, q16;
        bs_oct<true>(t, P, Q, pa, qa, 0, valid);
        bs_oct<true>(t, P, Q, pb, qb, 8, valid);
        bs_csa(p16, P.c[3], P.c[3], pa, pb);
        bs_csa(q16, Q.c[3], Q.c[3], qa, qb);
        bs_ripple16(P, p16);
        bs_ripple16(Q, q16);
    }
}

// Adds mask m at weight 2^W0 (a carry out of the carry-save tree's digit W0 - 1).
template <int W0>
__device__ __forceinline__ void bs_ripple_from(BsCount& k, uint32_t m) {
#pragma unroll
    for (int w = W0; w < 16; ++w) {
        const uint32_t carry = k.c[w] & m;
        k.c[w] ^= m;
        m = carry;
    }
}

// Exactly `units` walk steps of the 32 streams (the state ends exactly there): 16-step
// blocks, an 8-step sub-tree whose carry ripples in at weight 8, then single steps. The
// counters stay exact binary counts.
__device__ __forceinline__ void bs_walk_exact(BsTaus& t, BsCount& P, BsCount& Q, uint32_t units) {
    for (uint32_t b = units >> 4; b; --b) {
        uint32_t pa, qa, pb, qb, p16, q16;
        bs_oct<false>(t, P, Q, pa, qa, 0, 16);
        bs_oct<false>(t, P, Q, pb, qb, 8, 16);
        bs_csa(p16, P.c[3], P.c[3], pa, pb);
        bs_csa(q16, Q.c[3], Q.c[3], qa, qb);
        bs_ripple16(P, p16);
        bs_ripple16(Q, q16);
    }
    if (units & 8) {
        uint32_t p8, q8;
        bs_oct<false>(t, P, Q, p8, q8, 0, 16);
        bs_ripple_from<3>(P, p8);
        bs_ripple_from<3>(Q, q8);
    }
    for (uint32_t r = units & 7; r; --r) {  // (one copy of the step: the code stays in the I-cache)
        uint32_t pl, mi;
        bs_walk_step(t, pl, mi);
        bs_count_add1(P, pl);
        bs_count_add1(Q, mi);
    }
}

template <int P>
struct BsPipeWarp {
    uint32_t cnt[32][33];   // finished groups: P digits 0..15, Q digits 16..31 (+1 pad)
    long long grp[32];
    uint32_t late[32][33];  // wrap groups' late-chunk counters, by pipeline * S + wrap index
    __align__(16) uint32_t seed[2][P][kBsLive];  // the pipelines' next groups' bit planes, a step ahead
};

// cp.async of the next groups' 352-byte bit planes (22 pieces of 16 B per group) into
// shared memory: piece c of the warp's 22 * P goes to lane c % 32; gidx of pipeline j
// comes from its first lane.
template <int S>
__device__ __forceinline__ void bs_prefetch(uint32_t (*dst)[kBsLive], const uint32_t* __restrict__ bseeds,
                                            int64_t gidx, int lane) {
    constexpr int P = 32 / S, kPieces = kBsLive / 4;
#pragma unroll
    for (int c0 = 0; c0 < kPieces * P; c0 += 32) {
        const int c = c0 + lane, j = c / kPieces, k = c % kPieces;
        const int64_t gj = __shfl_sync(kFull, gidx, (j < P ? j : 0) * S);
        if (c < kPieces * P && gj >= 0) {
            const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst[j] + 4 * k));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(bseeds + gj * kBsLive + 4 * k)
                         : "memory");
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Per-stream dx of 32 streams from bitsliced counters (d[0..15] the +x digits P, d[16..31]
// the -x digits Q) plus, optionally, a second pair of counters d2 (the late chunks of a
// wrap group), written to out[0..31] (shared memory; out may alias d2, which is read
// first).
__device__ __forceinline__ void bs_dx_store(const uint32_t (&d)[32], const uint32_t* d2, int32_t* out) {
    // One transpose of both counters at once: row w < 16 holds P's digit w, row 16 + w Q's,
    // so column j comes out as stream j's P count in bits 0..15 and its Q count above
    // (half the transposes and the live registers of two separate ones).
    uint32_t v[32];
#pragma unroll
    for (int w = 0; w < 32; ++w) v[w] = d[w];
    transpose32(v);
    int32_t dx[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) dx[j] = static_cast<int32_t>(v[j] & 0xFFFFu) - static_cast<int32_t>(v[j] >> 16);
    if (d2) {
#pragma unroll
        for (int w = 0; w < 32; ++w) v[w] = d2[w];
        transpose32(v);
#pragma unroll
        for (int j = 0; j < 32; ++j) dx[j] += static_cast<int32_t>(v[j] & 0xFFFFu) - static_cast<int32_t>(v[j] >> 16);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) out[j] = dx[j];
}

// Walk WLP, bitsliced warp pipeline on the rotating schedule (PipeSched: L(t) steps per
// lane per pipeline step, any S consecutive L summing to n; bs_walk_exact advances the
// planes exactly, so chunks need not be whole 16-step blocks), S lanes per group of 32
// replications (32/S pipelines side by side in the warp: with S = 8 a step carries 125
// walk steps of 1,000 instead of 31, so the per-step hand-over of 120 words and the
// feed / emit bookkeeping cost a quarter as much), with the wrap of k_wlp_pipe: each
// pipeline owns S - 1 wrap groups besides the ones its warp grabs; at step 0 its lane p
// >= 1 starts wrap group p at its chunk p (the 32 seeds jumped by a lane table and
// transposed into planes), and after the grabbed groups its lane 0 is fed wrap groups
// S-1..1, whose early chunks end at the pipeline's last step; each wrap group's dx is the
// sum of its early and late counters. Feeding: the last lane of each pipeline, whose
// group has just been emitted, loads the next group's planes (prefetched into shared
// memory a step ahead by cp.async) and the hand-over rotates them to lane 0.
// (WRAP = false: straight pipelines, for runs too small to give every pipeline its wrap
// groups.)
#ifndef WLP_BS_MINB
#define WLP_BS_MINB 4  // 255 registers: no spills (6 blocks spilled ~700 B: 0.96 vs 0.92 ms at config 4)
#endif
template <int S, bool WRAP>
__global__ void __launch_bounds__(kBsPipeBlock, WLP_BS_MINB) k_wlp_walk_bs_pipe(RepArgs a, const uint32_t* __restrict__ bseeds,
                                                                    int64_t groups, PipeSched ps,
                                                                    const uint32_t* __restrict__ wtab) {
    constexpr int kW = kBsPipeBlock / 32, P = 32 / S, kWr = S - 1;
    __shared__ BsPipeWarp<P> sh[kW];
    BsPipeWarp<P>& E = sh[threadIdx.x >> 5];
    pdl_wait();
    const int lane = threadIdx.x & 31, g = lane / S, pos = lane % S;
    const int src = g * S + (pos + S - 1) % S;  // rotation within the pipeline: pos - 1, pos 0 <- pos S-1
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * kW + (threadIdx.x >> 5);
    const int64_t wrap0 = gwarp * (P * kWr) + g * kWr;  // wrap group k of this pipeline: wrap0 + k - 1
    const int64_t pool0 = WRAP ? static_cast<int64_t>(gridDim.x) * kW * (P * kWr) : 0;
    RepArgs ga = a;  // the grab scheduler hands out groups
    ga.count = groups;
    BsTaus t;
    BsCount Pc, Qc;
#pragma unroll
    for (int i = 0; i < 32; ++i) t.b1[i] = t.b2[i] = t.b3[i] = 0u;
    bs_count_init(Pc);
    bs_count_init(Qc);
    // item codes: g >= 0 a grabbed group, -1 idle, -1-k the late chunks of wrap group k,
    // -33-k its early chunks
    long long grp = -1;
    int left = 0;
    if (WRAP) {  // lane p >= 1: wrap group p's 32 seeds jumped to chunk p, as bit planes,
        // one component at a time through the lane's row of the (still unused) result
        // buffer, in loops that are not unrolled: the prologue stays small. The seeds come
        // from the group's bit planes (transposed back; the dead low bits read as 0 and
        // never reach a live bit), so the seeding writes no SoA keys for this kernel.
        const uint32_t* gpl = bseeds + (wrap0 + pos - 1) * kBsLive;
        uint32_t* row = E.cnt[lane];
#pragma unroll 1
        for (int comp = 0; comp < 3; ++comp) {
            if (pos > 0) {
                const int dead = comp == 0 ? 1 : (comp == 1 ? 3 : 4);  // rows below the live bits
                const int off = comp == 0 ? -1 : (comp == 1 ? 31 - 3 : 60 - 4);
                uint32_t k[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) k[i] = i < dead ? 0u : __ldg(gpl + off + i);
                transpose32(k);  // k[j]: stream j's component
#pragma unroll
                for (int j = 0; j < 32; ++j) row[j] = k[j];
                const uint32_t* tab = wtab + comp * 4096 + lane;
#pragma unroll 1
                for (int j = 0; j < 32; ++j) row[j] = nib_apply_g32(tab, row[j]);
            }
            __syncwarp();
            uint32_t w[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) w[j] = row[j];
            transpose32(w);
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (comp == 0) t.b1[i] = w[i];
                if (comp == 1) t.b2[i] = w[i];
                if (comp == 2) t.b3[i] = w[i];
            }
            __syncwarp();
        }
        if (pos > 0) {
            grp = -1 - pos;
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) t.b1[i] = t.b2[i] = t.b3[i] = 0u;
        }
    }
    int64_t cur = 0, cend = 0;
    bool more = true;   // the warp still grabs (warp-uniform)
    bool drain = false;  // this lane's pipeline takes no more grabbed groups
    bool fin = false;    // this lane's pipeline has run its last step
    int wraps = kWr, nemit = 0, phase = 0;
    // Stores group gg's 32 folded results from the dx row `row`: lane j writes element j,
    // so each store instruction covers 256 consecutive bytes (with a lane per group and 32
    // strided stores, the host-mirror writes over PCIe were 8-byte transactions).
    auto store_group = [&](long long gg, const uint32_t* row) {
        const int64_t r = gg * 32 + lane;
        if (r < a.count) put1(a, r, walk_fold(static_cast<int32_t>(row[lane]), a.chunks));
    };
    auto flush = [&](int cnt) {
        __syncwarp();
        if (lane < cnt) {
            uint32_t d[32];
#pragma unroll
            for (int w = 0; w < 32; ++w) d[w] = E.cnt[lane][w];
            bs_dx_store(d, nullptr, reinterpret_cast<int32_t*>(E.cnt[lane]));  // the slot's own row
        }
        __syncwarp();
        for (int sl = 0; sl < cnt; ++sl) store_group(E.grp[sl], E.cnt[sl]);
        __syncwarp();
    };
    // the item this lane's pipeline takes next (decided a step ahead, so its planes can
    // be prefetched): a grabbed group, then (WRAP) the early chunks of its wrap groups
    // S-1..1, then idle. The grab is warp-uniform; P groups per step.
    auto decide = [&](long long& code, int64_t& gidx) {
        if (more && cur >= cend) {
            const int64_t base = pool0 + grab_take(grab_issue(ga, lane));
            if (base >= groups) {
                more = false;
            } else {
                cur = base;
                cend = base + a.grab < groups ? base + a.grab : groups;
            }
        }
        code = gidx = -1;
        if (!drain) {
            const int64_t r = cur + g;
            if (more && r < cend)
                code = gidx = r;
            else
                drain = true;
        }
        if (drain && WRAP && wraps > 0) {
            code = -33 - wraps;
            gidx = wrap0 + wraps - 1;
            --wraps;
        }
        if (more) cur += P;
    };
    // lane `who` takes item (code, gidx) from the prefetch buffer, with fresh counters
    auto take = [&](bool who, long long code, int64_t gidx, const uint32_t* planes) {
        if (who) {
            grp = code;
            if (gidx >= 0) {
                const uint4* q = reinterpret_cast<const uint4*>(planes);
                uint32_t w[kBsLive];
#pragma unroll
                for (int k = 0; k < kBsLive / 4; ++k) {
                    const uint4 v = q[k];
                    w[4 * k] = v.x;
                    w[4 * k + 1] = v.y;
                    w[4 * k + 2] = v.z;
                    w[4 * k + 3] = v.w;
                }
#pragma unroll
                for (int i = 1; i < 32; ++i) t.b1[i] = w[i - 1];
#pragma unroll
                for (int i = 3; i < 32; ++i) t.b2[i] = w[31 + i - 3];
#pragma unroll
                for (int i = 4; i < 32; ++i) t.b3[i] = w[60 + i - 4];
                bs_count_init(Pc);
                bs_count_init(Qc);
                if (WRAP && code < -1) left = static_cast<int>(pipe_wrap_units(ps, static_cast<int>(-33 - code)));
            }
        }
    };
    long long feed, cur_feed;
    int64_t fidx;
    decide(feed, fidx);
    int buf = 0;
    bs_prefetch<S>(E.seed[buf], bseeds, fidx, lane);
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    take(pos == 0, feed, fidx, E.seed[buf][g]);  // step 0: the first lanes take their items directly
    cur_feed = feed;
    for (;;) {
        decide(feed, fidx);  // next step's items, prefetched while this step walks
        buf ^= 1;
        bs_prefetch<S>(E.seed[buf], bseeds, fidx, lane);
        uint32_t units = static_cast<uint32_t>(pipe_units(ps, phase));
        if (WRAP && grp <= -34) {  // early chunk `pos` of wrap group k: stop exactly at its late part
            const int k = static_cast<int>(-33 - grp);
            const int u = pos == k - 1 ? left : (left < static_cast<int>(units) ? left : static_cast<int>(units));
            left -= u;
            units = static_cast<uint32_t>(u);
        }
        if (grp != -1) bs_walk_exact(t, Pc, Qc, units);
        // the pipelines' last lanes: finished groups to the result buffer, late wrap chunks
        // to their counters
        const bool done = pos == S - 1 && grp >= 0;
        const unsigned dm = __ballot_sync(kFull, done);
        if (done) {
            const int slot = nemit + __popc(dm & ((1u << lane) - 1u));
#pragma unroll
            for (int w = 0; w < 16; ++w) {
                E.cnt[slot][w] = Pc.c[w];
                E.cnt[slot][16 + w] = Qc.c[w];
            }
            E.grp[slot] = grp;
        } else if (WRAP && pos == S - 1 && grp < -1 && grp >= -32) {
            const int k = static_cast<int>(-1 - grp);
#pragma unroll
            for (int w = 0; w < 16; ++w) {
                E.late[g * S + k][w] = Pc.c[w];
                E.late[g * S + k][16 + w] = Qc.c[w];
            }
        }
        nemit += __popc(dm);
        if (nemit > 32 - P) {
            flush(nemit);
            nemit = 0;
        }
        if (WRAP) {
            const bool last = cur_feed == -34;  // this pipeline's step ends its wrap groups' early chunks
            if (__any_sync(kFull, last)) {
                __syncwarp();
                const unsigned fm = __ballot_sync(kFull, last && pos < S - 1);
                if (last && pos < S - 1) {  // early counters (registers) + late counters (shared)
                    uint32_t d[32];
#pragma unroll
                    for (int w = 0; w < 16; ++w) {
                        d[w] = Pc.c[w];
                        d[16 + w] = Qc.c[w];
                    }
                    bs_dx_store(d, E.late[g * S + pos + 1], reinterpret_cast<int32_t*>(E.late[g * S + pos + 1]));
                }
                __syncwarp();
                for (unsigned mm = fm; mm; mm &= mm - 1) {  // wrap group of lane l: (l / S, l % S)
                    const int l = __ffs(static_cast<int>(mm)) - 1;
                    store_group(gwarp * (P * kWr) + (l / S) * kWr + l % S, E.late[l + 1]);
                }
                if (last) {
                    fin = true;
                    grp = -1;
                }
                __syncwarp();
            }
            if (__all_sync(kFull, fin)) break;
        }
        // feed: the last lane of each pipeline (its group emitted) takes the next item, and
        // the hand-over rotates it to the first lane
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        take(pos == S - 1 && !fin, feed, fidx, E.seed[buf][g]);
        cur_feed = fin ? -1 : feed;
#pragma unroll
        for (int i = 1; i < 32; ++i) t.b1[i] = __shfl_sync(kFull, t.b1[i], src);
#pragma unroll
        for (int i = 3; i < 32; ++i) t.b2[i] = __shfl_sync(kFull, t.b2[i], src);
#pragma unroll
        for (int i = 4; i < 32; ++i) t.b3[i] = __shfl_sync(kFull, t.b3[i], src);
#pragma unroll
        for (int w = 0; w < 16; ++w) {
            Pc.c[w] = __shfl_sync(kFull, Pc.c[w], src);
            Qc.c[w] = __shfl_sync(kFull, Qc.c[w], src);
        }
        grp = __shfl_sync(kFull, grp, src);
        if (WRAP) left = __shfl_sync(kFull, left, src);
        if (!WRAP && !more && !__any_sync(kFull, grp != -1)) break;
        phase = phase == S - 1 ? 0 : phase + 1;
    }
    flush(nemit);
}

// ---------------------------------------------------------------------------------
// Walk WLP, bitsliced lane chunks: one warp per group of 32 replications, lane l runs
// steps [l*K, (l+1)*K) of all 32 (as k_wlp_lanes does for one replication). Each lane
// jumps the 32 seeds to its chunk (lane_jump, nibble tables in shared memory), transposes
// them into bit planes, walks its chunk with the carry-save counters (all lanes run the
// same ceil(K/16) blocks; steps past a lane's chunk are masked out of the counts and its
// end state is never used), and the warp sums the lanes' counts as bitsliced two's-
// complement numbers by a butterfly of shuffles; lane j reads stream j's total, folds and
// stores it (coalesced). No drain: a warp per group from the first step,
// so it suits R too small for the pipeline (config 3). Chunk counts < 2^16: K < 65536.
// ---------------------------------------------------------------------------------
constexpr int kBsLanesBlock = 128;  // 2 blocks (8 warps) per SM at ~250 registers

__global__ void __launch_bounds__(kBsLanesBlock, 2) k_wlp_walk_bs_lanes(RepArgs a, const uint32_t* __restrict__ gtab,
                                                                    int64_t K) {
    extern __shared__ uint32_t tab[];  // kLaneTabWords
    stage_u32<kLaneTabWords>(tab, gtab);
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    int64_t mine = a.n - static_cast<int64_t>(lane) * K;
    mine = mine < 0 ? 0 : (mine > K ? K : mine);
    const uint32_t units = static_cast<uint32_t>(mine);
    const uint32_t blocks = static_cast<uint32_t>((K + 15) / 16);
    const int64_t groups = (a.count + 31) / 32;
    RepArgs ga = a;
    ga.count = groups;
    for (int64_t g = grab_take(grab_issue(ga, lane)); g < groups;) {
        const unsigned long long ticket = grab_issue(ga, lane);
        const int64_t gend = g + a.grab < groups ? g + a.grab : groups;
        for (; g < gend; ++g) {
            BsTaus t;
#pragma unroll
            for (int j = 0; j < 32; ++j) {  // every lane reads the same 32 seeds (broadcast)
                const int64_t r = g * 32 + j;
                const Taus st = lane_jump(tab, lane, r < a.count ? load_seed(a, r) : Taus{kMin1, kMin2, kMin3});
                t.b1[j] = st.s1;
                t.b2[j] = st.s2;
                t.b3[j] = st.s3;
            }
            transpose32(t.b1);
            transpose32(t.b2);
            transpose32(t.b3);
            BsCount P, Q;
            bs_count_init(P);
            bs_count_init(Q);
            bs_walk_units(t, P, Q, units, blocks);
            // dx = P - Q summed over the lanes without leaving bit-plane form: D = P + ~Q + 1
            // in 22-digit two's complement (|dx| <= n < 2^21), then a 5-round butterfly of
            // bitsliced additions (every lane ends with the warp total of all 32 streams),
            // then lane j reads stream j's digits: ~440 operations instead of two 32x32
            // transposes and a transpose-reduce (~960).
            constexpr int kD = 22;
            uint32_t D[kD];
            uint32_t carry = ~0u;  // the +1 of the negation, in every stream
#pragma unroll
            for (int w = 0; w < kD; ++w) {
                const uint32_t x = w < 16 ? P.c[w] : 0u, y = ~(w < 16 ? Q.c[w] : 0u);
                D[w] = x ^ y ^ carry;
                carry = (x & y) | (carry & (x ^ y));
            }
#pragma unroll
            for (int s = 16; s >= 1; s >>= 1) {
                uint32_t c = 0u;
#pragma unroll
                for (int w = 0; w < kD; ++w) {
                    const uint32_t o = __shfl_xor_sync(kFull, D[w], s);
                    const uint32_t t = D[w] ^ o ^ c;
                    c = (D[w] & o) | (c & (D[w] ^ o));
                    D[w] = t;
                }
            }
            int32_t dx = 0;
#pragma unroll
            for (int w = 0; w < kD; ++w) dx |= static_cast<int32_t>((D[w] >> lane) & 1u) << w;
            dx = static_cast<int32_t>(static_cast<uint32_t>(dx) << (32 - kD)) >> (32 - kD);  // sign-extend from digit 21
            const int64_t r = g * 32 + lane;
            if (r < a.count) put1(a, r, walk_fold(dx, a.chunks));
        }
        g = grab_take(ticket);
    }
}

// mm1 thread per replication: each lane runs its own queue; the exponentials of 4
// clients (8 draws) per lane go through the warp-cooperative batch log. Every thread of
// a warp takes part in each batch up to the warp's longest replication (`n_warp`).
struct TlpMm1Warp {
    NearList nl;
    double res[32 * kExpoB];
};

template <int DIV, bool FULL, bool COUNT = false>
__device__ __forceinline__ Queue mm1_thread_rep(Taus st, int64_t n, int64_t n_warp, double lambda, double mu,
                                                double inv_l, double inv_m, const double* logtab, TlpMm1Warp& W,
                                                unsigned mask, int lane, bool live = true,
                                                unsigned* events = nullptr) {
    Queue q;
    const unsigned act = COUNT ? __ballot_sync(mask, live) : 0u;  // lanes of real replications
    for (int64_t done = 0; done < n_warp; done += kExpoB / 2) {
        uint32_t d[kExpoB];
        double e[kExpoB];
#pragma unroll
        for (int j = 0; j < kExpoB; j += 2) taus_next2(st, d[j], d[j + 1]);
        neg_log1m_batch<kExpoB, FULL>(d, e, logtab, W.nl, W.res, mask, lane);
        const int64_t left = n - done;
        const int cnt = left <= 0 ? 0 : (left < kExpoB / 2 ? static_cast<int>(left) : kExpoB / 2);
#pragma unroll
        for (int c = 0; c < kExpoB / 2; ++c)
            if (c < cnt) {
                const bool dry =
                    q.client(scale<DIV>(e[2 * c], lambda, inv_l), scale<DIV>(e[2 * c + 1], mu, inv_m));
                if (COUNT && act) split_if(act, dry, *events, mask);  // models.cpp:199-201's if
            }
    }
    return q;
}

// mm1 WLP as a warp pipeline (many replications per warp). Replication r enters at lane
// 0 and moves one lane per step; lane l runs clients [l*K, (l+1)*K) of it strictly in
// order (the reference's recursion and ordered sums, models.hpp:65-79) from the queue
// and stream state lane l-1 hands over, so every operation happens in the reference's
// order on one lane and no chaining rounds or separate sum phase are needed. All 32 lanes
// work every step (each on a different replication's segment); the exponentials go
// through the warp-cooperative log batches as in TLP. Draws of a segment's last, partial
// batch are predicated so each lane hands over the state exactly at its segment's end.
// EXACT = false: every lane whose hand-over state matters (lanes 0-30) has whole panels
// (31*K <= n and K % kPanT == 0), so draws need no predication (lane 31, and lanes between
// replications, may overdraw: their stream state is never handed over).
// ---------------------------------------------------------------------------------
// mm1 exponential panels. A lane's next kPanT clients take 2*kPanT draws; their scaled
// exponentials (a, s) go to the lane's row of a shared-memory panel as 16-byte pairs,
// and the recursion then reads the pairs back in client order. The near-one inputs of
// the whole warp's panel (1 in 16, ~32 of 512) are listed once — their places in the
// list come from one lane scan of the per-lane counts, done before any log — and the
// warp evaluates them in one (rarely two) full passes that write straight into the
// panel slots: no per-batch compaction, no predicated patch-back into registers.
// ---------------------------------------------------------------------------------
constexpr int kPanT = 8;            // clients per lane per panel
static_assert(kPanT == kMm1PanelT, "the mm1 pipeline schedule counts panels of kMm1PanelT clients");
constexpr int kPanD = 2 * kPanT;    // draws per lane per panel
constexpr int kNearCap = 64;        // near list entries (expected 32 per panel; more: lane-local path)
constexpr uint32_t kNearMax = 0x10000000u;  // draw n is near one (1 - n 2^-32 >= 1 - 2^-4) iff n <= 2^28

// Column-major panel: client c of lane l is the 16-byte pair v[(c * 32 + l) * 2 ..], draw
// quad q of lane l is dr[(q * 32 + l) * 4 ..]. A quarter warp's STS.128 / LDS.128 of one
// column covers 128 consecutive bytes (all 32 banks), every offset is a compile-time
// immediate, and nothing is padded: 6.5 KB per warp, so 4 blocks of 8 warps fit an SM.
struct PanelWarp {
    double v[kPanT * 32 * 2];  // (a, s) of client c, lane l at [(c*32 + l)*2]
    uint32_t dr[kPanD * 32];   // draws 4q..4q+3 of lane l at [(q*32 + l)*4]
    uint2 nl[kNearCap];        // near list: {draw, panel slot (double index into v)}
};
// Slot (double index into PanelWarp::v) of draw j of lane l: client j/2, a (even j) or s.
__host__ __device__ constexpr int pan_slot(int j, int l) { return ((j >> 1) * 32 + l) * 2 + (j & 1); }

// e / mu for a service time (kDivPow2One: mu = 1, the identity)
template <int DIV>
__device__ __forceinline__ double scale_mu(double e, double mu, double inv_m) {
    if constexpr (DIV == kDivPow2One)
        return e;
    else
        return scale<DIV>(e, mu, inv_m);
}

// e / rate for panel slot parity `odd` (odd slots are services: mu; even arrivals: lambda)
template <int DIV>
__device__ __forceinline__ double scale_slot(double e, bool odd, double lambda, double mu, double inv_l, double inv_m) {
    if constexpr (DIV == kDivPow2One)
        return odd ? e : scale<DIV>(e, lambda, inv_l);
    else
        return scale<DIV>(e, odd ? mu : lambda, odd ? inv_m : inv_l);
}

#ifndef WLP_PAN_UNROLL
#define WLP_PAN_UNROLL 4
#endif
#ifndef WLP_PAN_MASK
#define WLP_PAN_MASK 1
#endif
constexpr int kPanUnroll = WLP_PAN_UNROLL;

// Near-one flag of draw n shifted into m: m = 2m + [n <= 2^28] (a subtract's borrow-out
// carried into an add: two integer ops, no predicate-to-register select).
__device__ __forceinline__ void near_bit(uint32_t& m, uint32_t n) {
#if WLP_PAN_MASK
    // the borrow-out of n - (2^28 + 1) is a carry flag of 0 (PTX sub.cc records a - b as
    // a + ~b + 1): the carry is 1 exactly when n > 2^28, so shift in its complement via
    // 2^28 - n, whose carry is 1 exactly when n <= 2^28
    asm("{\n\t.reg .u32 t;\n\tsub.cc.u32 t, %1, %2;\n\taddc.u32 %0, %0, %0;\n\t}"
        : "+r"(m)
        : "r"(kNearMax), "r"(n));
#else
    m = 2u * m + (n <= kNearMax ? 1u : 0u);
#endif
}

// List append of draw j (near iff bit kPanD-1-j of the lane's mask is set).
__device__ __forceinline__ void near_append_m(uint32_t& sp, uint32_t m, int j, uint32_t n, uint32_t slot) {
    const uint32_t bit = m & (1u << (kPanD - 1 - j));
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t"
                 "@p st.shared.v2.u32 [%0], {%2, %3};\n\t@p add.u32 %0, %0, 8;\n\t}"
                 : "+r"(sp)
                 : "r"(bit), "r"(n), "r"(slot)
                 : "memory");
}

// Fills the lane's panel row with the next `ndraw` draws' exponentials (EXACT: draws past
// ndraw are not taken, so the stream state ends exactly there; else all kPanD are taken).
// All lanes of `mask` (contiguous low lanes) take part. On return the row is final.
// Pass 1 draws into the lane's draw row and builds its near-one bit mask; one lane scan
// of the popcounts places each lane's near-ones in the list; pass 2 evaluates the table
// path for every draw and lists the near ones; then the warp evaluates the list into the
// panel.
template <int DIV, bool EXACT>
__device__ __forceinline__ void panel_fill(Taus& st, int ndraw, double lambda, double mu, double inv_l,
                                           double inv_m, const double* tab, PanelWarp& P, unsigned mask,
                                           int lane, unsigned* ev = nullptr) {
    uint4* dq = reinterpret_cast<uint4*>(P.dr) + lane;  // quad q at dq[q * 32]
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < kPanD; j += 4) {
        uint4 q4;
        if (EXACT) {
            // filler past ndraw: a table-path value (never listed, never read)
            q4.x = j < ndraw ? taus_next(st) : 0x80000000u;
            q4.y = j + 1 < ndraw ? taus_next(st) : 0x80000000u;
            q4.z = j + 2 < ndraw ? taus_next(st) : 0x80000000u;
            q4.w = j + 3 < ndraw ? taus_next(st) : 0x80000000u;
        } else {
            taus_next2(st, q4.x, q4.y);
            taus_next2(st, q4.z, q4.w);
        }
        near_bit(m, q4.x);
        near_bit(m, q4.y);
        near_bit(m, q4.z);
        near_bit(m, q4.w);
        dq[(j / 4) * 32] = q4;
    }
    const int c = __popc(m);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(mask, incl, o);
        if (lane >= o) incl += v;
    }
    const int width = mask == kFull ? 32 : __popc(mask);
    const int total = __shfl_sync(mask, incl, width - 1);
    const bool listed = total <= kNearCap;  // warp-uniform
    double2* vq = reinterpret_cast<double2*>(P.v) + lane;  // client c at vq[c * 32]
    const uint32_t slot0 = static_cast<uint32_t>(pan_slot(0, lane));
    uint32_t sp = static_cast<uint32_t>(__cvta_generic_to_shared(P.nl + (incl - c)));
#pragma unroll kPanUnroll
    for (int j = 0; j < kPanD; j += 4) {
        const uint4 q4 = dq[(j / 4) * 32];
        const double a0 = scale<DIV>(neg_log1m_table_dev(q4.x, tab), lambda, inv_l);
        const double s0 = scale<DIV>(neg_log1m_table_dev(q4.y, tab), mu, inv_m);
        const double a1 = scale<DIV>(neg_log1m_table_dev(q4.z, tab), lambda, inv_l);
        const double s1 = scale<DIV>(neg_log1m_table_dev(q4.w, tab), mu, inv_m);
        vq[(j / 2) * 32] = make_double2(a0, s0);
        vq[(j / 2 + 1) * 32] = make_double2(a1, s1);
        if (listed) {
            near_append_m(sp, m, j, q4.x, slot0 + pan_slot(j, 0));
            near_append_m(sp, m, j + 1, q4.y, slot0 + pan_slot(j + 1, 0));
            near_append_m(sp, m, j + 2, q4.z, slot0 + pan_slot(j + 2, 0));
            near_append_m(sp, m, j + 3, q4.w, slot0 + pan_slot(j + 3, 0));
        }
    }
    if (listed) {
        __syncwarp(mask);
        if (ev) *ev += loop_split_events(mask, lane < total ? static_cast<unsigned>((total - lane + width - 1) / width) : 0u);
        for (int k = lane; k < total; k += width) {
            const uint2 it = P.nl[k];
            const double e = it.x == 0u ? -0.0 : -log_near_one_dev(one_minus_u32_dev(it.x));
            P.v[it.y] = scale_slot<DIV>(e, it.y & 1u, lambda, mu, inv_l, inv_m);
        }
    } else {  // (rare: > kNearCap near draws in the panel) each lane fixes its own clients
        const uint32_t* dr = P.dr + lane * 4;
        for (int j = 0; j < kPanD; ++j) {
            const uint32_t n = dr[(j >> 2) * 128 + (j & 3)];
            if (n <= kNearMax) {
                const double e = n == 0u ? -0.0 : -log_near_one_dev(one_minus_u32_dev(n));
                P.v[pan_slot(j, lane)] = scale_slot<DIV>(e, j & 1, lambda, mu, inv_l, inv_m);
            }
        }
    }
    __syncwarp(mask);
}

// The recursion over `cnt` clients of the lane's panel row (cnt == kPanT: unpredicated).
// COUNT: warp-level splits of the `t < 0` branch (models.cpp:199-201) over lanes `act`.
template <bool COUNT = false>
__device__ __forceinline__ void panel_clients(Queue& q, const PanelWarp& P, int cnt, int lane, unsigned act = 0u,
                                              unsigned sync = 0u, unsigned* events = nullptr) {
    const double2* row = reinterpret_cast<const double2*>(P.v) + lane;  // client c at row[c * 32]
    if (!COUNT && cnt == kPanT) {
#pragma unroll
        for (int c = 0; c < kPanT; ++c) {
            const double2 v = row[c * 32];
            q.client(v.x, v.y);
        }
    } else {
#pragma unroll
        for (int c = 0; c < kPanT; ++c) {
            const bool on = c < cnt;
            bool dry = false;
            if (on) {
                const double2 v = row[c * 32];
                dry = q.client(v.x, v.y);
            }
            if (COUNT && act && on) split_if(act, dry, *events, sync);  // (cnt is warp-uniform in TLP)
        }
    }
}

// mm1 WLP as a warp pipeline, rotating schedule (PipeSched with G = kPanT clients: every
// lane runs the same number of whole panels per step, and any 32 consecutive steps cover
// a replication's n clients; with a fixed split ceil(n/32) lane 31 idled through 3 of 4
// panels at 1,000 clients). Lane 31 stores each finished replication's three outputs
// itself (three one-lane stores per step, ~1 % of a step's instructions), which frees the
// shared memory of a result buffer: with the column-major panel, 4 blocks of 8 warps fit.
// EXACT: some chunk has a partial panel (n % kPanT != 0), whose draws are predicated so
// the hand-over state is exact; otherwise lanes draw whole panels unpredicated.
template <int DIV, bool EXACT>
// 4 blocks of 8 warps per SM (64 registers, no spills; the compact near list keeps the
// panel kernel's block at 54 KB of shared memory): config 4 42.4 -> 41.7 ms against 3.
#ifndef WLP_MM1_MINB
#define WLP_MM1_MINB 4
#endif
__global__ void __launch_bounds__(kMm1Block, WLP_MM1_MINB) k_wlp_mm1_pipe_ragged(RepArgs a, PipeSched ps) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* logtab = reinterpret_cast<double*>(smraw);
    PanelWarp& P = reinterpret_cast<PanelWarp*>(logtab + 256)[threadIdx.x >> 5];
    stage_log_table(logtab);
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31;
    const double nd = static_cast<double>(a.n);
    Taus st{kMin1, kMin2, kMin3};
    Queue q;
    long long rep = -1;
    int64_t cur = 0, cend = 0;
    bool more = true;
    int phase = 0;
    for (;;) {
        if (more && cur >= cend) {
            const int64_t base = grab_take(grab_issue(a, lane));
            if (base >= a.count) {
                more = false;
            } else {
                cur = base;
                cend = base + a.grab < a.count ? base + a.grab : a.count;
            }
        }
        if (lane == 0) {  // feed: a fresh queue on the next replication's stream
            rep = more ? cur : -1;
            if (more) {
                st = load_seed(a, cur);
                q = Queue();
            }
        }
        if (more) ++cur;
        if (!__any_sync(kFull, rep >= 0)) break;
        const int units = rep >= 0 ? pipe_units(ps, phase) : 0;
        const int steps = (pipe_units(ps, phase) + kPanT - 1) / kPanT;  // warp-uniform
        for (int p = 0; p < steps; ++p) {
            const int left = units - p * kPanT;
            const int cnt = left <= 0 ? 0 : (left < kPanT ? left : kPanT);
            panel_fill<DIV, EXACT>(st, 2 * cnt, a.lambda, a.mu, a.inv_lambda, a.inv_mu, logtab, P, kFull, lane);
            panel_clients(q, P, cnt, lane);
        }
        if (lane == 31 && rep >= 0) {  // lane 31 finished a replication
            put3(a, rep, __ddiv_rn(q.idle, nd), __ddiv_rn(q.sumw, nd), __ddiv_rn(q.sums, nd));
        }
        st.s1 = __shfl_up_sync(kFull, st.s1, 1);
        st.s2 = __shfl_up_sync(kFull, st.s2, 1);
        st.s3 = __shfl_up_sync(kFull, st.s3, 1);
        q.u = __shfl_up_sync(kFull, q.u, 1);
        q.idle = __shfl_up_sync(kFull, q.idle, 1);
        q.sumw = __shfl_up_sync(kFull, q.sumw, 1);
        q.sums = __shfl_up_sync(kFull, q.sums, 1);
        rep = __shfl_up_sync(kFull, rep, 1);
        phase = (phase + 1) & 31;
    }
}

constexpr size_t kMm1PipeSmem = 256 * 8 + (kMm1Block / 32) * sizeof(PanelWarp);

// ---------------------------------------------------------------------------------
// mm1 WLP warp pipeline, single-pass panels with the recursion interleaved (the default
// for n % 8 == 0). Per lane and panel of kPanT clients:
// * one pass draws, evaluates the branch-free table path of every exponential and stores
//   the (a, s) pairs column-major; the draws go to a staging row (one STS.128 per two
//   clients) and their near-one flags into a per-lane bit mask (two integer ops a draw);
// * each lane claims room for its near-ones (1 in 16) in the panel's list with one
//   shared-memory atomic and writes one compact entry {lane, bit} per near draw (a loop
//   over the set bits of its mask only); the warp then evaluates the
//   list (one pass of the near-one polynomial across the lanes, straight into the slots).
//   More than the list capacity (never at random draws) makes each lane fix its own from
//   the staged draws;
// S lanes per replication (32, or 8: four pipelines per warp, 4x longer steps; mm1 has
// no wrap, its queue state is sequential, so the S-1 step drain remains: ~1 % at config 4).
// ---------------------------------------------------------------------------------
constexpr int kNearCap2 = 128;  // list entries per panel (expected 32 of 512 draws)

struct Mm1Pan {
    double2 v[kPanT][32];     // (a, s) of client c of lane l
    uint4 dr[kPanD / 4][32];  // the panel's draws: draws 4q..4q+3 of lane l at dr[q][l]
    uint32_t nl[kNearCap2];   // near list: lane << 5 | mask bit (draw 15 - bit of that lane)
    uint32_t cnt, pad_[3];    // list entries claimed (zero between panels)
};
constexpr size_t kMm1Pipe2Smem = 256 * 8 + (kMm1Block / 32) * sizeof(Mm1Pan);

// Clients c, c+1 of a panel: four draws, their table-path exponentials to the slots, the
// draws to the staging rows (one STS.128), their near-one flags into the lane's mask m
// (bit 15 - j for draw j: two integer ops per draw, no branch).
template <int DIV>
__device__ __forceinline__ void fill_pair(Taus& st, int c, int lane, uint32_t& m, double lambda, double mu,
                                          double inv_l, double inv_m, const double* tab, Mm1Pan& W) {
    uint4 q4;
    taus_next2(st, q4.x, q4.y);
    taus_next2(st, q4.z, q4.w);
    near_bit(m, q4.x);
    near_bit(m, q4.y);
    near_bit(m, q4.z);
    near_bit(m, q4.w);
    W.dr[c / 2][lane] = q4;
    W.v[c][lane] = make_double2(scale<DIV>(neg_log1m_table_dev(q4.x, tab), lambda, inv_l),
                                scale_mu<DIV>(neg_log1m_table_dev(q4.y, tab), mu, inv_m));
    W.v[c + 1][lane] = make_double2(scale<DIV>(neg_log1m_table_dev(q4.z, tab), lambda, inv_l),
                                    scale_mu<DIV>(neg_log1m_table_dev(q4.w, tab), mu, inv_m));
}

// The near-one draws of the panel just filled, into their slots. Each lane's flag mask m
// (~1 set bit of 16) is turned into list entries at the place one atomic on the panel's
// counter gives the lane (WLP_NEAR_ATOMS=0: a lane scan of the counts; config 4 42.14 vs
// 41.83 ms); the warp then evaluates the list in one pass across the lanes. More than `cap` near-ones (never at random draws: 128 of 512)
// fall back to each lane fixing its own from the staged draws. Idle lanes (on = false)
// list nothing.
#ifndef WLP_NEAR_ATOMS
#define WLP_NEAR_ATOMS 1
#endif
template <int DIV>
__device__ __forceinline__ void fix_near(Mm1Pan& W, int lane, bool on, uint32_t m, double lambda, double mu,
                                         double inv_l, double inv_m, uint32_t cap) {
    if (!on) m = 0u;
    const uint32_t c = static_cast<uint32_t>(__popc(m));
    double* v = reinterpret_cast<double*>(&W.v[0][0]);
    const uint32_t* dr = reinterpret_cast<const uint32_t*>(&W.dr[0][0]);
#if WLP_NEAR_ATOMS
    // Each lane claims its c entries with one shared-memory atomic on the panel counter
    // (lanes with no near-one skip it); the entries' order depends on the atomics' order,
    // the values do not. Five dependent shuffles of a lane scan cost more.
    __syncwarp();  // the previous panel's list reads and counter reset are done
    uint32_t pos = 0;
    if (c) pos = atomicAdd(&W.cnt, c);
    const bool fits = pos + c <= cap;  // (false on some lane => the total is over cap)
#else
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t pos = incl - c;
    const bool fits = incl <= cap;
    __syncwarp();
#endif
    const uint32_t m0 = m;
    if (fits) {
        // the set-bit loop runs as often as the lane with the most near-ones (~3 times a
        // panel), so each pass is kept to FLO, the bit clear, the entry and its store
        uint32_t* e = W.nl + pos;
        const uint32_t tag = static_cast<uint32_t>(lane) << 5;
        while (m) {
            const uint32_t b = 31u - static_cast<uint32_t>(__clz(m));
            m ^= 1u << b;
            *e++ = tag | b;
        }
    }
    __syncwarp();
#if WLP_NEAR_ATOMS
    const uint32_t total = W.cnt;
#else
    const uint32_t total = __shfl_sync(kFull, incl, 31);
#endif
    if (total <= cap) {
        for (uint32_t k = lane; k < total; k += 32) {
            const uint32_t it = W.nl[k], l = it >> 5, j = 15u - (it & 31u);
            const uint32_t n = dr[(j >> 2) * 128 + l * 4 + (j & 3)];
            const uint32_t slot = static_cast<uint32_t>(pan_slot(static_cast<int>(j), static_cast<int>(l)));
            const double e = n == 0u ? -0.0 : -log_near_one_dev(one_minus_u32_dev(n));
            v[slot] = scale_slot<DIV>(e, slot & 1u, lambda, mu, inv_l, inv_m);
        }
    } else {  // (never at random draws) each lane fixes its own near-ones from the staging rows
        m = m0;
        while (m) {
            const int j = __clz(m) - 16;
            m &= ~(0x8000u >> j);
            const uint32_t n = dr[(j >> 2) * 128 + lane * 4 + (j & 3)];
            const double e = n == 0u ? -0.0 : -log_near_one_dev(one_minus_u32_dev(n));
            v[pan_slot(j, lane)] = scale_slot<DIV>(e, j & 1, lambda, mu, inv_l, inv_m);
        }
    }
    __syncwarp();
#if WLP_NEAR_ATOMS
    if (lane == 0) W.cnt = 0u;  // (ordered before the next panel's atomics by its first sync)
#endif
}

// One pipeline step of a lane: np panels of its chunk (np >= 1, warp-uniform). Panel p's
// recursion runs two clients at a time interleaved with the fill of panel p + 1 into the
// same slots (each slot is read by the recursion before its own lane overwrites it).
template <int DIV>
__device__ __forceinline__ void mm1_chunk(Taus& st, Queue& q, int np, int lane, bool on, double lambda, double mu,
                                          double inv_l, double inv_m, const double* tab, Mm1Pan& W, uint32_t cap) {
    uint32_t m = 0;
#pragma unroll
    for (int c = 0; c < kPanT; c += 2) fill_pair<DIV>(st, c, lane, m, lambda, mu, inv_l, inv_m, tab, W);
    fix_near<DIV>(W, lane, on, m, lambda, mu, inv_l, inv_m, cap);
    for (int p = 1; p < np; ++p) {
        m = 0;
#pragma unroll
        for (int c = 0; c < kPanT; c += 2) {
            const double2 v0 = W.v[c][lane], v1 = W.v[c + 1][lane];  // panel p-1's clients c, c+1
            q.client(v0.x, v0.y);
            q.client(v1.x, v1.y);
            fill_pair<DIV>(st, c, lane, m, lambda, mu, inv_l, inv_m, tab, W);
        }
        fix_near<DIV>(W, lane, on, m, lambda, mu, inv_l, inv_m, cap);
    }
#pragma unroll
    for (int c = 0; c < kPanT; ++c) {
        const double2 v = W.v[c][lane];
        q.client(v.x, v.y);
    }
}

template <int DIV, int S>
__global__ void __launch_bounds__(kMm1Block, WLP_MM1_MINB) k_wlp_mm1_pipe(RepArgs a, PipeSched ps) {
    constexpr int P = 32 / S;
    extern __shared__ __align__(16) unsigned char smraw[];
    double* logtab = reinterpret_cast<double*>(smraw);
    Mm1Pan& W = reinterpret_cast<Mm1Pan*>(logtab + 256)[threadIdx.x >> 5];
    stage_log_table(logtab);
    if ((threadIdx.x & 31) == 0) W.cnt = 0u;
    __syncthreads();
    pdl_wait();
    const int lane = threadIdx.x & 31, g = lane / S, pos = lane % S;
    const double nd = static_cast<double>(a.n);
    Taus st{kMin1, kMin2, kMin3};
    Queue q;
    long long rep = -1;
    int64_t cur = 0, cend = 0;
    bool more = true;
    int phase = 0;
    for (;;) {
        if (more && cur >= cend) {  // next group (a multiple of P replications)
            const int64_t base = grab_take(grab_issue(a, lane));
            if (base >= a.count) {
                more = false;
            } else {
                cur = base;
                cend = base + a.grab < a.count ? base + a.grab : a.count;
            }
        }
        if (pos == 0) {  // feed each pipeline a fresh queue on its next replication's stream
            const int64_t r = cur + g;
            rep = more && r < cend ? r : -1;
            if (rep >= 0) {
                st = load_seed(a, r);
                q = Queue();
            }
        }
        if (more) cur += P;
        if (!more && !__any_sync(kFull, rep >= 0)) break;
        const int np = pipe_units(ps, phase) / kPanT;
        if (np > 0)
            mm1_chunk<DIV>(st, q, np, lane, rep >= 0, a.lambda, a.mu, a.inv_lambda, a.inv_mu, logtab, W, a.near_cap);
        if (pos == S - 1 && rep >= 0) {  // the pipeline's last lane finished a replication
            put3(a, rep, __ddiv_rn(q.idle, nd), __ddiv_rn(q.sumw, nd), __ddiv_rn(q.sums, nd));
        }
        st.s1 = __shfl_up_sync(kFull, st.s1, 1, S);
        st.s2 = __shfl_up_sync(kFull, st.s2, 1, S);
        st.s3 = __shfl_up_sync(kFull, st.s3, 1, S);
        q.u = __shfl_up_sync(kFull, q.u, 1, S);
        q.idle = __shfl_up_sync(kFull, q.idle, 1, S);
        q.sumw = __shfl_up_sync(kFull, q.sumw, 1, S);
        q.sums = __shfl_up_sync(kFull, q.sums, 1, S);
        rep = __shfl_up_sync(kFull, rep, 1, S);
        phase = phase == S - 1 ? 0 : phase + 1;
    }
}


__device__ __forceinline__ unsigned block_lane_mask() {  // partial last warp of odd-sized blocks
    const int in_warp = static_cast<int>(blockDim.x) - (static_cast<int>(threadIdx.x) & ~31);
    return in_warp >= 32 ? kFull : ((1u << in_warp) - 1u);
}

#ifndef WLP_TLP_MM1_MINB
#define WLP_TLP_MM1_MINB 4
#endif
// SMALL: blocks of at most 256 threads (the default TLP block), register budget for
// WLP_TLP_MM1_MINB blocks per SM; else any block size up to 1024.
template <int DIV, bool COUNT, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 1024, SMALL ? WLP_TLP_MM1_MINB : 1) k_tlp_mm1(RepArgs a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* logtab = reinterpret_cast<double*>(smraw);
    PanelWarp& W = reinterpret_cast<PanelWarp*>(logtab + 256)[threadIdx.x >> 5];
    stage_log_table(logtab);
    __syncthreads();
    pdl_wait();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const bool live = r < a.count;
    Taus st = live ? load_seed(a, r) : Taus{2u, 8u, 16u};  // tail threads: dummy stream
    const unsigned mask = block_lane_mask();
    unsigned events = 0, splits = 0;
    const unsigned act = COUNT ? __ballot_sync(mask, live) : 0u;  // lanes of real replications
    const long long t0 = COUNT ? hw_clock() : 0;
    Queue q;
    for (int64_t done = 0; done < a.n; done += kPanT) {  // every replication of the launch has a.n clients
        const int cnt = a.n - done < kPanT ? static_cast<int>(a.n - done) : kPanT;
        panel_fill<DIV, false>(st, 2 * kPanT, a.lambda, a.mu, a.inv_lambda, a.inv_mu, logtab, W, mask, lane,
                               COUNT ? &splits : nullptr);
        panel_clients<COUNT>(q, W, cnt, lane, act, mask, &events);
    }
    if (COUNT) {
        HwTally hw;
        hw.t0 = t0;
        hw.div = events;
        hw.splits = splits;
        const bool any_live = __any_sync(mask, live);
        // the seed loads are predicated, so a warp of dummy lanes still issues them
        hw.ld = staged_loads(256) + 3u;
        hw.st = any_live ? 3u : 0u;
        flush_tally(hw, a.hw);
    }
    if (!live) return;
    const double nd = static_cast<double>(a.n);
    put3(a, r, __ddiv_rn(q.idle, nd), __ddiv_rn(q.sumw, nd), __ddiv_rn(q.sums, nd));
}

// ---------------------------------------------------------------------------------
// Experimental plan (BASELINE config 5): heterogeneous factor-level sets, one launch.
// WLP warps take replications from a global counter (costs differ per set); pi/walk use
// fixed panels (kPlanT units per lane) so one pair of jump tables serves every set.
// ---------------------------------------------------------------------------------

__device__ __forceinline__ int find_set(const SetParam* __restrict__ s, int n, int64_t r) {
    int lo = 0, hi = n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s[mid].off <= r)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ Taus plan_seed(const PlanArgs& a, int64_t r) {
    return Taus{__ldg(a.seeds + r), __ldg(a.seeds + a.count + r), __ldg(a.seeds + 2 * a.count + r)};
}

__device__ __forceinline__ int64_t next_rep(const PlanArgs& a, int lane) {
    unsigned long long r = 0;
    if (lane == 0) r = atomicAdd(a.next, 1ull);
    return static_cast<int64_t>(__shfl_sync(kFull, r, 0));
}

template <int MODEL>
__global__ void __launch_bounds__(kWlpBlock, 3) k_plan_lanes(PlanArgs a, const uint32_t* __restrict__ gtab,
                                                              const uint32_t* __restrict__ gskip) {
    extern __shared__ uint32_t sm[];
    uint32_t* tab = sm;
    uint32_t* skip = sm + kLaneTabWords;
    stage_u32<kLaneTabWords>(tab, gtab);
    for (int i = threadIdx.x; i < kUniTabWords; i += blockDim.x) skip[i] = __ldg(gskip + i);
    __syncthreads();
    pdl_wait();  // (the seeding behind which it may launch: seeds and the grab counter)
    const int lane = threadIdx.x & 31;
    constexpr int64_t P = 32 * kPlanT;
    for (int64_t r = next_rep(a, lane); r < a.count; r = next_rep(a, lane)) {
        const SetParam S = a.sets[find_set(a.sets, a.n_sets, r)];
        Taus st = lane_jump(tab, lane, plan_seed(a, r));
        int64_t acc = 0;
        for (int64_t base = 0; base < S.n; base += P) {
            int64_t mine = S.n - base - static_cast<int64_t>(lane) * kPlanT;
            mine = mine < 0 ? 0 : (mine > kPlanT ? kPlanT : mine);
            if (MODEL == 0)
                acc += pi_hits(st, static_cast<uint32_t>(mine));
            else
                acc += walk_dx(st, static_cast<uint32_t>(mine));
            st = uni_jump(skip, st);
        }
        const int64_t total = warp_sum_i64(acc);
        if (lane == 0)
            a.out0[r] = MODEL == 0 ? __ddiv_rn(__dmul_rn(4.0, static_cast<double>(total)), static_cast<double>(S.n))
                                   : walk_fold(total, S.chunks);
    }
}

__global__ void __launch_bounds__(kMm1Block) k_plan_mm1(PlanArgs a, const uint32_t* __restrict__ gtab,
                                                         const uint32_t* __restrict__ gskip) {
    const Mm1Smem m = mm1_stage(gtab, gskip);
    pdl_wait();
    const int lane = threadIdx.x & 31;
    for (int64_t r = next_rep(a, lane); r < a.count; r = next_rep(a, lane)) {
        const SetParam S = a.sets[find_set(a.sets, a.n_sets, r)];
        const Taus st = lane_jump(m.tab, lane, plan_seed(a, r));
        auto rep = [&](auto div) {
            constexpr int D = decltype(div)::value;
            return S.lambda >= a.serial_rho * S.mu  // heavy traffic: ordered loop on lane 0
                       ? mm1_warp_rep_serial<D>(st, S.n, S.lambda, S.mu, S.inv_lambda, S.inv_mu, m.logtab, m.skip,
                                                *m.W, lane)
                       : mm1_warp_rep<D>(st, S.n, S.lambda, S.mu, S.inv_lambda, S.inv_mu, m.logtab, m.skip, *m.W,
                                         lane);
        };
        const double acc = S.div == kDivPow2  ? rep(std::integral_constant<int, kDivPow2>{})
                           : S.div == kDivRcp ? rep(std::integral_constant<int, kDivRcp>{})
                                              : rep(std::integral_constant<int, kDivIeee>{});
        if (lane < 3) {  // lanes 0/1/2 hold sumw/sums/idle
            double* out = lane == 0 ? a.out1 : (lane == 1 ? a.out2 : a.out0);
            out[r] = __ddiv_rn(acc, static_cast<double>(S.n));
        }
    }
}

template <int MODEL>
__global__ void k_plan_tlp(PlanArgs a) {
    pdl_wait();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= a.count) return;
    const SetParam S = a.sets[find_set(a.sets, a.n_sets, r)];
    const Taus st = plan_seed(a, r);
    a.out0[r] = MODEL == 0 ? pi_rep_tlp(st, S.n) : walk_rep_tlp(st, S.n, S.chunks);
}

__global__ void k_plan_tlp_mm1(PlanArgs a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    double* logtab = reinterpret_cast<double*>(smraw);
    TlpMm1Warp& W = reinterpret_cast<TlpMm1Warp*>(logtab + 256)[threadIdx.x >> 5];
    stage_log_table(logtab);
    __syncthreads();
    pdl_wait();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const unsigned mask = block_lane_mask();
    const bool live = r < a.count;
    const SetParam S = a.sets[find_set(a.sets, a.n_sets, live ? r : a.count - 1)];
    const int64_t n = live ? S.n : 0;
    const int64_t n_warp = static_cast<int64_t>(__reduce_max_sync(mask, static_cast<unsigned>(n)));
    const Taus st = live ? plan_seed(a, r) : Taus{2u, 8u, 16u};
    // lanes of one warp may belong to different sets: the reciprocal form takes per-lane
    // rates (an exact 2^-k reciprocal included); IEEE division when any set needs it
    auto rep = [&](auto div) {
        constexpr int D = decltype(div)::value;
        return mask == kFull ? mm1_thread_rep<D, true>(st, n, n_warp, S.lambda, S.mu, S.inv_lambda, S.inv_mu, logtab,
                                                       W, mask, lane)
                             : mm1_thread_rep<D, false>(st, n, n_warp, S.lambda, S.mu, S.inv_lambda, S.inv_mu, logtab,
                                                        W, mask, lane);
    };
    const Queue q = a.tlp_div == kDivRcp ? rep(std::integral_constant<int, kDivRcp>{})
                                         : rep(std::integral_constant<int, kDivIeee>{});
    if (!live) return;
    const double nd = static_cast<double>(S.n);
    a.out0[r] = __ddiv_rn(q.idle, nd);
    a.out1[r] = __ddiv_rn(q.sumw, nd);
    a.out2[r] = __ddiv_rn(q.sums, nd);
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

// One 1024-thread block per SM for pass 1 and 2 (the same threads in flight as 4 blocks of
// 256): 148 block partials, so the ordered device fold and the host merge of pass 2 walk
// a quarter of the entries (fold ~17 -> ~5 us).
constexpr int kStatsBlock = 1024;
constexpr int64_t kStatsSeqMax = 256;

__global__ void __launch_bounds__(kStatsBlock) k_stats(const double* __restrict__ x, int64_t n, int pass,
                                                       double center, double* __restrict__ partials,
                                                       const double* __restrict__ center_dev) {
    if (center_dev) center = *center_dev;  // pass 2 chained on the device (k_stats_fold's mean)
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

// The reference's naive loop (models.cpp:104-109) for any n, bit for bit: the block stages
// tiles of terms (x, or (x - center)^2) in shared memory, double buffered, and thread 0
// adds them in order while the other threads load the next tile. The dependent DADD
// chain (~8 cycles per sample) is the cost: ~4 ns per sample (opt-in, wlp_set_stats_order).
constexpr int kSeqTile = 2048;
__global__ void __launch_bounds__(kStatsBlock) k_stats_seq(const double* __restrict__ x, int64_t n, int pass,
                                                           double center, double* __restrict__ partials,
                                                           const double* __restrict__ center_dev) {
    if (center_dev) center = *center_dev;
    __shared__ double tile[2][kSeqTile];
    const int64_t tiles = (n + kSeqTile - 1) / kSeqTile;
    double s = 0.0;
    auto load = [&](int64_t t, int buf) {
        for (int j = threadIdx.x; j < kSeqTile; j += kStatsBlock) {
            const int64_t i = t * kSeqTile + j;
            if (i < n) tile[buf][j] = stat_term(__ldg(x + i), pass, center);
        }
    };
    load(0, 0);
    __syncthreads();
    for (int64_t t = 0; t < tiles; ++t) {
        const int buf = static_cast<int>(t & 1);
        if (threadIdx.x == 0) {
            const int64_t left = n - t * kSeqTile;
            const int m = left < kSeqTile ? static_cast<int>(left) : kSeqTile;
            const double* v = tile[buf];
            int j = 0;
            for (; j + 8 <= m; j += 8) {
                double r[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = v[j + k];
#pragma unroll
                for (int k = 0; k < 8; ++k) s = __dadd_rn(s, r[k]);
            }
            for (; j < m; ++j) s = __dadd_rn(s, v[j]);
        } else if (t + 1 < tiles) {
            // threads 1.. load the next tile (thread 0's share goes to thread 1)
            for (int j = threadIdx.x - 1; j < kSeqTile; j += kStatsBlock - 1) {
                const int64_t i = (t + 1) * kSeqTile + j;
                if (i < n) tile[buf ^ 1][j] = stat_term(__ldg(x + i), pass, center);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partials[0] = s;
        partials[1] = 0.0;
    }
}

// Pass 1's block partials [used][2] folded in block order into (hi, lo) and the mean, on
// the device (one thread): the same double-double merge, renormalisation and division the
// host does in stats_device, operation for operation, so pass 2 can follow without a round
// trip through the host (meta = {hi, lo, mean}).
// The merge is one thread's ordered loop (the host's order, bit for bit); the warp first
// stages the partials in shared memory, so the loop waits on DADD latencies only, not on
// a global load per partial (headline step: ~53 -> ~10 us under ncu).
constexpr int kFoldStage = 1024;  // partials staged (the stats grids have one block per SM)
__global__ void k_stats_fold(const double* __restrict__ partials, int used, int64_t n, double* __restrict__ meta) {
    __shared__ double sp[2 * kFoldStage];
    if (blockIdx.x != 0) return;
    const bool staged = used <= kFoldStage;
    if (staged) {
        for (int i = threadIdx.x; i < 2 * used; i += blockDim.x) sp[i] = partials[i];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    const double* src = staged ? sp : partials;
    double hi = 0.0, lo = 0.0;
#pragma unroll 4
    for (int b = 0; b < used; ++b) {
        const double v = src[2 * b];
        const double sm = __dadd_rn(hi, v);
        const double bb = __dsub_rn(sm, hi);
        const double err = __dadd_rn(__dsub_rn(hi, __dsub_rn(sm, bb)), __dsub_rn(v, bb));
        hi = sm;
        lo = __dadd_rn(lo, err);
        lo = __dadd_rn(lo, src[2 * b + 1]);
    }
    const double t = __dadd_rn(hi, lo);
    lo = __dsub_rn(lo, __dsub_rn(t, hi));
    hi = t;
    meta[0] = hi;
    meta[1] = lo;
    meta[2] = __ddiv_rn(__dadd_rn(hi, lo), static_cast<double>(n));
}

size_t tlp_mm1_smem(int block) { return 256 * 8 + static_cast<size_t>((block + 31) / 32) * sizeof(TlpMm1Warp); }
size_t tlp_mm1_panel_smem(int block) { return 256 * 8 + static_cast<size_t>((block + 31) / 32) * sizeof(PanelWarp); }

// Once per (device, kernel, size): the attribute calls cost ~1 us of host time each, which
// showed in small runs when they were repeated at every launch.
template <class K>
void allow_smem(K kernel, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    size_t& have = done[{dev, reinterpret_cast<const void*>(kernel)}];
    if (have != 0 && have >= bytes) return;
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    // the persistent grids are sized by the occupancy API, which assumes the largest
    // shared-memory carveout; ask for it so every planned block is resident at once
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    have = bytes;
}

// Launch with the programmatic stream-serialization attribute when t_pdl is set (the
// runtime sets it for model launches that directly follow the seeding kernel and are not
// bracketed by timing events): the kernel's prologue overlaps the seeding's tail.
thread_local bool t_pdl = false;

template <class... KP, class... Args>
cudaError_t launch_ex(void (*kernel)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = t_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KP>(args)...);
}

}  // namespace

void set_pdl_launch(bool on) { t_pdl = on; }

// ---------------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------------

int wlp_blocks_per_sm(int model) {
    int nb = 0;
    if (model == 1) {
        allow_smem(k_wlp_mm1<kDivIeee, false>, kMm1Smem);
        allow_smem(k_wlp_mm1<kDivIeee, true>, kMm1Smem);
        allow_smem(k_wlp_mm1<kDivPow2, false>, kMm1Smem);
        allow_smem(k_wlp_mm1<kDivPow2, true>, kMm1Smem);
        allow_smem(k_wlp_mm1<kDivRcp, false>, kMm1Smem);
        allow_smem(k_wlp_mm1<kDivRcp, true>, kMm1Smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_mm1<kDivIeee, false>, kMm1Block, kMm1Smem);
    } else {
        const size_t smem = kLaneTabWords * 4;
        allow_smem(k_wlp_lanes<0, false>, smem);
        allow_smem(k_wlp_lanes<0, true>, smem);
        allow_smem(k_wlp_lanes<2, false>, smem);
        allow_smem(k_wlp_lanes<2, true>, smem);
        if (model == 0)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_lanes<0, false>, kWlpBlock, smem);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_lanes<2, false>, kWlpBlock, smem);
    }
    return nb < 1 ? 1 : nb;
}

int tlp_blocks_per_sm(int model, int block) {
    int nb = 0;
    switch (model) {
        case 0: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp<0, false>, block, 0); break;
        case 1: {
            const size_t smem = tlp_mm1_panel_smem(block);
            if (block <= 256) {
                allow_smem(k_tlp_mm1<kDivIeee, false, true>, smem);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp_mm1<kDivIeee, false, true>, block, smem);
            } else {
                allow_smem(k_tlp_mm1<kDivIeee, false, false>, smem);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp_mm1<kDivIeee, false, false>, block, smem);
            }
            break;
        }
        default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_tlp<2, false>, block, 0); break;
    }
    return nb < 1 ? 1 : nb;
}

// Slots per thread by run size: a thread's cost is one jump-ahead (a chain of dependent
// table lookups) plus its slots, so large runs amortise the jump over 128 slots
// (R = 1e7: 0.155 ms against 0.245 ms at 32) while small runs want threads (R = 1e5: 25
// blocks at 128).
template <int PER>
cudaError_t launch_seed_per(const SeedArgs& a, cudaStream_t st) {
    const int64_t per_block = static_cast<int64_t>(kSeedBlock) * PER;
    const int64_t grid = (a.count + per_block - 1) / per_block;
    SeedArgs b = a;
    size_t smem = seed_stage_words(PER) * 4;
    if (PER == 8) {  // stage the binary powers up to the largest jump (3 x the last candidate)
        const uint64_t last = 3ull * static_cast<uint64_t>(a.slot_begin + a.count + a.n_rejected);
        b.stage_powers = 64 - __builtin_clzll(last | 1ull);
        smem += static_cast<size_t>(b.stage_powers) * kUniTabWords * 4;
    }
    allow_smem(k_seed<PER>, seed_stage_words(PER) * 4 + 64 * kUniTabWords * 4);
    // PDL: the seeding may launch while the previous run's kernels drain (it waits for them
    // before touching memory), so the launch latency overlaps their tail
    const bool prev = t_pdl;
    t_pdl = true;
    const cudaError_t e = launch_ex(k_seed<PER>, static_cast<unsigned>(grid), kSeedBlock, smem, st, b);
    t_pdl = prev;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_seed(const SeedArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (a.count >= (int64_t(1) << 22)) return launch_seed_per<128>(a, st);
    if (a.count >= (int64_t(1) << 18) || a.planes) return launch_seed_per<32>(a, st);  // planes: whole groups
    return launch_seed_per<8>(a, st);
}

cudaError_t launch_neg_log1m(const uint32_t* k, int64_t n, double* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t per_block = static_cast<int64_t>(kLogHookBlock) * kExpoB;
    k_neg_log1m<<<static_cast<unsigned>((n + per_block - 1) / per_block), kLogHookBlock, 0, st>>>(k, n, out);
    return cudaGetLastError();
}

cudaError_t launch_taus_stream(const uint32_t* powers, Taus seed, int64_t n, uint32_t* out, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t threads = (n + kTausPerThread - 1) / kTausPerThread;
    const int block = 128;
    k_taus<<<static_cast<unsigned>((threads + block - 1) / block), block, 0, st>>>(powers, seed, n, out);
    return cudaGetLastError();
}

// Calls f(std::integral_constant<int, div>) for a RepArgs::div value.
template <class F>
void by_div(int div, F&& f) {
    if (div == kDivPow2)
        f(std::integral_constant<int, kDivPow2>{});
    else if (div == kDivRcp)
        f(std::integral_constant<int, kDivRcp>{});
    else
        f(std::integral_constant<int, kDivIeee>{});
}

cudaError_t launch_wlp(int model, const RepArgs& a, const uint32_t* lane_tab, const uint32_t* uni_tab,
                       int64_t lane_units, int grid, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const bool count = a.hw != nullptr;
    if (model == 1) {
        auto go = [&](auto kernel) { launch_ex(kernel, grid, kMm1Block, kMm1Smem, st, a, lane_tab, uni_tab); };
        by_div(a.div, [&](auto d) {
            constexpr int D = decltype(d)::value;
            count ? go(k_wlp_mm1<D, true>) : go(k_wlp_mm1<D, false>);
        });
    } else {
        auto go = [&](auto kernel) { launch_ex(kernel, grid, kWlpBlock, kLaneTabWords * 4, st, a, lane_tab, lane_units); };
        if (model == 0)
            count ? go(k_wlp_lanes<0, true>) : go(k_wlp_lanes<0, false>);
        else
            count ? go(k_wlp_lanes<2, true>) : go(k_wlp_lanes<2, false>);
    }
    return cudaGetLastError();
}

template <int MODEL, bool WIDE>
void launch_wlp_pipe_m(const RepArgs& a, const PipeSched& s, const uint32_t* wrap_tab, int grid, cudaStream_t st) {
    auto go = [&](auto kernel) { launch_ex(kernel, grid, kWlpBlock, 0, st, a, s, wrap_tab); };
    if (s.S == 2)
        go(k_wlp_pipe<MODEL, WIDE, 2, true>);
    else if (s.S == 4)
        go(k_wlp_pipe<MODEL, WIDE, 4, true>);
    else if (s.S == 8)
        go(k_wlp_pipe<MODEL, WIDE, 8, true>);
    else if (s.S == 16)
        go(k_wlp_pipe<MODEL, WIDE, 16, true>);
    else if (wrap_tab)
        go(k_wlp_pipe<MODEL, WIDE, 32, true>);
    else
        go(k_wlp_pipe<MODEL, WIDE, 32, false>);
}

cudaError_t launch_wlp_pipe(int model, const RepArgs& a, const PipeSched& s, const uint32_t* wrap_tab, int grid,
                            cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (s.S != 32 && (!wrap_tab || (s.S != 16 && s.S != 8 && s.S != 4 && s.S != 2))) return cudaErrorInvalidValue;
    // 32-bit sums hold pi's hits (< n) and the walk's raw q sum (|sum| <= 12 n)
    const bool wide = a.n >= (int64_t(1) << 27) || a.count >= (int64_t(1) << 31);
    if (model == 0)
        wide ? launch_wlp_pipe_m<0, true>(a, s, wrap_tab, grid, st) : launch_wlp_pipe_m<0, false>(a, s, wrap_tab, grid, st);
    else
        wide ? launch_wlp_pipe_m<2, true>(a, s, wrap_tab, grid, st) : launch_wlp_pipe_m<2, false>(a, s, wrap_tab, grid, st);
    return cudaGetLastError();
}

cudaError_t launch_wlp_mm1_pipe(const RepArgs& a, const PipeSched& ps, int grid, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (ps.G == kPanT && ps.tail == 0 && ps.qb > 0) {  // whole panels at every step
        const bool mu_one = a.div == kDivPow2 && a.mu == 1.0;
        auto go = [&](auto kernel) {
            allow_smem(kernel, kMm1Pipe2Smem);
            launch_ex(kernel, grid, kMm1Block, kMm1Pipe2Smem, st, a, ps);
        };
        auto by_s = [&](auto d) {
            constexpr int D = decltype(d)::value;
            if (ps.S == 2)
                go(k_wlp_mm1_pipe<D, 2>);
            else if (ps.S == 4)
                go(k_wlp_mm1_pipe<D, 4>);
            else if (ps.S == 8)
                go(k_wlp_mm1_pipe<D, 8>);
            else if (ps.S == 16)
                go(k_wlp_mm1_pipe<D, 16>);
            else
                go(k_wlp_mm1_pipe<D, 32>);
        };
        if (mu_one)
            by_s(std::integral_constant<int, kDivPow2One>{});
        else
            by_div(a.div, by_s);
        return cudaGetLastError();
    }
    if (ps.S != 32) return cudaErrorInvalidValue;
    const bool exact = !(ps.G == kPanT && ps.tail == 0);  // some chunk ends inside a panel
    auto go = [&](auto kernel) { launch_ex(kernel, grid, kMm1Block, kMm1PipeSmem, st, a, ps); };
    by_div(a.div, [&](auto d) {
        constexpr int D = decltype(d)::value;
        exact ? go(k_wlp_mm1_pipe_ragged<D, true>) : go(k_wlp_mm1_pipe_ragged<D, false>);
    });
    return cudaGetLastError();
}

int wlp_mm1_pipe_blocks_per_sm() {
    int nb = 0;
    allow_smem(k_wlp_mm1_pipe_ragged<kDivIeee, true>, kMm1PipeSmem);
    allow_smem(k_wlp_mm1_pipe_ragged<kDivIeee, false>, kMm1PipeSmem);
    allow_smem(k_wlp_mm1_pipe_ragged<kDivPow2, true>, kMm1PipeSmem);
    allow_smem(k_wlp_mm1_pipe_ragged<kDivPow2, false>, kMm1PipeSmem);
    allow_smem(k_wlp_mm1_pipe_ragged<kDivRcp, true>, kMm1PipeSmem);
    allow_smem(k_wlp_mm1_pipe_ragged<kDivRcp, false>, kMm1PipeSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_mm1_pipe_ragged<kDivIeee, true>, kMm1Block, kMm1PipeSmem);
    int nb2 = 0;
    allow_smem(k_wlp_mm1_pipe<kDivIeee, 32>, kMm1Pipe2Smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, k_wlp_mm1_pipe<kDivIeee, 32>, kMm1Block, kMm1Pipe2Smem);
    nb = nb2 < nb ? nb2 : nb;  // one grid size serves both
    return nb < 1 ? 1 : nb;
}

int wlp_pipe_blocks_per_sm() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_pipe<0, true, 32, true>, kWlpBlock, 0);
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_tlp(int model, const RepArgs& a, int tlp_block, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int64_t block = a.count < tlp_block ? a.count : tlp_block;
    const int64_t grid = (a.count + block - 1) / block;
    const dim3 g(static_cast<unsigned>(grid)), b(static_cast<unsigned>(block));
    const bool count = a.hw != nullptr;
    switch (model) {
        case 0:
            if (count)
                launch_ex(k_tlp<0, true>, g, b, 0, st, a);
            else
                launch_ex(k_tlp<0, false>, g, b, 0, st, a);
            break;
        case 1: {
            const size_t smem = tlp_mm1_panel_smem(static_cast<int>(block));
            auto go = [&](auto kernel) {
                allow_smem(kernel, smem);
                launch_ex(kernel, g, b, smem, st, a);
            };
            by_div(a.div, [&](auto d) {
                constexpr int D = decltype(d)::value;
                if (block <= 256)
                    count ? go(k_tlp_mm1<D, true, true>) : go(k_tlp_mm1<D, false, true>);
                else
                    count ? go(k_tlp_mm1<D, true, false>) : go(k_tlp_mm1<D, false, false>);
            });
            break;
        }
        default:
            if (count)
                launch_ex(k_tlp<2, true>, g, b, 0, st, a);
            else
                launch_ex(k_tlp<2, false>, g, b, 0, st, a);
            break;
    }
    return cudaGetLastError();
}

cudaError_t launch_tlp_walk_bs(const RepArgs& a, cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    const int64_t threads = (a.count + 31) / 32;
    const int64_t grid = (threads + kBsBlock - 1) / kBsBlock;
    const size_t smem = a.n > kBsFlushBlocks * 16 ? kBsBlock * 33 * sizeof(int32_t) : 0;
    launch_ex(k_tlp_walk_bs, static_cast<unsigned>(grid), kBsBlock, smem, st, a);
    return cudaGetLastError();
}

cudaError_t launch_wlp_walk_bs_pipe(const RepArgs& a, uint32_t* bseeds, const PipeSched& s, const uint32_t* wrap_tab,
                                    int grid, cudaStream_t st, bool planes_ready) {
    if (a.count <= 0) return cudaSuccess;
    if (s.S != 32 && s.S != 16 && s.S != 8 && s.S != 4) return cudaErrorInvalidValue;
    const int64_t groups = (a.count + 31) / 32;
    if (!planes_ready)  // else the seeding kernel wrote them (SeedArgs::planes)
        launch_ex(k_bs_seeds, static_cast<unsigned>((groups + kBsBlock - 1) / kBsBlock), kBsBlock, 0, st, a, groups,
                  bseeds);
    auto go = [&](auto kernel) { launch_ex(kernel, grid, kBsPipeBlock, 0, st, a, bseeds, groups, s, wrap_tab); };
    if (wrap_tab) {
        if (s.S == 4)
            go(k_wlp_walk_bs_pipe<4, true>);
        else if (s.S == 8)
            go(k_wlp_walk_bs_pipe<8, true>);
        else if (s.S == 16)
            go(k_wlp_walk_bs_pipe<16, true>);
        else
            go(k_wlp_walk_bs_pipe<32, true>);
    } else {
        if (s.S == 4)
            go(k_wlp_walk_bs_pipe<4, false>);
        else if (s.S == 8)
            go(k_wlp_walk_bs_pipe<8, false>);
        else if (s.S == 16)
            go(k_wlp_walk_bs_pipe<16, false>);
        else
            go(k_wlp_walk_bs_pipe<32, false>);
    }
    return cudaGetLastError();
}

cudaError_t launch_wlp_walk_bs_lanes(const RepArgs& a, const uint32_t* lane_tab, int64_t K, int grid,
                                     cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    allow_smem(k_wlp_walk_bs_lanes, kLaneTabWords * 4);
    launch_ex(k_wlp_walk_bs_lanes, grid, kBsLanesBlock, kLaneTabWords * 4, st, a, lane_tab, K);
    return cudaGetLastError();
}

int wlp_walk_bs_pipe_blocks_per_sm() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_wlp_walk_bs_pipe<8, true>, kBsPipeBlock, 0);
    return nb < 1 ? 1 : nb;
}

int plan_blocks_per_sm(int model) {
    int nb = 0;
    if (model == 1) {
        allow_smem(k_plan_mm1, kMm1Smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_plan_mm1, kMm1Block, kMm1Smem);
    } else {
        const size_t smem = (kLaneTabWords + kUniTabWords) * 4;
        allow_smem(k_plan_lanes<0>, smem);
        allow_smem(k_plan_lanes<2>, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_plan_lanes<0>, kWlpBlock, smem);
    }
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_seed_jobs(const uint32_t* powers, const SeedJob* d_jobs, int n_jobs, int64_t total_blocks,
                             int64_t total_slots, uint32_t* out, void* specials, int64_t special_cap,
                             unsigned long long* n_special, cudaStream_t st, unsigned long long* zero_a,
                             unsigned int* done, unsigned long long* report) {
    if (total_blocks <= 0) return cudaSuccess;
    const size_t smem = seed_stage_words(kSeedJobPer) * 4;
    allow_smem(k_seed_jobs, smem);
    const bool prev = t_pdl;
    t_pdl = true;  // (as launch_seed_per: it waits for the previous kernels before touching memory)
    const cudaError_t e = launch_ex(k_seed_jobs, static_cast<unsigned>(total_blocks), kSeedBlock, smem, st, powers,
                                    d_jobs, n_jobs, out, total_slots, static_cast<SpecialRec*>(specials), special_cap,
                                    n_special, zero_a, done, report);
    t_pdl = prev;
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

cudaError_t launch_plan(int model, int mode, const PlanArgs& a, const uint32_t* lane_tab, const uint32_t* uni_tab,
                        const uint32_t* mm1_lane, const uint32_t* mm1_skip, int grid, int tlp_block,
                        cudaStream_t st) {
    if (a.count <= 0) return cudaSuccess;
    if (mode == 1) {  // TLP
        const int64_t block = a.count < tlp_block ? a.count : tlp_block;
        const dim3 g(static_cast<unsigned>((a.count + block - 1) / block)), b(static_cast<unsigned>(block));
        if (model == 1) {
            const size_t smem = tlp_mm1_smem(static_cast<int>(block));
            allow_smem(k_plan_tlp_mm1, smem);
            launch_ex(k_plan_tlp_mm1, g, b, smem, st, a);
        } else if (model == 0) {
            launch_ex(k_plan_tlp<0>, g, b, 0, st, a);
        } else {
            launch_ex(k_plan_tlp<2>, g, b, 0, st, a);
        }
        return cudaGetLastError();
    }
    if (model == 1) {
        launch_ex(k_plan_mm1, grid, kMm1Block, kMm1Smem, st, a, mm1_lane, mm1_skip);
    } else {
        const size_t smem = (kLaneTabWords + kUniTabWords) * 4;
        if (model == 0)
            launch_ex(k_plan_lanes<0>, grid, kWlpBlock, smem, st, a, lane_tab, uni_tab);
        else
            launch_ex(k_plan_lanes<2>, grid, kWlpBlock, smem, st, a, lane_tab, uni_tab);
    }
    return cudaGetLastError();
}

cudaError_t launch_stats(const double* x, int64_t n, int pass, double center, double* partials, int grid,
                         cudaStream_t st, bool reference_order, const double* center_dev) {
    if (reference_order && n > kStatsSeqMax) {
        k_stats_seq<<<1, kStatsBlock, 0, st>>>(x, n, pass, center, partials, center_dev);
        return cudaGetLastError();
    }
    if (n <= kStatsSeqMax) grid = 1;
    k_stats<<<grid, kStatsBlock, 0, st>>>(x, n, pass, center, partials, center_dev);
    return cudaGetLastError();
}

cudaError_t launch_stats_fold(const double* partials, int used, int64_t n, double* meta, cudaStream_t st) {
    k_stats_fold<<<1, 128, 0, st>>>(partials, used, n, meta);
    return cudaGetLastError();
}

}  // namespace wlp
