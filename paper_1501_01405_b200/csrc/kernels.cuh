// Launch interface of the sm_100a kernels (implemented in kernels.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "taus88.cuh"

namespace wlp {

// How the mm1 kernels divide a log by a rate (models.hpp:67,75); all three give IEEE
// e / rate bit for bit (kernels.cu scale()). kDivPow2: rate = 2^k, inv = 1/rate exactly;
// kDivRcp: inv = RN(1/rate), rate in [2^-900, 2^900]; kDivIeee: anything else.
// kDivPow2One: lambda = 2^k and mu = 1 (the reference's default service rate): the
// services' division is the identity, one FP64 operation fewer per client.
enum : int { kDivIeee = 0, kDivPow2 = 1, kDivRcp = 2, kDivPow2One = 3 };

// Replication-kernel arguments shared by every model/mapping.
struct RepArgs {
    const uint32_t* seeds;  // SoA: s1[count], s2[count], s3[count]
    int64_t count;          // replications in this launch
    int64_t n;              // units per replication (draws / clients / steps)
    int64_t chunks;         // walk
    double lambda, mu;      // mm1 rates
    double inv_lambda, inv_mu;  // reciprocals for `div` (0 under kDivIeee)
    int div = kDivIeee;
    double* out0;
    double* out1;
    double* out2;
    // optional host mirrors (mapped pinned host memory, device-accessible): every output
    // is also stored there as it is produced, so results reach the host during the run
    // instead of by a copy after it (the device arrays still feed the statistics)
    double* h0 = nullptr;
    double* h1 = nullptr;
    double* h2 = nullptr;
    // WLP: warps take `grab` consecutive replications at a time from *next (zeroed
    // before launch), so warps the arbiter favours do not leave a tail behind them
    unsigned long long* next = nullptr;
    int grab = 1;
    // Hardware counters (SimReport, device.hpp:62-71): when non-null, the kernels run an
    // instrumented variant that adds, per warp, [0] the warp-level branch splits of the
    // model's data-dependent `if`s (the reference's event definition,
    // warp_exec.cpp:272-284), [1] global load and [2] global store warp-instructions.
    unsigned long long* hw = nullptr;
    // mm1 WLP with segment chaining: replications with lambda >= serial_rho * mu run the
    // heavy-traffic ordered loop on lane 0 instead (0.75 by default, runtime.cu)
    double serial_rho = 2.0;
    // mm1 pipeline: near-one list entries used per panel (a power of two <= the 128 the
    // shared memory holds; smaller only as a test hook, to exercise the overflow redo)
    uint32_t near_cap = 128;
};

// Per-warp instrumentation tally (identical in every lane; the leader flushes it), and the
// warp's clock64 at kernel entry (set by the instrumented kernels).
struct HwTally {
    unsigned div = 0, ld = 0, st = 0;
    unsigned splits = 0;  // implementation splits (lane-divergent loops), beyond the model's `div`
    long long t0 = 0;
};

// Layout of RepArgs::hw: [0] model-branch events, [1] loads, [2] stores, [3] implementation
// splits, then per SM the earliest warp start and the latest warp end in that SM's clock64
// (the host takes max over SMs of end - start: the kernel's makespan in SM cycles).
constexpr int kHwMaxSms = 256;
constexpr int kHwClk = 4;
constexpr int kHwWords = kHwClk + 2 * kHwMaxSms;

// Rotating schedule of the warp pipelines (k_wlp_pipe, k_wlp_walk_bs_pipe,
// k_wlp_mm1_pipe). A replication's units are split into S chunks, one per lane of an
// S-lane pipeline (S = 32: the whole warp). At pipeline step t every lane runs the same
// number of units,
//   L(t) = G * (qb + [t % S < rb]) + [t % S == S-1] * tail,   n = G * (S qb + rb) + tail,
// so any S consecutive steps sum to n: a replication entering at lane 0 at any step is
// covered exactly by its S chunks, and no lane waits on a longer chunk of another (a
// fixed split ceil(n/32) leaves lane 31 short: 1000 units = 31 x 32 + 8 idles 2.3 %).
// G is the kernel's unrolled block (8 units, 8 walk steps for the bitsliced counters).
struct PipeSched {
    int G = 1, S = 32, qb = 0, rb = 0, tail = 0;
};
__host__ __device__ inline PipeSched pipe_sched(int64_t n, int G, int S = 32) {
    PipeSched s;
    s.G = G;
    s.S = S;
    const int64_t nb = n / G;
    s.qb = static_cast<int>(nb / S);
    s.rb = static_cast<int>(nb % S);
    s.tail = static_cast<int>(n % G);
    return s;
}
__host__ __device__ inline int pipe_units(const PipeSched& s, int phase) {
    return s.G * (s.qb + (phase < s.rb ? 1 : 0)) + (phase == s.S - 1 ? s.tail : 0);
}
// Units of chunks 0..k-1 of a replication that would have entered at step -k (the steps
// -k..-1, i.e. phases S-k..S-1): where the wrapped pipelines start chunk k at step 0.
__host__ __device__ inline int64_t pipe_wrap_units(const PipeSched& s, int k) {
    const int extra = s.rb - (s.S - k);
    return static_cast<int64_t>(s.G) * (static_cast<int64_t>(k) * s.qb + (extra > 0 ? extra : 0)) +
           (k > 0 ? s.tail : 0);
}
// Replications per warp reserved for the wrap: S - 1 per S-lane pipeline (lanes 1..S-1
// of the first step).
__host__ __device__ constexpr int pipe_wrap_per_warp(int S) { return 32 - 32 / S; }
constexpr int kWrap = 31;  // S = 32

// Seeding: stream slots [slot_begin, slot_begin+count) of a run.
struct SeedArgs {
    const uint32_t* powers;  // [64][3][8][16] binary powers of the taus88 step as nibble tables
    Taus master;
    int64_t slot_begin, count;
    const int64_t* rejected;  // sorted global candidate indices
    int64_t n_rejected;
    uint32_t* out;  // SoA: plane p of slot i at out[p*stride + out_off + i]
    void* specials;  // wlp_special[cap]
    int64_t special_cap;
    unsigned long long* n_special;
    int64_t out_off = 0;
    int64_t stride = 0;  // 0: count
    // optional: the walk's bit planes of each group of 32 slots (88 live words per group,
    // the layout k_bs_seeds writes), so the bitsliced pipeline needs no separate pass
    uint32_t* planes = nullptr;  // (when set, the SoA keys are not written: the pipeline reads the planes alone)
    // optional words the seeding zeroes (block 0, before the model launch that follows):
    // the next run's specials count and the model's work counter (no memset launches)
    unsigned long long* zero_a = nullptr;
    unsigned long long* zero_b = nullptr;
    int stage_powers = 0;  // (set by launch_seed) binary powers staged in shared memory
    // optional: the last block to finish stores the final specials count to `report`
    // (mapped pinned host memory: the host reads it after a stream sync, no copy launch)
    // and rearms `done` (a block counter, zero between launches)
    unsigned int* done = nullptr;
    unsigned long long* report = nullptr;
};

// Experimental plan (BASELINE config 5): many factor-level sets in one launch.
struct SetParam {
    int64_t off;     // first replication of the set in the concatenated launch
    int64_t n;       // units per replication
    int64_t chunks;  // walk
    double lambda, mu, inv_lambda, inv_mu;
    int div;
};

struct PlanArgs {
    const uint32_t* seeds;  // SoA over all replications of all sets
    int64_t count;          // total replications
    const SetParam* sets;
    int n_sets;
    double* out0;
    double* out1;
    double* out2;
    unsigned long long* next;  // dynamic work counter (zeroed before launch)
    double serial_rho = 2.0;   // as RepArgs::serial_rho, per set
    int tlp_div = kDivIeee;    // TLP plan: kDivRcp when every set allows it
};

// Batched seeding of many independent random_spacing runs (one per set).
struct SeedJob {
    Taus master;
    uint32_t pad;
    int64_t count;    // slots of this job
    int64_t out_off;  // first slot in the concatenated SoA
    int64_t block0;   // first block of this job in the launch
};

constexpr int kPlanT = 32;          // pi/walk plan kernels: units per lane per panel
constexpr int kWlpBlock = 512;     // pi / walk WLP block (16 warps; 3 blocks = 48 warps per SM)
constexpr int kMm1Block = 256;     // mm1 WLP block (8 warps)
constexpr int kMm1PanelT = 8;      // mm1: clients per lane per panel
constexpr int kSeedBlock = 32;     // seeding threads per block (slots per thread by run size)
constexpr int kSeedJobPer = 8;     // slots per thread of the plan seeding (small runs)

// Layout of wlp_special (include/wlp_b200.h).
struct SpecialRec {
    int64_t index;
    uint32_t s1, s2, s3, pad;
};

// Resident blocks per SM for each WLP kernel (occupancy API), for persistent grids.
int wlp_blocks_per_sm(int model);
// Resident blocks per SM of the TLP kernel at a given block size.
int tlp_blocks_per_sm(int model, int block);

cudaError_t launch_seed(const SeedArgs& a, cudaStream_t st);
// Model launches on this thread use programmatic dependent launch (overlap with the
// seeding kernel they follow) while set; off for launches bracketed by timing events.
void set_pdl_launch(bool on);
cudaError_t launch_neg_log1m(const uint32_t* k, int64_t n, double* out, cudaStream_t st);
cudaError_t launch_taus_stream(const uint32_t* powers, Taus seed, int64_t n, uint32_t* out,
                               cudaStream_t st);
// WLP: persistent grid of `grid` blocks; lane_tab = lane-start nibble tables (device),
// uni_tab = panel-skip table (mm1 only).
cudaError_t launch_wlp(int model, const RepArgs& a, const uint32_t* lane_tab,
                       const uint32_t* uni_tab, int64_t lane_units, int grid, cudaStream_t st);
// WLP as a warp pipeline (pi / walk): no per-replication lane jumps; s.S lanes per
// replication (32, 16 or 8). wrap_tab: lane tables of the distances
// 2 * pipe_wrap_units(s, lane % S) draws (null: no wrap, S = 32 only; with it a.count >=
// pipe_wrap_per_warp(S) * warps).
cudaError_t launch_wlp_pipe(int model, const RepArgs& a, const PipeSched& s, const uint32_t* wrap_tab, int grid,
                            cudaStream_t st);
int wlp_pipe_blocks_per_sm();
// mm1 WLP as a warp pipeline on a rotating schedule (s.S = 32; G = 8 clients, a panel, or 1).
cudaError_t launch_wlp_mm1_pipe(const RepArgs& a, const PipeSched& s, int grid, cudaStream_t st);
int wlp_mm1_pipe_blocks_per_sm();
// TLP: thread per replication, block = tlp_block, grid = ceil(count / tlp_block).
cudaError_t launch_tlp(int model, const RepArgs& a, int tlp_block, cudaStream_t st);
// Walk, bitsliced thread per 32 replications (needs n < 2^31).
cudaError_t launch_tlp_walk_bs(const RepArgs& a, cudaStream_t st);
// Walk WLP, bitsliced warp pipeline (groups of 32 replications; n < 65536) on the
// rotating schedule s (S = 32). bseeds: scratch of 88 words per group; a.next zeroed,
// a.grab groups per grab. wrap_tab: lane tables of 2 * pipe_wrap_units(s, lane) draws
// (null: no wrap; with it groups >= kWrap * warps).
cudaError_t launch_wlp_walk_bs_pipe(const RepArgs& a, uint32_t* bseeds, const PipeSched& s, const uint32_t* wrap_tab,
                                    int grid, cudaStream_t st, bool planes_ready = false);
int wlp_walk_bs_pipe_blocks_per_sm();
// Walk WLP, bitsliced lane chunks: a warp per group of 32 replications (K < 65536; lane
// jump table of stride 2K draws; a.next zeroed, a.grab groups per grab).
cudaError_t launch_wlp_walk_bs_lanes(const RepArgs& a, const uint32_t* lane_tab, int64_t K, int grid, cudaStream_t st);
constexpr int kBsPipeBlock = 64;  // threads per block of the bitsliced walk pipeline
// Plan: batched seeding (specials carry the job index in `pad`), then one model launch.
cudaError_t launch_seed_jobs(const uint32_t* powers, const SeedJob* d_jobs, int n_jobs, int64_t total_blocks,
                             int64_t total_slots, uint32_t* out, void* specials, int64_t special_cap,
                             unsigned long long* n_special, cudaStream_t st, unsigned long long* zero_a = nullptr,
                             unsigned int* done = nullptr, unsigned long long* report = nullptr);
// grid: persistent blocks for WLP; TLP uses `tlp_block` threads per block over all replications.
cudaError_t launch_plan(int model, int mode, const PlanArgs& a, const uint32_t* lane_tab, const uint32_t* uni_tab,
                        const uint32_t* mm1_lane, const uint32_t* mm1_skip, int grid, int tlp_block,
                        cudaStream_t st);
int plan_blocks_per_sm(int model);

// The reference's *_replication_u bodies over caller-given uniforms (uniforms.cu):
// replication r reads u[r*2n, r*2n + 2n), one thread per replication.
struct UniArgs {
    int model;
    const double* u;
    int64_t count, n, chunks;
    double lambda, mu;
    double* out0;
    double* out1;
    double* out2;
};
cudaError_t launch_uniform_reps(const UniArgs& a, cudaStream_t st);
// exponential_from_u (rng.cpp:58-61) over u[n]; *bad (init ~0) gets the lowest index
// with u outside [0, 1).
cudaError_t launch_exponentials(const double* u, int64_t n, double rate, double* out, unsigned long long* bad,
                                cudaStream_t st);

// Stats: per-block partials [grid][2] (sum_hi, sum_lo or ss_hi, ss_lo) of x (pass 1
// about 0, pass 2 about `center`). n <= 256 or reference_order: one partial, the
// reference's sequential sum (models.cpp:104-109) bit for bit.
cudaError_t launch_stats(const double* x, int64_t n, int pass, double center, double* partials,
                         int grid, cudaStream_t st, bool reference_order = false,
                         const double* center_dev = nullptr);
// Folds pass-1 partials [used][2] into meta = {hi, lo, mean} on the device (the host's
// stats_device merge, bit for bit), so pass 2 (center_dev = meta + 2) needs no round trip.
cudaError_t launch_stats_fold(const double* partials, int used, int64_t n, double* meta, cudaStream_t st);

}  // namespace wlp
