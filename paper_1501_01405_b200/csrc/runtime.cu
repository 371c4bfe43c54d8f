// C-ABI implementation (include/wlp_b200.h): per-device context and scratch, the exact
// random-spacing fixpoint, model dispatch, device statistics, and the host-side
// reference utilities (validate_params, plan_launch, rng_state_from_seed,
// inverse_normal_cdf) the drop-in API needs.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/wlp_b200.h"
#include "glibc_log.cuh"
#include "jump.hpp"
#include "ir_interp.cuh"
#include "kernels.cuh"

static_assert(sizeof(wlp_special) == sizeof(wlp::SpecialRec), "wlp_special layout");

namespace wlp {
namespace {

thread_local std::string g_err;
thread_local bool g_hw_counters = false;  // wlp_set_hw_counters
thread_local int g_wlp_variant = 0;       // wlp_set_wlp_variant: 0 auto, 1 lane jumps, 2 pipeline
thread_local const char* g_last_kernel = "";  // wlp_last_kernel
thread_local int g_pipe_lanes = 0;       // wlp_set_pipe_lanes: 0 auto, else 8 / 16 / 32
thread_local uint32_t g_near_cap = 128;  // wlp_debug_set_near_cap (test hook)
thread_local int g_tlp_variant = 0;       // wlp_set_tlp_variant: 0 auto, 1 per replication, 2 bitsliced walk
thread_local int g_stats_order = 0;       // wlp_set_stats_order: 0 accurate (double-double), 1 reference

// mm1 WLP segment chaining hands replications with lambda >= rho * mu to the serial
// heavy-traffic loop; WLP_MM1_SERIAL_RHO overrides the measured default.
double mm1_serial_rho() {
    static const double rho = [] {
        const char* e = std::getenv("WLP_MM1_SERIAL_RHO");
        return e ? std::atof(e) : 0.75;
    }();
    return rho;
}

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define WLP_CUDA(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(WLP_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e_) +    \
                                       " at " #expr);                                        \
    } while (0)

#define WLP_TRY(expr)            \
    do {                         \
        int s_ = (expr);         \
        if (s_ != WLP_OK) return s_; \
    } while (0)

template <class T>
struct DevBuf {
    T* p = nullptr;
    int64_t cap = 0;
    cudaError_t ensure(int64_t n) {
        if (n <= cap) return cudaSuccess;
        release();
        const cudaError_t e = cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T));
        if (e == cudaSuccess)
            cap = n;
        else
            p = nullptr;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

constexpr int64_t kSpecialCap = 4096;
constexpr int kMaxLaneTabs = 64;

constexpr unsigned long long kCountPending = ~0ull;  // mapped count word before the seeding stores it

struct DevCtx {
    int dev = 0;
    int sms = 0;
    int clock_khz = 0;
    int wlp_bps[3] = {1, 1, 1};
    int pipe_bps = 1, mm1_pipe_bps = 1, bs_pipe_bps = 1;
    std::mutex mu;
    bool ready = false;
    DevBuf<uint32_t> powers;
    std::map<uint64_t, DevBuf<uint32_t>> lane_tabs;  // by lane jump stride (draws)
    std::map<std::tuple<int, int, int, int>, DevBuf<uint32_t>> wrap_tabs;  // by pipeline schedule
    DevBuf<uint32_t> mm1_lane, mm1_skip;
    DevBuf<uint32_t> seeds, in_seeds;
    DevBuf<uint32_t> bseeds;  // walk bitsliced pipeline: group seed bit planes
    const uint32_t* planes_of = nullptr;  // bseeds holds the planes of these seeds ...
    int64_t planes_count = -1;            // ... (count), written by the last seed_async
    DevBuf<double> outs, partials, stats_in;
    DevBuf<SpecialRec> specials;
    DevBuf<unsigned long long> counter;  // [0] special candidates of the last seeding, [1] its grab counter
    // counter[0], [1]: the specials counts of alternate seedings (each seeding zeroes the
    // other for the next one, so no memset precedes it); [2]: the grab counter of the model
    // launch behind a seeding (zeroed by that seeding); [3], [4]: the plan's specials count
    // (cleared by the plan seeding's last block) and grab counter (zeroed by the seeding)
    int spec_slot = 0;                   // the next seeding counts its specials in counter[spec_slot]
    int spec_read = 0;                   // the slot read_specials reads
    bool work_zeroed = false;            // counter[2] was cleared by the seeding just launched
    bool pdl_next = false;               // the next model launch directly follows a seeding kernel
    double* hm[3] = {nullptr, nullptr, nullptr};  // host mirrors for the next model launch
    bool time_model = false;  // model_async records ev0 right before its launch
    unsigned long long* h_counter = nullptr;  // pinned host word for the specials count readback
    unsigned long long* h_mapped = nullptr;   // mapped pinned word the seeding stores the count to
    unsigned long long* d_mapped = nullptr;   // (its device alias)
    bool spec_mapped = false;                 // the last seeding reports through h_mapped
    DevBuf<unsigned int> seed_done;           // the seeding's finished-block counter
    unsigned char* h_stage = nullptr;         // pinned staging of small uploads (plan tables)
    size_t h_stage_cap = 0;
    DevBuf<unsigned char> plan_blob;          // the plan's SeedJob[] then SetParam[]
    std::vector<unsigned char> plan_blob_host;  // ... as last uploaded (skip re-uploads of the same plan)
    const unsigned char* plan_blob_dev = nullptr;
    DevBuf<int64_t> rejected;
    DevBuf<unsigned long long> work;
    DevBuf<unsigned long long> hw;  // instrumentation tallies [div, ld, st]
    DevBuf<SeedJob> jobs;
    DevBuf<SetParam> setp;
    DevBuf<uint32_t> plan_lane, plan_skip;
    int plan_bps[3] = {1, 1, 1};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t done = nullptr;  // end of the last library work (cross-stream ordering)
    cudaStream_t last_stream = nullptr;
    bool last_used = false;
};

std::mutex g_ctx_mu;
std::map<int, std::unique_ptr<DevCtx>> g_ctx;

int upload_u32(DevBuf<uint32_t>& b, const std::vector<uint32_t>& v) {
    WLP_CUDA(b.ensure(static_cast<int64_t>(v.size())));
    WLP_CUDA(cudaMemcpy(b.p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    return WLP_OK;
}

int ctx_init(DevCtx& c) {
    if (c.ready) return WLP_OK;
    WLP_CUDA(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, c.dev));
    if (cudaDeviceGetAttribute(&c.clock_khz, cudaDevAttrClockRate, c.dev) != cudaSuccess) c.clock_khz = 0;
    WLP_TRY(upload_u32(c.powers, flat_nibble_powers()));
    WLP_TRY(upload_u32(c.mm1_lane, lane_tables(2ull * kMm1PanelT)));
    WLP_TRY(upload_u32(c.mm1_skip, uniform_table(2ull * 31 * kMm1PanelT)));
    WLP_TRY(upload_u32(c.plan_lane, lane_tables(2ull * kPlanT)));
    WLP_TRY(upload_u32(c.plan_skip, uniform_table(2ull * 31 * kPlanT)));
    c.pipe_bps = wlp_pipe_blocks_per_sm();
    c.mm1_pipe_bps = wlp_mm1_pipe_blocks_per_sm();
    c.bs_pipe_bps = wlp_walk_bs_pipe_blocks_per_sm();
    for (int m = 0; m < 3; ++m) {
        c.wlp_bps[m] = wlp_blocks_per_sm(m);
        c.plan_bps[m] = plan_blocks_per_sm(m);
    }
    WLP_CUDA(c.specials.ensure(kSpecialCap));
    WLP_CUDA(c.counter.ensure(5));
    WLP_CUDA(cudaMemset(c.counter.p, 0, 5 * sizeof(unsigned long long)));
    WLP_CUDA(c.work.ensure(1));
    WLP_CUDA(cudaMallocHost(&c.h_counter, sizeof(unsigned long long)));
    WLP_CUDA(cudaHostAlloc(&c.h_mapped, sizeof(unsigned long long), cudaHostAllocMapped));
    WLP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c.d_mapped), c.h_mapped, 0));
    WLP_CUDA(c.seed_done.ensure(1));
    WLP_CUDA(cudaMemset(c.seed_done.p, 0, sizeof(unsigned int)));
    WLP_CUDA(c.hw.ensure(kHwWords));
    WLP_CUDA(cudaEventCreate(&c.ev0));
    WLP_CUDA(cudaEventCreate(&c.ev1));
    WLP_CUDA(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming));
    WLP_CUDA(cudaGetLastError());
    c.ready = true;
    return WLP_OK;
}

// Context of the calling thread's current device, locked.
int acquire(DevCtx*& out, std::unique_lock<std::mutex>& lk) {
    // the device count is asked once per process (the call costs ~1 us on every run)
    static const std::pair<cudaError_t, int> count = [] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        return std::make_pair(e, n);
    }();
    if (count.first != cudaSuccess || count.second == 0)
        return fail(WLP_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(count.first));
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(WLP_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    DevCtx* c;
    {
        std::lock_guard<std::mutex> g(g_ctx_mu);
        auto& slot = g_ctx[dev];
        if (!slot) {
            slot = std::make_unique<DevCtx>();
            slot->dev = dev;
        }
        c = slot.get();
    }
    lk = std::unique_lock<std::mutex>(c->mu);
    WLP_TRY(ctx_init(*c));
    out = c;
    return WLP_OK;
}

// The device scratch (seed keys, work counter, specials) is shared by every call on a
// device. Calls on one stream are ordered by the stream; a call on a different stream
// first waits for the last library work, and every call records its end.
// (The event is recorded at the end of every call, on that call's stream: recording it
// lazily on the previous stream when the stream changes would touch streams callers may
// have destroyed meanwhile, as wlp_run_devices' worker streams are.)
struct StreamOrder {
    DevCtx& c;
    cudaStream_t st;
    StreamOrder(DevCtx& ctx, cudaStream_t s) : c(ctx), st(s) {
        if (c.last_used && c.last_stream != st) cudaStreamWaitEvent(st, c.done, 0);
    }
    ~StreamOrder() {
        cudaEventRecord(c.done, st);
        c.last_stream = st;
        c.last_used = true;
    }
};

int64_t units_of(int model, const wlp_params& p) {
    return model == WLP_MODEL_PI ? p.draws : model == WLP_MODEL_MM1 ? p.clients : p.steps;
}

// 1/rate when rate = 2^k (|k| <= 512): then x/rate == x*(1/rate) exactly.
double exact_reciprocal(double rate) {
    int e = 0;
    const double m = std::frexp(rate, &e);
    if (m != 0.5 || e < -510 || e > 512) return 0.0;
    return std::ldexp(1.0, 1 - e);
}

// The mm1 division mode for a pair of rates (kernels.cuh kDiv*) and the reciprocals it
// uses: exact ones for powers of two, RN(1/rate) inside [2^-900, 2^900].
struct DivMode {
    int div;
    double inv_lambda, inv_mu;
};
DivMode div_mode(double lambda, double mu) {
    const double el = exact_reciprocal(lambda), em = exact_reciprocal(mu);
    if (el != 0.0 && em != 0.0) return {kDivPow2, el, em};
    auto ok = [](double r) { return r >= 0x1p-900 && r <= 0x1p900; };
    if (ok(lambda) && ok(mu)) return {kDivRcp, 1.0 / lambda, 1.0 / mu};
    return {kDivIeee, 0.0, 0.0};
}

int lane_table(DevCtx& c, uint64_t stride, const uint32_t*& out) {
    auto it = c.lane_tabs.find(stride);
    if (it == c.lane_tabs.end()) {
        if (static_cast<int>(c.lane_tabs.size()) >= kMaxLaneTabs) {
            WLP_CUDA(cudaDeviceSynchronize());
            for (auto& kv : c.lane_tabs) kv.second.release();
            c.lane_tabs.clear();
        }
        DevBuf<uint32_t>& b = c.lane_tabs[stride];
        WLP_TRY(upload_u32(b, lane_tables(stride)));
        out = b.p;
        return WLP_OK;
    }
    out = it->second.p;
    return WLP_OK;
}


// Lane tables of the wrapped pipelines: lane l jumps 2 * pipe_wrap_units(s, l) draws (every
// model here takes two draws per unit), cached per schedule.
int wrap_table(DevCtx& c, const PipeSched& s, const uint32_t*& out) {
    const auto key = std::make_tuple(s.G * 64 + s.S, s.qb, s.rb, s.tail);
    auto it = c.wrap_tabs.find(key);
    if (it != c.wrap_tabs.end()) {
        out = it->second.p;
        return WLP_OK;
    }
    if (static_cast<int>(c.wrap_tabs.size()) >= kMaxLaneTabs) {
        WLP_CUDA(cudaDeviceSynchronize());
        for (auto& kv : c.wrap_tabs) kv.second.release();
        c.wrap_tabs.clear();
    }
    std::array<uint64_t, 32> dist{};
    for (int l = 0; l < 32; ++l) dist[l] = 2ull * static_cast<uint64_t>(pipe_wrap_units(s, l % s.S));
    DevBuf<uint32_t>& b = c.wrap_tabs[key];
    WLP_TRY(upload_u32(b, lane_tables_dist(dist)));
    out = b.p;
    return WLP_OK;
}

int check_model_mode(int model, int mode) {
    if (model < 0 || model > 2) return fail(WLP_EDOMAIN, "unknown model id");
    if (mode < 0 || mode > 2) return fail(WLP_EDOMAIN, "unknown execution mode id");
    return WLP_OK;
}

// ---- host reference utilities -------------------------------------------------------

// validate_params (models.cpp:26-44)
int validate(int model, const wlp_params* p, std::string* warning) {
    if (!p) return fail(WLP_EDOMAIN, "params: null");
    if (p->replications < 1) return fail(WLP_EDOMAIN, "params: replications must be >= 1");
    switch (model) {
        case WLP_MODEL_PI:
            if (p->draws < 1) return fail(WLP_EDOMAIN, "pi: draws must be >= 1");
            break;
        case WLP_MODEL_MM1:
            if (p->clients < 1) return fail(WLP_EDOMAIN, "mm1: clients must be >= 1");
            if (!(p->lambda > 0.0) || !(p->mu > 0.0)) return fail(WLP_EDOMAIN, "mm1: rates must be > 0");
            if (p->lambda >= p->mu && warning)
                *warning = "mm1: lambda >= mu, queue is unstable; steady-state comparisons are off";
            break;
        case WLP_MODEL_WALK:
            if (p->steps < 1) return fail(WLP_EDOMAIN, "walk: steps must be >= 1");
            if (p->chunks < 2) return fail(WLP_EDOMAIN, "walk: chunks must be >= 2");
            break;
        default: return fail(WLP_EDOMAIN, "unknown model");
    }
    // device limit of this engine: per-lane counters are 32-bit
    if (units_of(model, *p) >= (int64_t(1) << 36))
        return fail(WLP_EPLAN, "units per replication exceed the device limit of 2^36");
    return WLP_OK;
}

// plan_launch (wlp.cpp:71-105) with the launch_warning text (kernel_ir.cpp:150-156).
int plan(int64_t R, int mode, int tlp_block, int64_t grid_limit, wlp_launch_cfg* cfg, std::string* warning) {
    if (R < 1) return fail(WLP_EPLAN, "plan_launch: need at least one replication");
    if (tlp_block < 1) return fail(WLP_EPLAN, "plan_launch: tlp_block_size must be >= 1");
    // CUDA's hardware limit, checked after the reference's own checks (wlp.cpp:73-76); the
    // profile's maxThreadsPerBlock is the C++ layer's (warpsim_api.cpp plan_launch)
    if (tlp_block > 1024)
        return fail(WLP_EPLAN, "plan_launch: tlp_block_size exceeds the device limit of 1024 threads per block");
    wlp_launch_cfg c{1, 1, 1, 1, 1, 32};
    if (mode == WLP_MODE_SEQUENTIAL) {
        c.warp_size = 1;
    } else if (mode == WLP_MODE_WLP) {
        c.block_x = 32;
        c.grid_x = R;
    } else if (mode == WLP_MODE_TLP) {
        c.block_x = std::min<int64_t>(R, tlp_block);
        c.grid_x = (R + c.block_x - 1) / c.block_x;
    } else {
        return fail(WLP_EDOMAIN, "unknown execution mode id");
    }
    if (c.grid_x > grid_limit || c.grid_y > grid_limit)
        return fail(WLP_EPLAN, "plan_launch: " + std::to_string(R) + " replications exceed the grid limit of " +
                                   std::to_string(grid_limit) + " blocks per dimension");
    const int64_t tpb = c.block_x * c.block_y * c.block_z;
    if (warning && tpb % c.warp_size != 0)
        *warning = "block size " + std::to_string(tpb) + " is not a multiple of warpSize " +
                   std::to_string(c.warp_size) + "; trailing warp runs partially populated";
    if (cfg) *cfg = c;
    return WLP_OK;
}

uint64_t splitmix64(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// rng_state_from_seed (rng.cpp:36-40) as the reference's g++ build behaves: its three
// word() calls are arguments of one call, evaluated right to left, so s3 takes the
// first splitmix64 output and s1 the third (pinned by tests/golden/spacing.json).
Taus master_from_seed(uint64_t seed) {
    uint64_t x = seed;
    const uint32_t first = static_cast<uint32_t>(splitmix64(x) >> 32);
    const uint32_t second = static_cast<uint32_t>(splitmix64(x) >> 32);
    const uint32_t third = static_cast<uint32_t>(splitmix64(x) >> 32);
    return make_state(third, second, first);
}

// inverse_normal_cdf (models.cpp:61-97): Acklam's rational guess + two Halley steps.
int inv_normal(double p, double* out) {
    if (!(p > 0.0 && p < 1.0)) return fail(WLP_EDOMAIN, "inverse_normal_cdf: p outside (0,1)");
    static const double A[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                                1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
    static const double B[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                                6.680131188771972e+01,  -1.328068155288572e+01};
    static const double C[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                                -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
    static const double D[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                                3.754408661907416e+00};
    const double plow = 0.02425;
    double x;
    if (p < plow) {
        const double q = std::sqrt(-2.0 * std::log(p));
        x = (((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    } else if (p <= 1.0 - plow) {
        const double q = p - 0.5, r = q * q;
        x = (((((A[0] * r + A[1]) * r + A[2]) * r + A[3]) * r + A[4]) * r + A[5]) * q /
            (((((B[0] * r + B[1]) * r + B[2]) * r + B[3]) * r + B[4]) * r + 1.0);
    } else {
        const double q = std::sqrt(-2.0 * std::log(1.0 - p));
        x = -(((((C[0] * q + C[1]) * q + C[2]) * q + C[3]) * q + C[4]) * q + C[5]) /
            ((((D[0] * q + D[1]) * q + D[2]) * q + D[3]) * q + 1.0);
    }
    const double sqrt2 = 1.4142135623730951, pi = 3.141592653589793;
    for (int k = 0; k < 2; ++k) {
        const double e = 0.5 * std::erfc(-x / sqrt2) - p;
        const double u = e * std::sqrt(2.0 * pi) * std::exp(x * x / 2.0);
        x = x - u / (1.0 + x * u / 2.0);
    }
    *out = x;
    return WLP_OK;
}

void dd_add(double& hi, double& lo, double v) {  // TwoSum
    const double s = hi + v;
    const double bb = s - hi;
    const double err = (hi - (s - bb)) + (v - bb);
    hi = s;
    lo += err;
}

// Rejections from specials (see wlp_spacing_rejections).
int spacing_rejections(std::vector<SpecialRec> sp, const std::vector<int64_t>& prev, std::vector<int64_t>& out) {
    std::sort(sp.begin(), sp.end(), [](const SpecialRec& a, const SpecialRec& b) { return a.index < b.index; });
    std::set<std::tuple<uint32_t, uint32_t, uint32_t>> seen;
    out = prev;
    for (const SpecialRec& s : sp) {
        if (!seen.insert({s.s1, s.s2, s.s3}).second) out.push_back(s.index);
    }
    std::sort(out.begin(), out.end());
    out.erase(std::unique(out.begin(), out.end()), out.end());
    // rng.cpp:80-82: one stream redrawn 1000 times is an Error.
    int64_t run = 0;
    for (size_t i = 0; i < out.size(); ++i) {
        run = (i > 0 && out[i] == out[i - 1] + 1) ? run + 1 : 1;
        if (run >= 1000) return fail(WLP_ESPACING, "random_spacing: could not find a distinct stream seed");
    }
    return WLP_OK;
}

// ---- device building blocks ------------------------------------------------------------

// Seed slots [slot_begin, slot_begin+count) into d_out (SoA), async; specials counted.
int seed_async(DevCtx& c, Taus master, int64_t slot_begin, int64_t count, const std::vector<int64_t>& rej,
               uint32_t* d_out, cudaStream_t st, bool planes = false) {
    if (!rej.empty()) {
        WLP_CUDA(c.rejected.ensure(static_cast<int64_t>(rej.size())));
        WLP_CUDA(cudaMemcpyAsync(c.rejected.p, rej.data(), rej.size() * 8, cudaMemcpyHostToDevice, st));
    }
    // counter[spec_slot] is zero (the previous seeding cleared it); this seeding clears the
    // other slot and the grab counter of the model launch behind it
    const int slot = c.spec_slot;
    c.spec_slot = 1 - slot;
    c.spec_read = slot;
    c.work_zeroed = true;
    SeedArgs a;
    a.powers = c.powers.p;
    a.master = master;
    a.slot_begin = slot_begin;
    a.count = count;
    a.rejected = rej.empty() ? nullptr : c.rejected.p;
    a.n_rejected = static_cast<int64_t>(rej.size());
    a.out = d_out;
    a.specials = c.specials.p;
    a.special_cap = kSpecialCap;
    a.n_special = c.counter.p + slot;
    a.zero_a = c.counter.p + (1 - slot);
    a.zero_b = c.counter.p + 2;
    a.done = c.seed_done.p;
    a.report = c.d_mapped;
    c.spec_mapped = true;
    *reinterpret_cast<volatile unsigned long long*>(c.h_mapped) = kCountPending;  // (no seeding in flight writes it)
    c.planes_of = nullptr;
    c.planes_count = -1;
    if (planes) {  // the walk's bitsliced pipeline follows: write its bit planes as well
        WLP_CUDA(c.bseeds.ensure((count + 31) / 32 * 88));
        a.planes = c.bseeds.p;
        c.planes_of = d_out;
        c.planes_count = count;
    }
    WLP_CUDA(launch_seed(a, st));
    c.pdl_next = true;
    return WLP_OK;
}

// Specials of the last seed_async (synchronises the stream).
// seed_only: wait for the seeding alone (its last block stores the count to mapped host
// memory) and leave the model running on the stream: a run into device buffers then
// returns while its model kernel works, and the caller's next launches queue behind it.
int read_specials(DevCtx& c, cudaStream_t st, std::vector<SpecialRec>& sp, int64_t& n_total, bool seed_only = false) {
    c.work_zeroed = false;
    unsigned long long n = 0;
    if (c.spec_mapped) {  // the seeding's last block stored it in mapped host memory
        volatile unsigned long long* v = reinterpret_cast<volatile unsigned long long*>(c.h_mapped);
        bool synced = !seed_only;
        if (seed_only) {
            // spin on the word; every ~4k polls ask the stream, so a failed launch or a
            // finished stream (the count then must be there) ends the wait
            for (unsigned it = 1; *v == kCountPending; ++it) {
                if ((it & 4095u) == 0u) {
                    const cudaError_t q = cudaStreamQuery(st);
                    if (q != cudaErrorNotReady) {
                        synced = true;
                        break;
                    }
                }
            }
        }
        if (synced) WLP_CUDA(cudaStreamSynchronize(st));
        n = *v;
        if (n == kCountPending) return fail(WLP_EINTERNAL, "random_spacing: the seeding did not report its count");
    } else {
        WLP_CUDA(cudaMemcpyAsync(c.h_counter, c.counter.p + c.spec_read, 8, cudaMemcpyDeviceToHost, st));
        WLP_CUDA(cudaStreamSynchronize(st));
        n = *c.h_counter;
    }
    n_total = static_cast<int64_t>(n);
    if (n_total > kSpecialCap) return fail(WLP_EINTERNAL, "random_spacing: too many special candidates");
    sp.resize(static_cast<size_t>(n_total));
    if (n_total) WLP_CUDA(cudaMemcpy(sp.data(), c.specials.p, n_total * sizeof(SpecialRec), cudaMemcpyDeviceToHost));
    return WLP_OK;
}

int wlp_grid(DevCtx& c, int model, int64_t count) {
    const int warps_per_block = (model == WLP_MODEL_MM1 ? kMm1Block : kWlpBlock) / 32;
    const int64_t cap = static_cast<int64_t>(c.sms) * c.wlp_bps[model];
    const int64_t need = (count + warps_per_block - 1) / warps_per_block;
    return static_cast<int>(std::max<int64_t>(1, std::min(cap, need)));
}

// Which WLP walk kernel (wlp_set_wlp_variant numbering): 3 bitsliced pipeline, 4 bitsliced
// lane chunks, 0 the per-replication kernels. Automatic: the pipeline once every resident
// warp gets 8 or more groups of 32 replications (its 31-step drain is then small; R >=
// ~3.8e5 on 148 SMs), lane chunks from one group per SM up to there (config 3, R = 1e5:
// 0.051 ms against 0.143 per replication), per replication below that or when the
// counts could pass 2^16 per chunk.
int walk_bs_choice(const DevCtx& c, int64_t count, int64_t n) {
    const bool pipe_ok = n < 65536, lanes_ok = (n + 31) / 32 < 65536;
    if (g_wlp_variant == 3) return pipe_ok ? 3 : 0;
    if (g_wlp_variant == 4) return lanes_ok ? 4 : 0;
    if (g_wlp_variant != 0) return 0;
    const int64_t groups = (count + 31) / 32;
    if (pipe_ok && groups >= 8 * static_cast<int64_t>(c.sms) * c.bs_pipe_bps * (kBsPipeBlock / 32)) return 3;
    if (lanes_ok && groups >= c.sms) return 4;
    return 0;
}

// Whether the seeding should also write the walk's bit planes (the bitsliced pipeline
// will run, and then needs no separate transposition pass).
bool walk_planes(const DevCtx& c, int model, int mode, const wlp_params& p, int64_t count) {
    return model == WLP_MODEL_WALK && mode != WLP_MODE_TLP && !g_hw_counters && walk_bs_choice(c, count, p.steps) == 3;
}

// Device aliases of the caller's host output arrays when they are pinned and mapped into
// this device's address space (cudaHostAlloc, cudaHostRegister; torch pin_memory): the
// model kernel then stores every output there as well, as it is produced, and no copy
// follows the run. Pageable arrays keep the device buffer and the copy.
bool host_mirrors(DevCtx& c, int model, double* h0, double* h1, double* h2, double* (&out)[3]) {
    double* hs[3] = {h0, h1, h2};
    out[0] = out[1] = out[2] = nullptr;
    for (int k = 0; k < (model == WLP_MODEL_MM1 ? 3 : 1); ++k) {
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, hs[k]) != cudaSuccess) {
            cudaGetLastError();  // (an unregistered pointer is not an error for the run)
            return false;
        }
        if (at.type != cudaMemoryTypeHost || at.devicePointer == nullptr || at.device != c.dev) return false;
        out[k] = static_cast<double*>(at.devicePointer);
    }
    return true;
}

// The model kernel's start event: recorded by model_async right before its launch, after
// any host-side preparation (lane tables are built on first use), when c.time_model is set.
int mark_model_start(DevCtx& c, cudaStream_t st) {
    if (c.time_model) WLP_CUDA(cudaEventRecord(c.ev0, st));
    // the model kernel may overlap the seeding's tail (PDL) unless events bracket it
    set_pdl_launch(c.pdl_next && !c.time_model);
    return WLP_OK;
}

// Launch the model over d_seeds (count replications). Async. With c.time_model the caller
// records c.ev1 after it (c.ev0 is recorded here).
int model_async(DevCtx& c, int model, const wlp_params& p, int mode, int tlp_block, const uint32_t* d_seeds,
                int64_t count, double* o0, double* o1, double* o2, cudaStream_t st, int& grid_out) {
    const bool zeroed = c.work_zeroed;  // valid only for the launch right after seed_async
    c.work_zeroed = false;
    struct PdlReset {  // PDL only for the launch right after seed_async, never past this call
        DevCtx& c;
        ~PdlReset() {
            c.pdl_next = false;
            set_pdl_launch(false);
        }
    } pdl_reset{c};
    if (!zeroed || g_hw_counters) c.pdl_next = false;  // memsets would sit between seeding and model
    RepArgs a;
    a.seeds = d_seeds;
    a.count = count;
    a.n = units_of(model, p);
    a.chunks = p.chunks;
    a.lambda = p.lambda;
    a.mu = p.mu;
    if (model == WLP_MODEL_MM1) {
        const DivMode d = div_mode(p.lambda, p.mu);
        a.div = d.div;
        a.inv_lambda = d.inv_lambda;
        a.inv_mu = d.inv_mu;
    } else {
        a.inv_lambda = a.inv_mu = 0.0;
    }
    a.out0 = o0;
    a.out1 = o1;
    a.out2 = o2;
    a.h0 = c.hm[0];  // (set by the caller for this launch only)
    a.h1 = c.hm[1];
    a.h2 = c.hm[2];
    c.hm[0] = c.hm[1] = c.hm[2] = nullptr;
    a.serial_rho = mm1_serial_rho();
    a.near_cap = g_near_cap;
    if (g_hw_counters) {
        WLP_CUDA(cudaMemsetAsync(c.hw.p, 0, kHwClk * sizeof(unsigned long long), st));
        WLP_CUDA(cudaMemsetAsync(c.hw.p + kHwClk, 0xFF, kHwMaxSms * sizeof(unsigned long long), st));  // starts: min
        WLP_CUDA(cudaMemsetAsync(c.hw.p + kHwClk + kHwMaxSms, 0, kHwMaxSms * sizeof(unsigned long long), st));
        a.hw = c.hw.p;
    }
    if (mode == WLP_MODE_TLP) {
        if (model == WLP_MODEL_WALK && g_tlp_variant == 2 && !g_hw_counters && a.n < (int64_t(1) << 31)) {
            grid_out = static_cast<int>((count + 32 * 128 - 1) / (32 * 128));
            g_last_kernel = "k_tlp_walk_bs";
            WLP_TRY(mark_model_start(c, st));
            WLP_CUDA(launch_tlp_walk_bs(a, st));
            return WLP_OK;
        }
        const int64_t block = std::min<int64_t>(count, tlp_block);
        grid_out = static_cast<int>((count + block - 1) / block);
        g_last_kernel = model == WLP_MODEL_PI ? "k_tlp<pi>" : (model == WLP_MODEL_MM1 ? "k_tlp_mm1" : "k_tlp<walk>");
        WLP_TRY(mark_model_start(c, st));
        WLP_CUDA(launch_tlp(model, a, tlp_block, st));
        return WLP_OK;
    }
    // WLP, and SEQUENTIAL (replication order is irrelevant to the per-replication result;
    // the engine has no host execution path).
    grid_out = wlp_grid(c, model, count);
    const int64_t warps = static_cast<int64_t>(grid_out) * ((model == WLP_MODEL_MM1 ? kMm1Block : kWlpBlock) / 32);
    a.grab = static_cast<int>(std::clamp<int64_t>(count / (warps * 32), 1, 32));  // ~32 grabs per warp
    if (zeroed) {  // seed_async just cleared counter[1] on this stream
        a.next = c.counter.p + 2;
    } else {
        a.next = c.work.p;
        WLP_CUDA(cudaMemsetAsync(c.work.p, 0, sizeof(unsigned long long), st));
    }
    if (model == WLP_MODEL_MM1) {
        // The pipeline runs each segment's recursion and sums in order on one lane (TLP's
        // per-client cost) but drains 31 steps per warp; segment chaining pays ~1.8x per
        // client but has no drain. Pipeline when the drain is the smaller loss.
        const double per_warp = static_cast<double>(count) / static_cast<double>(warps);
        const bool pipe = !g_hw_counters && (g_wlp_variant == 2 || (g_wlp_variant == 0 && per_warp > 30.0));
        if (pipe) {
            // its own occupancy (4 blocks of 8 warps), not the segment-chaining kernel's
            const int64_t cap = static_cast<int64_t>(c.sms) * c.mm1_pipe_bps;
            grid_out = static_cast<int>(std::clamp<int64_t>((count + kMm1Block / 32 - 1) / (kMm1Block / 32), 1, cap));
            a.grab = static_cast<int>(
                std::clamp<int64_t>(count / (static_cast<int64_t>(grid_out) * (kMm1Block / 32) * 32), 1, 32));
            g_last_kernel = "k_wlp_mm1_pipe";
            WLP_TRY(mark_model_start(c, st));
            // whole panels at every step (n % 8 == 0). S lanes per replication: 2 when
            // every pipeline of the grid gets >= 4 replications (one drain step instead of
            // S - 1, and the least hand-over: config 4 41.87 ms at S = 8, 41.31 at S = 2);
            // on smaller runs 8, or 32 when a lane's chunk is long (more panels a step)
            int S = g_pipe_lanes;
            if (S == 0) {
                const int64_t pipes2 = static_cast<int64_t>(grid_out) * (kMm1Block / 32) * 16;
                S = count >= 4 * pipes2 ? 2 : (a.n >= 32 * kMm1PanelT * 8 ? 32 : 8);
            }
            int G = kMm1PanelT;
            if (a.n % kMm1PanelT != 0 || a.n < static_cast<int64_t>(S) * kMm1PanelT) {  // the ragged kernel
                S = 32;
                G = a.n >= 32 * kMm1PanelT ? kMm1PanelT : 1;
            }
            const int64_t P = 32 / S;
            a.grab = static_cast<int>(P * std::clamp<int64_t>(a.grab / P, 1, 32));
            const PipeSched ps = pipe_sched(a.n, G, S);
            WLP_CUDA(launch_wlp_mm1_pipe(a, ps, grid_out, st));
        } else {
            g_last_kernel = "k_wlp_mm1";
            WLP_TRY(mark_model_start(c, st));
            WLP_CUDA(launch_wlp(model, a, c.mm1_lane.p, c.mm1_skip.p, 0, grid_out, st));
        }
    } else if (model == WLP_MODEL_WALK && !g_hw_counters && walk_bs_choice(c, count, a.n) == 4) {
        // bitsliced lane chunks: a warp per group of 32 replications
        const int64_t groups = (count + 31) / 32;
        const int64_t K = (a.n + 31) / 32;
        const int64_t cap = static_cast<int64_t>(c.sms) * 2;  // 2 blocks of 4 warps per SM
        grid_out = static_cast<int>(std::clamp<int64_t>((groups + 3) / 4, 1, cap));
        a.grab = static_cast<int>(std::clamp<int64_t>(groups / (4 * grid_out * 8), 1, 32));
        const uint32_t* tab = nullptr;
        WLP_TRY(lane_table(c, 2ull * static_cast<uint64_t>(K), tab));
        g_last_kernel = "k_wlp_walk_bs_lanes";
        WLP_TRY(mark_model_start(c, st));
        WLP_CUDA(launch_wlp_walk_bs_lanes(a, tab, K, grid_out, st));
    } else if (model == WLP_MODEL_WALK && !g_hw_counters && walk_bs_choice(c, count, a.n) == 3) {
        // bitsliced pipeline: groups of 32 replications, rotating schedule; each warp owns
        // kWrap wrap groups (no fill or drain) when there are at least 2 * kWrap per warp
        const int64_t groups = (count + 31) / 32;
        const int64_t cap = static_cast<int64_t>(c.sms) * c.bs_pipe_bps;
        constexpr int64_t kBsW = kBsPipeBlock / 32;
        // S lanes per group: the most lanes that still give every lane >= 250 walk steps
        // per pipeline step (config 4, 1,000 steps: S = 4, eight pipelines per warp; the
        // hand-over of 120 words per step then costs ~1 % instead of ~9 % at S = 32)
        int S = g_pipe_lanes;
        if (S == 0) S = a.n >= 32 * 250 ? 32 : (a.n >= 16 * 250 ? 16 : (a.n >= 8 * 250 ? 8 : 4));
        if (S < 4) S = 4;  // (the bitsliced pipeline comes in 4, 8, 16 and 32 lanes)
        const int64_t blocks = std::clamp<int64_t>((std::max<int64_t>(1, groups / 64) + 1) / 2, 1, cap);
        const int64_t wpw = pipe_wrap_per_warp(S);
        const bool wrap = groups >= wpw * kBsW * blocks;
        grid_out = static_cast<int>(blocks);
        const int64_t pool = groups - (wrap ? wpw * kBsW * blocks : 0);
        const int64_t P = 32 / S;
        a.grab = static_cast<int>(P * std::clamp<int64_t>(pool / (kBsW * blocks * 32 * P), 1, 32));
        const PipeSched ps = pipe_sched(a.n, a.n >= 16 * S ? 16 : 1, S);
        const uint32_t* wtab = nullptr;
        if (wrap) WLP_TRY(wrap_table(c, ps, wtab));
        g_last_kernel = "k_wlp_walk_bs_pipe";
        const bool ready = c.planes_of == d_seeds && c.planes_count == count;  // from the seeding
        if (!ready) WLP_CUDA(c.bseeds.ensure(groups * 88));
        WLP_TRY(mark_model_start(c, st));
        WLP_CUDA(launch_wlp_walk_bs_pipe(a, c.bseeds.p, ps, wtab, grid_out, st, ready));
    } else {
        const int64_t K = (a.n + 31) / 32;
        // Lane jumps cost ~80 instructions per lane per replication against K units of
        // ~31-39. The pipeline has none; with the wrap (every S-lane pipeline owns S - 1
        // replications beyond the ones its warp grabs) it has no fill or drain either;
        // without it a 31-step triangle per warp idles.
        int pgrid = static_cast<int>(std::min<int64_t>(grid_out, static_cast<int64_t>(c.sms) * c.pipe_bps));
        // S lanes per replication: 2 (each replication two chunks, one hand-over; config 4
        // pi 10.89 ms vs 11.06 at S = 4, config 2 10.81 vs 11.18 at S = 32) when the run
        // fills the grid with wrapped two-lane pipelines; on smaller runs the most lanes that
        // give every lane >= 250 units per step
        int S = g_pipe_lanes;
        if (S == 0) {
            S = a.n >= 32 * 250 ? 32 : (a.n >= 16 * 250 ? 16 : (a.n >= 8 * 250 ? 8 : 4));
            if (count >= 2 * pipe_wrap_per_warp(2) * static_cast<int64_t>(pgrid) * (kWlpBlock / 32)) S = 2;
        }
        const int64_t wpw = pipe_wrap_per_warp(S);
        bool wrap = count >= 2 * wpw * static_cast<int64_t>(pgrid) * (kWlpBlock / 32);
        if (!wrap && (g_wlp_variant == 2 || S < 32) && count >= 2 * wpw * (kWlpBlock / 32)) {
            // fewer warps, each with its wrap replications (a forced pipeline on a small run)
            pgrid = static_cast<int>(count / (2 * wpw * (kWlpBlock / 32)));
            wrap = true;
        }
        if (!wrap) S = 32;  // only the whole-warp pipeline runs without the wrap
        const int64_t pwarps = static_cast<int64_t>(pgrid) * (kWlpBlock / 32);
        const double per_warp = static_cast<double>(count) / static_cast<double>(pwarps);
        const bool pipe = !g_hw_counters &&
                          (g_wlp_variant == 2 ||
                           (g_wlp_variant == 0 && ((wrap && pgrid >= c.sms) ||
                                                   31.0 / (per_warp + 31.0) < 80.0 / (35.0 * K + 80.0))));
        if (pipe) {
            grid_out = pgrid;
            const int P = 32 / S;
            const int64_t pool = count - (wrap ? wpw * pwarps : 0);
            a.grab = P * static_cast<int>(std::clamp<int64_t>(pool / (pwarps * 32 * P), 1, 32));
            const PipeSched ps = pipe_sched(a.n, a.n >= 8 * S ? 8 : 1, S);
            const uint32_t* wtab = nullptr;
            if (wrap) WLP_TRY(wrap_table(c, ps, wtab));
            g_last_kernel = model == WLP_MODEL_PI ? "k_wlp_pipe<pi>" : "k_wlp_pipe<walk>";
            WLP_TRY(mark_model_start(c, st));
            WLP_CUDA(launch_wlp_pipe(model, a, ps, wtab, grid_out, st));
        } else {
            // With few replications per warp the last groups leave a tail: 3 of the 4
            // resident blocks per SM then do better (config 3: 0.143 vs 0.148 ms).
            if (per_warp < 32.0) grid_out = std::min(grid_out, 3 * c.sms);
            const uint32_t* tab = nullptr;
            WLP_TRY(lane_table(c, 2ull * static_cast<uint64_t>(K), tab));
            g_last_kernel = model == WLP_MODEL_PI ? "k_wlp_lanes<pi>" : "k_wlp_lanes<walk>";
            WLP_TRY(mark_model_start(c, st));
            WLP_CUDA(launch_wlp(model, a, tab, nullptr, K, grid_out, st));
        }
    }
    return WLP_OK;
}

void fill_report(DevCtx& c, int model, int mode, int tlp_block, int64_t count, int grid, float ms, wlp_report* rep) {
    if (!rep) return;
    std::memset(rep, 0, sizeof *rep);
    rep->kernel_ms = ms;
    rep->total_cycles = static_cast<int64_t>(std::llround(static_cast<double>(ms) * c.clock_khz));
    int64_t bps, warps_per_block;
    if (mode == WLP_MODE_TLP) {
        const int block = static_cast<int>(std::min<int64_t>(count, tlp_block));
        bps = tlp_blocks_per_sm(model, block);
        warps_per_block = (block + 31) / 32;
    } else {
        bps = c.wlp_bps[model];
        warps_per_block = (model == WLP_MODEL_MM1 ? kMm1Block : kWlpBlock) / 32;
    }
    const int64_t resident = bps * c.sms;
    rep->waves_executed = (grid + resident - 1) / resident;
    rep->peak_resident_warps = std::min<int64_t>(grid, resident) * warps_per_block;
    if (g_hw_counters) {  // tallies of the instrumented kernels (the stream is synchronised)
        std::vector<unsigned long long> h(kHwWords, 0ull);
        if (cudaMemcpy(h.data(), c.hw.p, kHwWords * sizeof(unsigned long long), cudaMemcpyDeviceToHost) ==
            cudaSuccess) {
            rep->divergence_events = h[0];
            rep->mem_reads = h[1];
            rep->mem_writes = h[2];
            rep->warp_splits = h[0] + h[3];
            // makespan in SM cycles: per SM its own clock64, latest end - earliest start
            unsigned long long span = 0;
            for (int sm = 0; sm < kHwMaxSms; ++sm) {
                const unsigned long long t0 = h[kHwClk + sm], t1 = h[kHwClk + kHwMaxSms + sm];
                if (t0 != ~0ull && t1 >= t0) span = std::max(span, t1 - t0);
            }
            if (span) rep->total_cycles = static_cast<int64_t>(span);
        }
    }
}

int stats_device(DevCtx& c, const double* x, int64_t n, int pass, wlp_stats* s, cudaStream_t st) {
    const int grid = std::max(1, std::min<int>(c.sms, static_cast<int>((n + 1023) / 1024)));
    WLP_CUDA(c.partials.ensure(2 * grid));
    const double center = pass == 1 ? 0.0 : s->center;
    const bool seq = g_stats_order == 1;
    WLP_CUDA(launch_stats(x, n, pass, center, c.partials.p, grid, st, seq));
    const int used = n <= 256 || seq ? 1 : grid;
    std::vector<double> h(2 * used);
    WLP_CUDA(cudaMemcpyAsync(h.data(), c.partials.p, h.size() * 8, cudaMemcpyDeviceToHost, st));
    WLP_CUDA(cudaStreamSynchronize(st));
    double hi = 0.0, lo = 0.0;
    for (int b = 0; b < used; ++b) {
        dd_add(hi, lo, h[2 * b]);
        lo += h[2 * b + 1];
    }
    // renormalise
    const double t = hi + lo;
    lo = lo - (t - hi);
    hi = t;
    if (pass == 1) {
        s->n = n;
        s->sum_hi = hi;
        s->sum_lo = lo;
        s->center = (hi + lo) / static_cast<double>(n);
    } else {
        s->ss_hi = hi;
        s->ss_lo = lo;
    }
    return WLP_OK;
}

int ci_from_stats(const wlp_stats* s, double level, wlp_ci* ci) {
    if (s->n < 2) return fail(WLP_EDOMAIN, "confidence_interval: need at least 2 samples");
    if (!(level > 0.0 && level < 1.0)) return fail(WLP_EDOMAIN, "confidence_interval: level outside (0,1)");
    const double n = static_cast<double>(s->n);
    const double mean = (s->sum_hi + s->sum_lo) / n;
    const double sd = std::sqrt((s->ss_hi + s->ss_lo) / static_cast<double>(s->n - 1));
    double z = 0.0;
    WLP_TRY(inv_normal(0.5 + level / 2.0, &z));
    ci->mean = mean;
    ci->half_width = z * sd / std::sqrt(n);
    ci->level = level;
    ci->n = s->n;
    ci->warn_small_sample = s->n < 30 ? 1 : 0;
    return WLP_OK;
}

int ci_device(DevCtx& c, const double* d_x, int64_t n, double level, wlp_ci* ci, cudaStream_t st) {
    if (n < 2) return fail(WLP_EDOMAIN, "confidence_interval: need at least 2 samples");
    if (!(level > 0.0 && level < 1.0)) return fail(WLP_EDOMAIN, "confidence_interval: level outside (0,1)");
    wlp_stats s{};
    WLP_TRY(stats_device(c, d_x, n, 1, &s, st));
    WLP_TRY(stats_device(c, d_x, n, 2, &s, st));
    return ci_from_stats(&s, level, ci);
}

// All outputs' confidence intervals with one host synchronisation: per output, pass 1, the
// device fold of its partials (mean on the device), pass 2 about that mean; one copy of
// every output's {hi, lo, mean} and pass-2 partials; then the host merge of pass 2 as in
// stats_device. Same numbers as ci_device, bit for bit. ci_enqueue launches; the caller
// synchronises the stream (e.g. with the specials read-back) and calls ci_finish.
struct CiPlan {
    int nout = 0, grid = 1, used = 1;
    int64_t n = 0;
    double level = 0.95;
    std::vector<double> host;  // per output: meta[4] then pass-2 partials [2 * grid]
};

int ci_enqueue(DevCtx& c, const double* const* d_x, int nout, int64_t n, double level, CiPlan& plan,
               cudaStream_t st) {
    if (n < 2) return fail(WLP_EDOMAIN, "confidence_interval: need at least 2 samples");
    if (!(level > 0.0 && level < 1.0)) return fail(WLP_EDOMAIN, "confidence_interval: level outside (0,1)");
    plan.nout = nout;
    plan.n = n;
    plan.level = level;
    plan.grid = std::max(1, std::min<int>(c.sms, static_cast<int>((n + 1023) / 1024)));
    const bool seq = g_stats_order == 1;
    plan.used = n <= 256 || seq ? 1 : plan.grid;
    const int64_t per = 4 + 4 * static_cast<int64_t>(plan.grid);  // meta[4], pass 1 [2g], pass 2 [2g]
    WLP_CUDA(c.partials.ensure(per * nout));
    for (int k = 0; k < nout; ++k) {
        double* base = c.partials.p + k * per;
        double* p1 = base + 4;
        double* p2 = base + 4 + 2 * plan.grid;
        WLP_CUDA(launch_stats(d_x[k], n, 1, 0.0, p1, plan.grid, st, seq));
        WLP_CUDA(launch_stats_fold(p1, plan.used, n, base, st));
        WLP_CUDA(launch_stats(d_x[k], n, 2, 0.0, p2, plan.grid, st, seq, base + 2));
    }
    plan.host.resize(static_cast<size_t>(per * nout));
    WLP_CUDA(cudaMemcpyAsync(plan.host.data(), c.partials.p, plan.host.size() * 8, cudaMemcpyDeviceToHost, st));
    return WLP_OK;
}

int ci_finish(const CiPlan& plan, wlp_ci* ci) {  // after the stream is synchronised
    const int64_t per = 4 + 4 * static_cast<int64_t>(plan.grid);
    for (int k = 0; k < plan.nout; ++k) {
        const double* base = plan.host.data() + k * per;
        const double* p2 = base + 4 + 2 * plan.grid;
        wlp_stats s{};
        s.n = plan.n;
        s.sum_hi = base[0];
        s.sum_lo = base[1];
        s.center = base[2];
        double hi = 0.0, lo = 0.0;
        for (int b = 0; b < plan.used; ++b) {
            dd_add(hi, lo, p2[2 * b]);
            lo += p2[2 * b + 1];
        }
        const double t = hi + lo;
        lo = lo - (t - hi);
        hi = t;
        s.ss_hi = hi;
        s.ss_lo = lo;
        WLP_TRY(ci_from_stats(&s, plan.level, &ci[k]));
    }
    return WLP_OK;
}

void copy_warning(const std::string& w, char* buf, int cap) {
    if (!buf || cap <= 0) return;
    const size_t n = std::min<size_t>(w.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, w.data(), n);
    buf[n] = 0;
}

int n_outputs(int model) { return model == WLP_MODEL_MM1 ? 3 : 1; }

}  // namespace
}  // namespace wlp

using namespace wlp;

extern "C" {

const char* wlp_last_error(void) { return g_err.c_str(); }
int wlp_version(void) { return 1; }

int wlp_set_wlp_variant(int variant) {
    if (variant < 0 || variant > 4) return fail(WLP_EDOMAIN, "wlp variant must be 0 (auto), 1, 2, 3 or 4");
    g_wlp_variant = variant;
    return WLP_OK;
}

const char* wlp_last_kernel(void) { return g_last_kernel; }

int wlp_debug_set_near_cap(int cap) {
    if (cap < 1 || cap > 128 || (cap & (cap - 1)) != 0)
        return fail(WLP_EDOMAIN, "near-one list capacity must be a power of two in [1, 128]");
    g_near_cap = static_cast<uint32_t>(cap);
    return WLP_OK;
}

int wlp_set_pipe_lanes(int lanes) {
    if (lanes != 0 && lanes != 2 && lanes != 4 && lanes != 8 && lanes != 16 && lanes != 32)
        return fail(WLP_EDOMAIN, "pipeline lanes per replication must be 0 (auto), 2, 4, 8, 16 or 32");
    g_pipe_lanes = lanes;
    return WLP_OK;
}

int wlp_set_tlp_variant(int variant) {
    if (variant < 0 || variant > 2) return fail(WLP_EDOMAIN, "tlp variant must be 0 (auto), 1 or 2");
    g_tlp_variant = variant;
    return WLP_OK;
}

int wlp_set_stats_order(int order) {
    if (order < 0 || order > 1) return fail(WLP_EDOMAIN, "stats order must be 0 or 1");
    g_stats_order = order;
    return WLP_OK;
}

int wlp_set_hw_counters(int enable) {
    g_hw_counters = enable != 0;
    return WLP_OK;
}

int wlp_validate_params(int model, const wlp_params* p, char* warn, int warn_cap) {
    std::string w;
    WLP_TRY(validate(model, p, &w));
    copy_warning(w, warn, warn_cap);
    return WLP_OK;
}

int wlp_plan_launch(int64_t replications, int mode, int tlp_block_size, int64_t grid_limit, wlp_launch_cfg* cfg,
                    char* warn, int warn_cap) {
    std::string w;
    WLP_TRY(plan(replications, mode, tlp_block_size, grid_limit, cfg, &w));
    copy_warning(w, warn, warn_cap);
    return WLP_OK;
}

int wlp_master_from_seed(uint64_t seed, uint32_t out[3]) {
    const Taus t = master_from_seed(seed);
    out[0] = t.s1;
    out[1] = t.s2;
    out[2] = t.s3;
    return WLP_OK;
}

int wlp_make_state(uint32_t s1, uint32_t s2, uint32_t s3, uint32_t out[3]) {
    const Taus t = make_state(s1, s2, s3);
    out[0] = t.s1;
    out[1] = t.s2;
    out[2] = t.s3;
    return WLP_OK;
}

int wlp_jump_host(const uint32_t s[3], uint64_t n, uint32_t out[3]) {
    const Taus t = jump_state(Taus{s[0], s[1], s[2]}, n);
    out[0] = t.s1;
    out[1] = t.s2;
    out[2] = t.s3;
    return WLP_OK;
}

int wlp_inverse_normal_cdf(double p, double* z) { return inv_normal(p, z); }

int wlp_taus_next(uint32_t state[3], uint32_t* out) {
    Taus t{state[0], state[1], state[2]};
    const uint32_t o = taus_next(t);
    state[0] = t.s1;
    state[1] = t.s2;
    state[2] = t.s3;
    if (out) *out = o;
    return WLP_OK;
}

int wlp_uniform01(uint32_t state[3], double* out) {
    uint32_t o = 0;
    wlp_taus_next(state, &o);
    *out = static_cast<double>(o) * 0x1p-32;
    return WLP_OK;
}

int wlp_exponential_from_u(double u, double rate, double* out) {
    if (!(rate > 0.0)) return fail(WLP_EDOMAIN, "exponential: rate must be > 0");
    if (!(u >= 0.0 && u < 1.0)) return fail(WLP_EDOMAIN, "exponential: u outside [0,1)");
    *out = -glibc_log_tab(1.0 - u, kLogTabHost) / rate;
    return WLP_OK;
}

int wlp_spacing_rejections(const wlp_special* specials, int64_t n_special, const int64_t* prev, int64_t n_prev,
                           int64_t* out, int64_t out_cap, int64_t* n_out) {
    std::vector<SpecialRec> sp(n_special);
    if (n_special) std::memcpy(sp.data(), specials, n_special * sizeof(SpecialRec));
    std::vector<int64_t> pv(prev, prev + n_prev), res;
    WLP_TRY(spacing_rejections(sp, pv, res));
    if (static_cast<int64_t>(res.size()) > out_cap) return fail(WLP_EINTERNAL, "rejection buffer too small");
    std::copy(res.begin(), res.end(), out);
    *n_out = static_cast<int64_t>(res.size());
    return WLP_OK;
}

int wlp_stats_merge(wlp_stats* a, const wlp_stats* b) {
    a->n += b->n;
    dd_add(a->sum_hi, a->sum_lo, b->sum_hi);
    a->sum_lo += b->sum_lo;
    dd_add(a->ss_hi, a->ss_lo, b->ss_hi);
    a->ss_lo += b->ss_lo;
    return WLP_OK;
}

int wlp_ci_from_stats(const wlp_stats* s, double level, wlp_ci* ci) { return ci_from_stats(s, level, ci); }

int wlp_device_count(int* n) {
    WLP_CUDA(cudaGetDeviceCount(n));
    return WLP_OK;
}

int wlp_taus_stream(uint32_t s1, uint32_t s2, uint32_t s3, int64_t n, uint32_t* out, int out_on_device,
                    void* stream) {
    if (n < 0) return fail(WLP_EDOMAIN, "taus_stream: negative count");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    uint32_t* d = out;
    if (!out_on_device) {
        WLP_CUDA(c->seeds.ensure(std::max<int64_t>(n, 1)));
        d = c->seeds.p;
    }
    WLP_CUDA(launch_taus_stream(c->powers.p, make_state(s1, s2, s3), n, d, st));
    if (!out_on_device) {
        WLP_CUDA(cudaMemcpyAsync(out, d, n * 4, cudaMemcpyDeviceToHost, st));
        WLP_CUDA(cudaStreamSynchronize(st));
    }
    return WLP_OK;
}

int wlp_debug_neg_log1m(const uint32_t* k, int64_t n, double* out) {
    if (n < 0) return fail(WLP_EDOMAIN, "neg_log1m: negative count");
    if (n == 0) return WLP_OK;
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    StreamOrder so(*c, nullptr);
    WLP_CUDA(c->in_seeds.ensure(n));
    WLP_CUDA(c->outs.ensure(n));
    WLP_CUDA(cudaMemcpy(c->in_seeds.p, k, n * 4, cudaMemcpyHostToDevice));
    WLP_CUDA(launch_neg_log1m(c->in_seeds.p, n, c->outs.p, nullptr));
    WLP_CUDA(cudaMemcpy(out, c->outs.p, n * 8, cudaMemcpyDeviceToHost));
    return WLP_OK;
}

int wlp_seed_streams(uint64_t master_seed, int64_t slot_begin, int64_t count, const int64_t* rejected,
                     int64_t n_rejected, uint32_t* s_out, int out_on_device, void* stream, wlp_special* specials,
                     int64_t special_cap, int64_t* n_special) {
    if (count < 0 || slot_begin < 0) return fail(WLP_EDOMAIN, "seed_streams: negative range");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    uint32_t* d = s_out;
    if (!out_on_device) {
        WLP_CUDA(c->seeds.ensure(3 * std::max<int64_t>(count, 1)));
        d = c->seeds.p;
    }
    std::vector<int64_t> rej(rejected, rejected + n_rejected);
    WLP_TRY(seed_async(*c, master_from_seed(master_seed), slot_begin, count, rej, d, st));
    std::vector<SpecialRec> sp;
    int64_t nt = 0;
    WLP_TRY(read_specials(*c, st, sp, nt));
    if (n_special) *n_special = nt;
    if (specials) std::memcpy(specials, sp.data(), std::min<int64_t>(nt, special_cap) * sizeof(SpecialRec));
    if (!out_on_device) {
        WLP_CUDA(cudaMemcpy(s_out, d, 3 * count * 4, cudaMemcpyDeviceToHost));
    }
    return WLP_OK;
}

}  // extern "C"

namespace wlp {
namespace {
// Whole-run exact random_spacing from a master state; *n_rejected = redraws used.
int seed_exact(Taus master, int64_t count, uint32_t* s_out, int out_on_device, void* stream, int64_t* n_rejected) {
    if (count < 0) return fail(WLP_EDOMAIN, "seed_streams: negative count");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    uint32_t* d = s_out;
    if (!out_on_device) {
        WLP_CUDA(c->seeds.ensure(3 * std::max<int64_t>(count, 1)));
        d = c->seeds.p;
    }
    std::vector<int64_t> rej;
    for (;;) {
        WLP_TRY(seed_async(*c, master, 0, count, rej, d, st));
        c->work_zeroed = false;  // no model launch follows
        std::vector<SpecialRec> sp;
        int64_t nt = 0;
        WLP_TRY(read_specials(*c, st, sp, nt));
        if (nt < 2) break;
        std::vector<int64_t> next;
        WLP_TRY(spacing_rejections(sp, rej, next));
        if (next == rej) break;
        rej.swap(next);
    }
    if (!out_on_device && count) WLP_CUDA(cudaMemcpy(s_out, d, 3 * count * 4, cudaMemcpyDeviceToHost));
    if (n_rejected) *n_rejected = static_cast<int64_t>(rej.size());
    return WLP_OK;
}
}  // namespace
}  // namespace wlp

extern "C" {

int wlp_seed_streams_exact(uint64_t master_seed, int64_t count, uint32_t* s_out, int out_on_device, void* stream) {
    return seed_exact(master_from_seed(master_seed), count, s_out, out_on_device, stream, nullptr);
}

int wlp_seed_streams_state(const uint32_t master[3], int64_t count, uint32_t* s_out, int out_on_device,
                           void* stream, uint32_t master_out[3]) {
    const Taus m{master[0], master[1], master[2]};
    int64_t nrej = 0;
    WLP_TRY(seed_exact(m, count, s_out, out_on_device, stream, &nrej));
    if (master_out) {
        const Taus after = jump_state(m, 3ull * static_cast<uint64_t>(count + nrej));
        master_out[0] = after.s1;
        master_out[1] = after.s2;
        master_out[2] = after.s3;
    }
    return WLP_OK;
}

int wlp_run_streams(int model, const wlp_params* p, int mode, const uint32_t* s, int64_t count, int s_on_device,
                    double* out0, double* out1, double* out2, int out_on_device, void* stream, wlp_report* report) {
    WLP_TRY(check_model_mode(model, mode));
    if (count < 0) return fail(WLP_EDOMAIN, "run_streams: negative count");
    wlp_params q = *p;
    q.replications = std::max<int64_t>(count, 1);
    WLP_TRY(validate(model, &q, nullptr));
    if (count == 0) return WLP_OK;
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    const uint32_t* ds = s;
    if (!s_on_device) {
        WLP_CUDA(c->in_seeds.ensure(3 * count));
        WLP_CUDA(cudaMemcpyAsync(c->in_seeds.p, s, 3 * count * 4, cudaMemcpyHostToDevice, st));
        ds = c->in_seeds.p;
    }
    double *o0 = out0, *o1 = out1, *o2 = out2;
    if (!out_on_device) {
        WLP_CUDA(c->outs.ensure(3 * count));
        o0 = c->outs.p;
        o1 = c->outs.p + count;
        o2 = c->outs.p + 2 * count;
    }
    int grid = 0;
    c->time_model = report != nullptr;
    WLP_TRY(model_async(*c, model, q, mode, 256, ds, count, o0, o1, o2, st, grid));
    c->time_model = false;
    if (report) WLP_CUDA(cudaEventRecord(c->ev1, st));
    if (!out_on_device) {
        WLP_CUDA(cudaMemcpyAsync(out0, o0, count * 8, cudaMemcpyDeviceToHost, st));
        if (model == WLP_MODEL_MM1) {
            WLP_CUDA(cudaMemcpyAsync(out1, o1, count * 8, cudaMemcpyDeviceToHost, st));
            WLP_CUDA(cudaMemcpyAsync(out2, o2, count * 8, cudaMemcpyDeviceToHost, st));
        }
    }
    if (report || !out_on_device) WLP_CUDA(cudaStreamSynchronize(st));
    if (report) {
        float ms = 0.f;
        WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(*c, model, mode, 256, count, grid, ms, report);
    }
    return WLP_OK;
}

int wlp_run_shard(int model, const wlp_params* p, int mode, uint64_t master_seed, int tlp_block_size,
                  int64_t r_begin, int64_t r_count, const int64_t* rejected, int64_t n_rejected, double* out0,
                  double* out1, double* out2, int out_on_device, void* stream, wlp_special* specials,
                  int64_t special_cap, int64_t* n_special, wlp_report* report) {
    WLP_TRY(check_model_mode(model, mode));
    WLP_TRY(validate(model, p, nullptr));
    WLP_TRY(plan(p->replications, mode, tlp_block_size, 0x7FFFFFFF, nullptr, nullptr));
    if (r_begin < 0 || r_count < 0 || r_begin + r_count > p->replications)
        return fail(WLP_EDOMAIN, "run_shard: shard outside [0, replications)");
    if (r_count == 0) {
        if (n_special) *n_special = 0;
        return WLP_OK;
    }
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    WLP_CUDA(c->seeds.ensure(3 * r_count));
    double *o0 = out0, *o1 = out1, *o2 = out2;
    if (!out_on_device) {
        WLP_CUDA(c->outs.ensure(3 * r_count));
        o0 = c->outs.p;
        o1 = c->outs.p + r_count;
        o2 = c->outs.p + 2 * r_count;
    }
    double* mirror[3];
    const bool mirrored = !out_on_device && host_mirrors(*c, model, out0, out1, out2, mirror);
    std::vector<int64_t> rej(rejected, rejected + n_rejected);
    WLP_TRY(seed_async(*c, master_from_seed(master_seed), r_begin, r_count, rej, c->seeds.p, st,
                       walk_planes(*c, model, mode, *p, r_count)));
    int grid = 0;
    c->time_model = report != nullptr;
    if (mirrored) std::copy(mirror, mirror + 3, c->hm);
    WLP_TRY(model_async(*c, model, *p, mode, tlp_block_size, c->seeds.p, r_count, o0, o1, o2, st, grid));
    c->time_model = false;
    if (report) WLP_CUDA(cudaEventRecord(c->ev1, st));
    if (!out_on_device && !mirrored) {
        WLP_CUDA(cudaMemcpyAsync(out0, o0, r_count * 8, cudaMemcpyDeviceToHost, st));
        if (model == WLP_MODEL_MM1) {
            WLP_CUDA(cudaMemcpyAsync(out1, o1, r_count * 8, cudaMemcpyDeviceToHost, st));
            WLP_CUDA(cudaMemcpyAsync(out2, o2, r_count * 8, cudaMemcpyDeviceToHost, st));
        }
    }
    if (specials || n_special || report || !out_on_device) {
        std::vector<SpecialRec> sp;
        int64_t nt = 0;
        WLP_TRY(read_specials(*c, st, sp, nt, out_on_device && !report));
        if (n_special) *n_special = nt;
        if (specials) std::memcpy(specials, sp.data(), std::min<int64_t>(nt, special_cap) * sizeof(SpecialRec));
    }
    if (report) {
        float ms = 0.f;
        WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(*c, model, mode, tlp_block_size, r_count, grid, ms, report);
    }
    return WLP_OK;
}

int wlp_run(int model, const wlp_params* p, int mode, uint64_t master_seed, int tlp_block_size, double* out0,
            double* out1, double* out2, int out_on_device, void* stream, wlp_report* report, wlp_ci* ci,
            double level, char* warn, int warn_cap) {
    WLP_TRY(check_model_mode(model, mode));
    std::string pw, lw;
    WLP_TRY(validate(model, p, &pw));
    WLP_TRY(plan(p->replications, mode, tlp_block_size, 0x7FFFFFFF, nullptr, &lw));
    // build_kernel (models.cpp:294-299): params warning "; " plan warning
    copy_warning(!pw.empty() && !lw.empty() ? pw + "; " + lw : (!pw.empty() ? pw : lw), warn, warn_cap);
    const int64_t R = p->replications;
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    WLP_CUDA(c->seeds.ensure(3 * R));
    double *o0 = out0, *o1 = out1, *o2 = out2;
    if (!out_on_device) {
        WLP_CUDA(c->outs.ensure(3 * R));
        o0 = c->outs.p;
        o1 = c->outs.p + R;
        o2 = c->outs.p + 2 * R;
    }
    const Taus master = master_from_seed(master_seed);
    double* mirror[3];
    const bool mirrored = !out_on_device && host_mirrors(*c, model, out0, out1, out2, mirror);
    std::vector<int64_t> rej;
    int grid = 0;
    CiPlan plan;
    for (;;) {
        // Seeding and the model run back to back; the spacing check below only forces a
        // re-run when two special candidates actually share a key.
        WLP_TRY(seed_async(*c, master, 0, R, rej, c->seeds.p, st, walk_planes(*c, model, mode, *p, R)));
        c->time_model = report != nullptr;
        if (mirrored) std::copy(mirror, mirror + 3, c->hm);
        WLP_TRY(model_async(*c, model, *p, mode, tlp_block_size, c->seeds.p, R, o0, o1, o2, st, grid));
        c->time_model = false;
        if (report) WLP_CUDA(cudaEventRecord(c->ev1, st));
        if (ci) {  // both statistics passes of every output, behind the model, before the sync
            const double* d[3] = {o0, o1, o2};
            WLP_TRY(ci_enqueue(*c, d, n_outputs(model), R, level, plan, st));
        }
        std::vector<SpecialRec> sp;
        int64_t nt = 0;
        WLP_TRY(read_specials(*c, st, sp, nt, out_on_device && !report && !ci));
        if (nt < 2) break;
        std::vector<int64_t> next;
        WLP_TRY(spacing_rejections(sp, rej, next));
        if (next == rej) break;
        rej.swap(next);
    }
    if (ci) WLP_TRY(ci_finish(plan, ci));
    if (!out_on_device && !mirrored) {
        WLP_CUDA(cudaMemcpyAsync(out0, o0, R * 8, cudaMemcpyDeviceToHost, st));
        if (model == WLP_MODEL_MM1) {
            WLP_CUDA(cudaMemcpyAsync(out1, o1, R * 8, cudaMemcpyDeviceToHost, st));
            WLP_CUDA(cudaMemcpyAsync(out2, o2, R * 8, cudaMemcpyDeviceToHost, st));
        }
        WLP_CUDA(cudaStreamSynchronize(st));
    }
    if (report) {
        float ms = 0.f;
        WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        fill_report(*c, model, mode, tlp_block_size, R, grid, ms, report);
    }
    return WLP_OK;
}

// ---- the reference's *_replication_u bodies and exponential_from_u on the device ----

int wlp_run_uniforms(int model, const wlp_params* p, const double* u, int64_t count, int u_on_device,
                     double* out0, double* out1, double* out2, int out_on_device, void* stream) {
    if (model < 0 || model > 2) return fail(WLP_EDOMAIN, "unknown model id");
    if (count < 0) return fail(WLP_EDOMAIN, "run_uniforms: negative count");
    wlp_params q = *p;
    q.replications = 1;
    WLP_TRY(validate(model, &q, nullptr));  // the templates' DomainErrors (models.hpp:51, 63-64, 88-89)
    if (count == 0) return WLP_OK;
    const int64_t n = units_of(model, q);
    if (n > (int64_t(1) << 40) / std::max<int64_t>(count, 1)) return fail(WLP_EPLAN, "run_uniforms: too many uniforms");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    const int64_t nu = 2 * n * count;
    const double* du = u;
    DevBuf<double> ubuf, obuf;
    if (!u_on_device) {
        WLP_CUDA(ubuf.ensure(nu));
        WLP_CUDA(cudaMemcpyAsync(ubuf.p, u, nu * 8, cudaMemcpyHostToDevice, st));
        du = ubuf.p;
    }
    const int nout = n_outputs(model);
    UniArgs a{model, du, count, n, q.chunks, q.lambda, q.mu, out0, out1, out2};
    if (!out_on_device) {
        WLP_CUDA(obuf.ensure(nout * count));
        a.out0 = obuf.p;
        a.out1 = obuf.p + count;
        a.out2 = obuf.p + 2 * count;
    }
    WLP_CUDA(launch_uniform_reps(a, st));
    g_last_kernel = "k_uniform_reps";
    if (!out_on_device) {
        double* host[3] = {out0, out1, out2};
        double* dev[3] = {a.out0, a.out1, a.out2};
        for (int k = 0; k < nout; ++k) WLP_CUDA(cudaMemcpyAsync(host[k], dev[k], count * 8, cudaMemcpyDeviceToHost, st));
    }
    WLP_CUDA(cudaStreamSynchronize(st));  // the scratch buffers are released on return
    ubuf.release();
    obuf.release();
    return WLP_OK;
}

int wlp_exponentials(const double* u, int64_t n, double rate, double* out, int on_device, void* stream) {
    if (!(rate > 0.0)) return fail(WLP_EDOMAIN, "exponential: rate must be > 0");
    if (n < 0) return fail(WLP_EDOMAIN, "exponentials: negative count");
    if (n == 0) return WLP_OK;
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    DevBuf<double> buf;
    const double* du = u;
    double* dout = out;
    if (!on_device) {
        WLP_CUDA(buf.ensure(2 * n));
        WLP_CUDA(cudaMemcpyAsync(buf.p, u, n * 8, cudaMemcpyHostToDevice, st));
        du = buf.p;
        dout = buf.p + n;
    }
    WLP_CUDA(cudaMemsetAsync(c->work.p, 0xFF, 8, st));
    WLP_CUDA(launch_exponentials(du, n, rate, dout, c->work.p, st));
    unsigned long long bad = 0;
    WLP_CUDA(cudaMemcpyAsync(&bad, c->work.p, 8, cudaMemcpyDeviceToHost, st));
    if (!on_device) WLP_CUDA(cudaMemcpyAsync(out, dout, n * 8, cudaMemcpyDeviceToHost, st));
    WLP_CUDA(cudaStreamSynchronize(st));
    buf.release();
    if (bad != ~0ull) return fail(WLP_EDOMAIN, "exponential: u outside [0,1)");
    return WLP_OK;
}

// ---- run_model over several GPUs of this process ----------------------------------

}  // extern "C"

namespace wlp {
namespace {

// Host barrier for the per-device worker threads; abort() releases every waiter (a
// worker failed) and later waits return false.
class Barrier {
public:
    explicit Barrier(int n) : n_(n) {}
    bool wait() {
        std::unique_lock<std::mutex> l(m_);
        if (aborted_) return false;
        const int64_t gen = gen_;
        if (++arrived_ == n_) {
            arrived_ = 0;
            ++gen_;
            cv_.notify_all();
            return true;
        }
        cv_.wait(l, [&] { return gen_ != gen || aborted_; });
        return !aborted_;
    }
    void abort() {
        std::lock_guard<std::mutex> l(m_);
        aborted_ = true;
        cv_.notify_all();
    }

private:
    std::mutex m_;
    std::condition_variable cv_;
    int n_, arrived_ = 0;
    int64_t gen_ = 0;
    bool aborted_ = false;
};

struct DevShard {
    int dev = 0;
    int64_t begin = 0, count = 0;
    std::vector<SpecialRec> specials;
    wlp_stats first[3]{}, second[3]{};
    wlp_report rep{};
    const char* kernel = "";
    int rc = WLP_OK;
    std::string err;
};

// The calling thread's settings, applied in each worker (they are thread-local).
struct ThreadSettings {
    bool hw;
    int wv, tv, so, pl;
    void apply() const {
        g_hw_counters = hw;
        g_wlp_variant = wv;
        g_pipe_lanes = pl;
        g_tlp_variant = tv;
        g_stats_order = so;
    }
};

wlp_stats merged(const std::vector<DevShard>& sh, int k, bool second) {
    wlp_stats acc{};
    for (const DevShard& s : sh) {  // device order: every worker computes the same numbers
        const wlp_stats& b = second ? s.second[k] : s.first[k];
        acc.n += b.n;
        dd_add(acc.sum_hi, acc.sum_lo, b.sum_hi);
        acc.sum_lo += b.sum_lo;
        dd_add(acc.ss_hi, acc.ss_lo, b.ss_hi);
        acc.ss_lo += b.ss_lo;
    }
    return acc;
}

// One slice of wlp_run_devices, on its worker thread: seed + model into the slice's own
// buffers, the global spacing check (every worker reads every slice's specials after a
// barrier), the two statistics passes about the merged mean, and the slice's outputs to
// the host. The device context is locked per phase only, never across a barrier, so a
// device listed twice runs its slices one phase after another.
int run_device_shard(int model, const wlp_params& p, int mode, Taus master, int tlp_block, std::vector<DevShard>& sh,
                     int k, Barrier& bar, double* const host[3], std::vector<int64_t>& rej_out) {
    DevShard& me = sh[k];
    WLP_CUDA(cudaSetDevice(me.dev));
    cudaStream_t st = nullptr;
    WLP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Local {
        cudaStream_t s;
        DevBuf<uint32_t> seeds;
        DevBuf<double> outs;
        ~Local() {
            cudaStreamSynchronize(s);
            seeds.release();
            outs.release();
            cudaStreamDestroy(s);
        }
    } loc{st};
    const int64_t n = me.count;
    const int nout = n_outputs(model);
    WLP_CUDA(loc.seeds.ensure(3 * n));
    WLP_CUDA(loc.outs.ensure(3 * n));
    double* o[3] = {loc.outs.p, loc.outs.p + n, loc.outs.p + 2 * n};
    const std::string peer_failed = "another device failed";
    std::vector<int64_t> rej;
    for (;;) {
        {
            DevCtx* c;
            std::unique_lock<std::mutex> lk;
            WLP_TRY(acquire(c, lk));
            StreamOrder so(*c, st);
            int grid = 0;
            WLP_TRY(seed_async(*c, master, me.begin, n, rej, loc.seeds.p, st, walk_planes(*c, model, mode, p, n)));
            c->time_model = true;
            WLP_TRY(model_async(*c, model, p, mode, tlp_block, loc.seeds.p, n, o[0], o[1], o[2], st, grid));
            c->time_model = false;
            WLP_CUDA(cudaEventRecord(c->ev1, st));
            int64_t nt = 0;
            WLP_TRY(read_specials(*c, st, me.specials, nt));  // synchronises the stream
            float ms = 0.f;
            WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
            fill_report(*c, model, mode, tlp_block, n, grid, ms, &me.rep);
            me.kernel = g_last_kernel;
        }
        if (!bar.wait()) return fail(WLP_EINTERNAL, peer_failed);
        std::vector<SpecialRec> all;
        for (const DevShard& s : sh) all.insert(all.end(), s.specials.begin(), s.specials.end());
        std::vector<int64_t> next = rej;
        if (all.size() >= 2) WLP_TRY(spacing_rejections(all, rej, next));
        if (!bar.wait()) return fail(WLP_EINTERNAL, peer_failed);  // every slice's specials read
        if (next == rej) break;
        rej.swap(next);
    }
    {
        DevCtx* c;
        std::unique_lock<std::mutex> lk;
        WLP_TRY(acquire(c, lk));
        StreamOrder so(*c, st);
        for (int j = 0; j < nout; ++j) WLP_TRY(stats_device(*c, o[j], n, 1, &me.first[j], st));
    }
    if (!bar.wait()) return fail(WLP_EINTERNAL, peer_failed);
    {
        DevCtx* c;
        std::unique_lock<std::mutex> lk;
        WLP_TRY(acquire(c, lk));
        StreamOrder so(*c, st);
        for (int j = 0; j < nout; ++j) {
            const wlp_stats tot = merged(sh, j, false);
            me.second[j].center = (tot.sum_hi + tot.sum_lo) / static_cast<double>(tot.n);
            WLP_TRY(stats_device(*c, o[j], n, 2, &me.second[j], st));
        }
    }
    for (int j = 0; j < nout; ++j)
        WLP_CUDA(cudaMemcpyAsync(host[j] + me.begin, o[j], n * 8, cudaMemcpyDeviceToHost, st));
    WLP_CUDA(cudaStreamSynchronize(st));
    if (k == 0) rej_out = rej;
    return WLP_OK;
}

}  // namespace
}  // namespace wlp

extern "C" {

int wlp_run_devices(int model, const wlp_params* p, int mode, uint64_t master_seed, int tlp_block_size,
                    const int* devices, int n_devices, double* out0, double* out1, double* out2, wlp_report* report,
                    wlp_ci* ci, double level, char* warn, int warn_cap) {
    WLP_TRY(check_model_mode(model, mode));
    std::string pw, lw;
    WLP_TRY(validate(model, p, &pw));
    WLP_TRY(plan(p->replications, mode, tlp_block_size, 0x7FFFFFFF, nullptr, &lw));
    if (n_devices < 1 || !devices) return fail(WLP_EDOMAIN, "run_devices: need at least one device");
    int have = 0;
    WLP_CUDA(cudaGetDeviceCount(&have));
    for (int k = 0; k < n_devices; ++k)
        if (devices[k] < 0 || devices[k] >= have)
            return fail(WLP_EDOMAIN, "run_devices: device " + std::to_string(devices[k]) + " does not exist (" +
                                         std::to_string(have) + " visible)");
    if (!out0 || (model == WLP_MODEL_MM1 && (!out1 || !out2))) return fail(WLP_EDOMAIN, "run_devices: null output");
    if (ci && !(level > 0.0 && level < 1.0)) return fail(WLP_EDOMAIN, "confidence_interval: level outside (0,1)");
    const int64_t R = p->replications;
    // A run below 2^15 replications per device stays on the first device (the sums are
    // then wlp_run's, bit for bit, and sharding would only add launch latency).
    const int nd = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n_devices, R >> 15)));
    std::vector<DevShard> sh(nd);
    for (int k = 0; k < nd; ++k) {
        sh[k].dev = devices[k];
        sh[k].begin = R * k / nd;
        sh[k].count = R * (k + 1) / nd - sh[k].begin;
    }
    int prev_dev = 0;
    WLP_CUDA(cudaGetDevice(&prev_dev));
    if (nd == 1) {
        WLP_CUDA(cudaSetDevice(devices[0]));
        const int rc = wlp_run(model, p, mode, master_seed, tlp_block_size, out0, out1, out2, 0, nullptr, report, ci,
                               level, warn, warn_cap);
        cudaSetDevice(prev_dev);
        return rc;
    }
    copy_warning(!pw.empty() && !lw.empty() ? pw + "; " + lw : (!pw.empty() ? pw : lw), warn, warn_cap);
    const ThreadSettings ts{g_hw_counters, g_wlp_variant, g_tlp_variant, g_stats_order, g_pipe_lanes};
    const Taus master = master_from_seed(master_seed);
    double* const host[3] = {out0, out1, out2};
    Barrier bar(nd);
    std::vector<int64_t> rej;
    std::vector<std::thread> th;
    for (int k = 0; k < nd; ++k)
        th.emplace_back([&, k] {
            ts.apply();
            sh[k].rc = run_device_shard(model, *p, mode, master, tlp_block_size, sh, k, bar, host, rej);
            if (sh[k].rc != WLP_OK) {
                sh[k].err = g_err;
                bar.abort();
            }
        });
    for (auto& t : th) t.join();
    cudaSetDevice(prev_dev);
    for (const DevShard& s : sh)  // the first real failure (not "another device failed")
        if (s.rc != WLP_OK && s.err != "another device failed") return fail(s.rc, s.err);
    for (const DevShard& s : sh)
        if (s.rc != WLP_OK) return fail(s.rc, s.err);
    g_last_kernel = sh[0].kernel;
    if (ci) {
        for (int j = 0; j < n_outputs(model); ++j) {
            wlp_stats s = merged(sh, j, false);
            const wlp_stats s2 = merged(sh, j, true);
            s.center = (s.sum_hi + s.sum_lo) / static_cast<double>(s.n);
            s.ss_hi = s2.ss_hi;
            s.ss_lo = s2.ss_lo;
            WLP_TRY(ci_from_stats(&s, level, &ci[j]));
        }
    }
    if (report) {
        std::memset(report, 0, sizeof *report);
        for (const DevShard& s : sh) {
            report->kernel_ms = std::max(report->kernel_ms, s.rep.kernel_ms);
            report->total_cycles = std::max(report->total_cycles, s.rep.total_cycles);
            report->waves_executed = std::max(report->waves_executed, s.rep.waves_executed);
            report->peak_resident_warps += s.rep.peak_resident_warps;
            report->divergence_events += s.rep.divergence_events;
            report->mem_reads += s.rep.mem_reads;
            report->mem_writes += s.rep.mem_writes;
        }
    }
    return WLP_OK;
}

int wlp_run_plan(int model, const wlp_params* sets, const uint64_t* master_seeds, int n_sets, int mode,
                 int tlp_block_size, double* out0, double* out1, double* out2, int out_on_device, void* stream,
                 wlp_report* report) {
    WLP_TRY(check_model_mode(model, mode));
    if (n_sets < 1 || !sets || !master_seeds) return fail(WLP_EDOMAIN, "plan: need at least one set");
    std::vector<SetParam> sp(n_sets);
    std::vector<SeedJob> jobs(n_sets);
    int64_t R = 0, blocks = 0;
    bool all_rcp = true;
    const int64_t per_block = static_cast<int64_t>(kSeedBlock) * kSeedJobPer;
    for (int k = 0; k < n_sets; ++k) {
        WLP_TRY(validate(model, &sets[k], nullptr));
        const int64_t n = units_of(model, sets[k]);
        if (n > 0xFFFFFFFFll) return fail(WLP_EPLAN, "plan: units per replication must be < 2^32");
        const DivMode d = model == WLP_MODEL_MM1 ? div_mode(sets[k].lambda, sets[k].mu) : DivMode{kDivIeee, 0.0, 0.0};
        sp[k] = SetParam{R, n, sets[k].chunks, sets[k].lambda, sets[k].mu, d.inv_lambda, d.inv_mu, d.div};
        all_rcp = all_rcp && d.div != kDivIeee;
        jobs[k] = SeedJob{master_from_seed(master_seeds[k]), 0u, sets[k].replications, R, blocks};
        R += sets[k].replications;
        blocks += (sets[k].replications + per_block - 1) / per_block;
    }
    WLP_TRY(plan(R, mode, tlp_block_size, 0x7FFFFFFF, nullptr, nullptr));
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);
    WLP_CUDA(c->seeds.ensure(3 * R));
    // both tables in one upload from pinned staging (a pageable copy is a synchronous
    // staging round trip per call); the stream is synchronised before this call returns,
    // so the staging buffer is free again by the next call
    const size_t jobs_bytes = (n_sets * sizeof(SeedJob) + 255) / 256 * 256;
    const size_t blob = jobs_bytes + n_sets * sizeof(SetParam);
    if (c->h_stage_cap < blob) {
        if (c->h_stage) cudaFreeHost(c->h_stage);
        c->h_stage = nullptr;
        c->h_stage_cap = 0;
        WLP_CUDA(cudaMallocHost(&c->h_stage, blob));
        c->h_stage_cap = blob;
    }
    std::memcpy(c->h_stage, jobs.data(), n_sets * sizeof(SeedJob));
    std::memcpy(c->h_stage + jobs_bytes, sp.data(), n_sets * sizeof(SetParam));
    WLP_CUDA(c->plan_blob.ensure(static_cast<int64_t>(blob)));
    // a plan re-run with the same sets (the usual sweep loop) finds its tables on the device
    if (c->plan_blob_dev != c->plan_blob.p || c->plan_blob_host.size() != blob ||
        std::memcmp(c->plan_blob_host.data(), c->h_stage, blob) != 0) {
        WLP_CUDA(cudaMemcpyAsync(c->plan_blob.p, c->h_stage, blob, cudaMemcpyHostToDevice, st));
        c->plan_blob_host.assign(c->h_stage, c->h_stage + blob);
        c->plan_blob_dev = c->plan_blob.p;
    }
    const SeedJob* d_jobs = reinterpret_cast<const SeedJob*>(c->plan_blob.p);
    const SetParam* d_setp = reinterpret_cast<const SetParam*>(c->plan_blob.p + jobs_bytes);
    double *o0 = out0, *o1 = out1, *o2 = out2;
    if (!out_on_device) {
        WLP_CUDA(c->outs.ensure(3 * R));
        o0 = c->outs.p;
        o1 = c->outs.p + R;
        o2 = c->outs.p + 2 * R;
    }
    // one batched seeding launch for all sets, and the model right behind it (PDL: its
    // prologue overlaps the seeding); the spacing check below re-runs the model only when
    // two special candidates share a key. The seeding zeroes the model's grab counter
    // (counter[4]), reports the specials count through mapped host memory and clears
    // counter[3] behind it, so no memset or copy launch brackets the plan.
    c->spec_read = 3;
    c->spec_mapped = true;
    *reinterpret_cast<volatile unsigned long long*>(c->h_mapped) = kCountPending;
    WLP_CUDA(launch_seed_jobs(c->powers.p, d_jobs, n_sets, blocks, R, c->seeds.p, c->specials.p, kSpecialCap,
                              c->counter.p + 3, st, c->counter.p + 4, c->seed_done.p, c->d_mapped));
    PlanArgs pa;
    pa.serial_rho = mm1_serial_rho();
    pa.tlp_div = all_rcp ? kDivRcp : kDivIeee;
    pa.seeds = c->seeds.p;
    pa.count = R;
    pa.sets = d_setp;
    pa.n_sets = n_sets;
    pa.out0 = o0;
    pa.out1 = o1;
    pa.out2 = o2;
    pa.next = c->counter.p + 4;
    const int wpb = (model == WLP_MODEL_MM1 ? kMm1Block : kWlpBlock) / 32;
    const int grid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(static_cast<int64_t>(c->sms) * c->plan_bps[model], (R + wpb - 1) / wpb)));
    bool first = true, first_pdl = true;
    auto run_model_launch = [&]() -> int {
        if (!first) WLP_CUDA(cudaMemsetAsync(pa.next, 0, 8, st));  // (the first was cleared with the count)
        first = false;
        if (report) WLP_CUDA(cudaEventRecord(c->ev0, st));
        set_pdl_launch(!report && first_pdl);  // (directly behind the seeding, not timed)
        const cudaError_t e = launch_plan(model, mode, pa, c->plan_lane.p, c->plan_skip.p, c->mm1_lane.p,
                                          c->mm1_skip.p, grid, tlp_block_size, st);
        set_pdl_launch(false);
        first_pdl = false;
        WLP_CUDA(e);
        if (report) WLP_CUDA(cudaEventRecord(c->ev1, st));
        return WLP_OK;
    };
    WLP_TRY(run_model_launch());
    std::vector<SpecialRec> specials;
    int64_t nt = 0;
    // into device buffers without a report the call returns once the seeding has reported
    // its specials count; the model keeps running on the stream
    WLP_TRY(read_specials(*c, st, specials, nt, out_on_device && !report));
    // per set, a key collision (only ever between special candidates) re-seeds that set
    // exactly with its rejection list
    std::map<uint32_t, std::vector<SpecialRec>> by_job;
    for (const SpecialRec& s : specials) by_job[s.pad].push_back(s);
    bool reseeded = false;
    for (auto& kv : by_job) {
        if (kv.second.size() < 2) continue;
        const int k = static_cast<int>(kv.first);
        std::vector<int64_t> rej, next;
        WLP_TRY(spacing_rejections(kv.second, rej, next));
        while (next != rej) {  // re-seed set k in place (its slice of the SoA) until no new redraw
            reseeded = true;
            rej.swap(next);
            WLP_CUDA(c->rejected.ensure(static_cast<int64_t>(rej.size())));
            WLP_CUDA(cudaMemcpyAsync(c->rejected.p, rej.data(), rej.size() * 8, cudaMemcpyHostToDevice, st));
            WLP_CUDA(cudaMemsetAsync(c->counter.p + 3, 0, 8, st));
            c->spec_read = 3;
            c->spec_mapped = false;
            SeedArgs a{};
            a.powers = c->powers.p;
            a.master = jobs[k].master;
            a.slot_begin = 0;
            a.count = jobs[k].count;
            a.rejected = c->rejected.p;
            a.n_rejected = static_cast<int64_t>(rej.size());
            a.out = c->seeds.p;
            a.out_off = jobs[k].out_off;
            a.stride = R;
            a.specials = c->specials.p;
            a.special_cap = kSpecialCap;
            a.n_special = c->counter.p + 3;
            WLP_CUDA(launch_seed(a, st));
            std::vector<SpecialRec> sp2;
            int64_t n2 = 0;
            WLP_TRY(read_specials(*c, st, sp2, n2));
            WLP_TRY(spacing_rejections(sp2, rej, next));
        }
    }
    if (reseeded) {
        WLP_CUDA(cudaMemsetAsync(c->counter.p + 3, 0, 8, st));  // (the plan seeding expects it zero)
        WLP_TRY(run_model_launch());
    }
    if (!out_on_device) {
        WLP_CUDA(cudaMemcpyAsync(out0, o0, R * 8, cudaMemcpyDeviceToHost, st));
        if (model == WLP_MODEL_MM1) {
            WLP_CUDA(cudaMemcpyAsync(out1, o1, R * 8, cudaMemcpyDeviceToHost, st));
            WLP_CUDA(cudaMemcpyAsync(out2, o2, R * 8, cudaMemcpyDeviceToHost, st));
        }
    }
    if (report || !out_on_device) WLP_CUDA(cudaStreamSynchronize(st));
    if (report) {
        float ms = 0.f;
        WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        const int g = mode == WLP_MODE_TLP ? static_cast<int>((R + std::min<int64_t>(R, tlp_block_size) - 1) /
                                                              std::min<int64_t>(R, tlp_block_size))
                                           : grid;
        fill_report(*c, model, mode, tlp_block_size, R, g, ms, report);
    }
    return WLP_OK;
}

int wlp_stats_device(const double* x, int64_t n, int pass, wlp_stats* stats, void* stream) {
    if (n < 1) return fail(WLP_EDOMAIN, "stats: empty input");
    if (pass != 1 && pass != 2) return fail(WLP_EDOMAIN, "stats: pass must be 1 or 2");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    StreamOrder so(*c, static_cast<cudaStream_t>(stream));
    return stats_device(*c, x, n, pass, stats, static_cast<cudaStream_t>(stream));
}

int wlp_confidence_interval(const double* samples, int64_t n, double level, wlp_ci* ci) {
    if (n < 2) return fail(WLP_EDOMAIN, "confidence_interval: need at least 2 samples");
    if (!(level > 0.0 && level < 1.0)) return fail(WLP_EDOMAIN, "confidence_interval: level outside (0,1)");
    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    StreamOrder so(*c, nullptr);
    WLP_CUDA(c->stats_in.ensure(n));
    WLP_CUDA(cudaMemcpy(c->stats_in.p, samples, n * 8, cudaMemcpyHostToDevice));
    return ci_device(*c, c->stats_in.p, n, level, ci, nullptr);
}

// ---- kernel IR interpreter ---------------------------------------------------------

}  // extern "C"

namespace wlp {
namespace {

// Structural check of a flattened program, so that nothing malformed reaches the device:
// every index in range, every expression well formed, stack within WLP_IR_MAX_STACK.
int ir_check(const wlp_ir_program& p) {
    auto bad = [](const std::string& m) { return fail(WLP_EDOMAIN, "ir program: " + m); };
    if (p.n_stmts < 0 || p.n_code < 1 || !p.code || (p.n_stmts > 0 && !p.stmts)) return bad("empty tables");
    if (p.n_locals < 0 || p.n_locals > WLP_IR_MAX_LOCALS)
        return bad("more than " + std::to_string(WLP_IR_MAX_LOCALS) + " locals");
    if (p.n_params < 0 || (p.n_params > 0 && (!p.param_bits || !p.param_is_array))) return bad("params");
    if (p.n_locals > 0 && !p.local_init) return bad("local_init");
    // expressions: walk the code, each expression ends with END at stack depth 1
    std::vector<char> starts(p.n_code, 0);
    for (int pc = 0; pc < p.n_code;) {
        starts[pc] = 1;
        int depth = 0;
        for (;;) {
            if (pc >= p.n_code) return bad("unterminated expression");
            const int op = p.code[pc++];
            int need = 0, push = 0, args = 0;
            switch (op) {
                case WLP_IR_OP_END: need = 1; break;
                case WLP_IR_OP_CONST: push = 1; args = 2; break;
                case WLP_IR_OP_LOCAL: case WLP_IR_OP_PARAM: case WLP_IR_OP_SREG: push = 1; args = 1; break;
                case WLP_IR_OP_DRAW: push = 1; break;
                case WLP_IR_OP_I2R_0: case WLP_IR_OP_TRUTH_0: case WLP_IR_OP_NEG_I: case WLP_IR_OP_NEG_R:
                case WLP_IR_OP_LOG: case WLP_IR_OP_FLOOR: need = 1; break;
                case WLP_IR_OP_I2R_1: case WLP_IR_OP_TRUTH_1: need = 2; break;
                default:
                    if (op < WLP_IR_OP_ADD_I || op >= WLP_IR_OP_COUNT) return bad("unknown opcode " + std::to_string(op));
                    need = 2;
                    push = -1;
                    break;
            }
            if (pc + args > p.n_code) return bad("truncated operand");
            if (op == WLP_IR_OP_LOCAL && (p.code[pc] < 0 || p.code[pc] >= p.n_locals)) return bad("local slot");
            if (op == WLP_IR_OP_PARAM &&
                (p.code[pc] < 0 || p.code[pc] >= p.n_params || p.param_is_array[p.code[pc]]))
                return bad("param slot");
            if (op == WLP_IR_OP_SREG && (p.code[pc] < 0 || p.code[pc] > 10)) return bad("special register");
            pc += args;
            if (depth < need) return bad("stack underflow");
            if (op == WLP_IR_OP_END) {
                if (depth != 1) return bad("expression leaves " + std::to_string(depth) + " values");
                break;
            }
            depth += push;
            if (depth > WLP_IR_MAX_STACK)
                return bad("expression deeper than " + std::to_string(WLP_IR_MAX_STACK) + " values");
        }
    }
    auto expr_ok = [&](int off) { return off >= 0 && off < p.n_code && starts[off]; };
    auto range_ok = [&](int b, int e) { return 0 <= b && b <= e && e <= p.n_stmts; };
    if (!range_ok(p.top_begin, p.top_end)) return bad("body range");
    for (int i = 0; i < p.n_stmts; ++i) {
        const wlp_ir_stmt& st = p.stmts[i];
        const bool arr_slot = st.slot >= 0 && st.slot < p.n_params && p.param_is_array[st.slot];
        switch (st.kind) {
            case WLP_IR_ASSIGN:
                if (st.slot < 0 || st.slot >= p.n_locals || !expr_ok(st.code_a)) return bad("assign");
                break;
            case WLP_IR_LOAD:
                if (st.slot < 0 || st.slot >= p.n_locals || st.arr < 0 || st.arr >= p.n_params ||
                    !p.param_is_array[st.arr] || !expr_ok(st.code_a))
                    return bad("load");
                break;
            case WLP_IR_STORE:
                if (!arr_slot || !expr_ok(st.code_a) || !expr_ok(st.code_b)) return bad("store");
                break;
            case WLP_IR_IF:
                if (!expr_ok(st.code_a) || !range_ok(st.b1_begin, st.b1_end) || !range_ok(st.b2_begin, st.b2_end))
                    return bad("if");
                break;
            case WLP_IR_WHILE:
                if (!expr_ok(st.code_a) || !range_ok(st.b1_begin, st.b1_end)) return bad("while");
                break;
            case WLP_IR_HALT: break;
            default: return bad("statement kind");
        }
    }
    // The body ranges must form a tree: walked from the top range, every statement is
    // reached at most once (a range containing its own IF/WHILE, or two overlapping
    // ranges, reaches one twice) and nesting stays below kMaxNest, so the interpreter
    // and the JIT generator's recursion (ir_jit.cu list()/stmt()) always terminate.
    constexpr int kMaxNest = 1024;
    std::vector<char> seen(p.n_stmts, 0);
    struct Range { int b, e, depth; };
    std::vector<Range> todo{{p.top_begin, p.top_end, 0}};
    while (!todo.empty()) {
        const Range r = todo.back();
        todo.pop_back();
        if (r.depth > kMaxNest) return bad("bodies nested deeper than " + std::to_string(kMaxNest));
        for (int i = r.b; i < r.e; ++i) {
            if (seen[i]) return bad("statement " + std::to_string(i) + " reached twice (body ranges overlap)");
            seen[i] = 1;
            const wlp_ir_stmt& st = p.stmts[i];
            if (st.kind == WLP_IR_IF || st.kind == WLP_IR_WHILE) todo.push_back({st.b1_begin, st.b1_end, r.depth + 1});
            if (st.kind == WLP_IR_IF) todo.push_back({st.b2_begin, st.b2_end, r.depth + 1});
        }
    }
    return WLP_OK;
}

std::string ir_fault_message(const IrFault& f, int mask_depth) {
    const std::string a = std::to_string(f.a), b = std::to_string(f.b);
    switch (f.code) {  // the reference's messages (kernel_ir.cpp:46-107, warp_exec.cpp)
        case 1: return "kernel: integer division by zero";
        case 2: return "kernel: division by zero";
        case 3: return "kernel: integer modulo by zero";
        case 4: return "kernel: modulo by zero";
        case 5: return "kernel: log of a non-positive value";
        case 6: return "kernel: floor result outside the integer range";
        case 7: return "load: non-integer index";
        case 8: return "load: index " + a + " out of bounds for array of " + b;
        case 9: return "store: non-integer index";
        case 10: return "store: index " + a + " out of bounds for array of " + b;
        case 11: return "assign: real value into int local #" + a;
        case 12: return "mask stack overflow: nesting deeper than " + std::to_string(mask_depth) + " levels";
        case 13: return "issue budget exhausted: an IR warp issued " + a + " statements";
    }
    return "kernel: fault " + std::to_string(f.code);
}

template <class T>
struct Scratch {  // per-call device allocation
    T* p = nullptr;
    ~Scratch() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(int64_t n) { return cudaMalloc(&p, static_cast<size_t>(std::max<int64_t>(n, 1)) * sizeof(T)); }
};

}  // namespace
}  // namespace wlp

namespace wlp {
std::string ir_jit_source(const wlp_ir_program& p);
int ir_jit_kernel(const wlp_ir_program& p, int device, void** kernel, std::string& err);
namespace {

int ir_run(const wlp_ir_program* prog, const wlp_launch_cfg* cfg, int64_t max_threads_per_block,
           double* const* arrays, const int64_t* array_len, int arrays_on_device, const uint32_t* streams,
           int64_t n_streams, int streams_on_device, int mask_depth, int64_t max_issues, void* stream,
           wlp_report* report, bool jit) {
    if (!prog || !cfg) return fail(WLP_EDOMAIN, "ir_simulate: null program or launch");
    if (cfg->block_x < 1 || cfg->block_y < 1 || cfg->block_z < 1)
        return fail(WLP_EDOMAIN, "launch: blockDim components must be >= 1");
    if (cfg->grid_x < 1 || cfg->grid_y < 1) return fail(WLP_EDOMAIN, "launch: gridDim components must be >= 1");
    if (cfg->warp_size < 1 || cfg->warp_size > 64) return fail(WLP_EDOMAIN, "launch: warpSize must be in [1,64]");
    if (cfg->warp_size > 32)
        return fail(WLP_EDOMAIN, "launch: the B200 interpreter maps an IR warp onto one hardware warp; warpSize "
                                 "must be <= 32");
    if (mask_depth < 1 || mask_depth > 64) return fail(WLP_EDOMAIN, "mask stack depth must be in [1, 64]");
    if (max_issues < 1) return fail(WLP_EDOMAIN, "ir_simulate: max_issues must be >= 1");
    const int64_t tpb = cfg->block_x * cfg->block_y * cfg->block_z;
    if (tpb > max_threads_per_block)
        return fail(WLP_EPLAN, "block of " + std::to_string(tpb) + " threads exceeds maxThreadsPerBlock " +
                                   std::to_string(max_threads_per_block));
    if (n_streams < 0 || (n_streams > 0 && !streams)) return fail(WLP_EDOMAIN, "ir_simulate: streams");
    WLP_TRY(ir_check(*prog));
    for (int i = 0; i < prog->n_params; ++i)
        if (prog->param_is_array[i] && (!array_len || array_len[i] < 0 || (array_len[i] > 0 && !arrays[i])))
            return fail(WLP_EDOMAIN, "ir_simulate: array argument #" + std::to_string(i));
    const int64_t ws = cfg->warp_size;
    const int64_t wpb = (tpb + ws - 1) / ws;
    const int64_t total_warps = wpb * cfg->grid_x * cfg->grid_y;

    DevCtx* c;
    std::unique_lock<std::mutex> lk;
    WLP_TRY(acquire(c, lk));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamOrder so(*c, st);

    const int np = std::max(prog->n_params, 1);
    Scratch<wlp_ir_stmt> d_stmts;
    Scratch<int32_t> d_code;
    Scratch<int64_t> d_init, d_params, d_alen;
    Scratch<double*> d_arrs;
    Scratch<uint32_t> d_streams;
    Scratch<unsigned long long> d_cnt;
    Scratch<IrFault> d_fault;
    std::vector<Scratch<double>> host_arrays(np);
    WLP_CUDA(d_stmts.alloc(prog->n_stmts));
    WLP_CUDA(d_code.alloc(prog->n_code));
    WLP_CUDA(d_init.alloc(prog->n_locals));
    WLP_CUDA(d_params.alloc(np));
    WLP_CUDA(d_alen.alloc(np));
    WLP_CUDA(d_arrs.alloc(np));
    WLP_CUDA(d_cnt.alloc(5));
    WLP_CUDA(d_fault.alloc(1));
    if (prog->n_stmts)
        WLP_CUDA(cudaMemcpyAsync(d_stmts.p, prog->stmts, prog->n_stmts * sizeof(wlp_ir_stmt), cudaMemcpyHostToDevice, st));
    WLP_CUDA(cudaMemcpyAsync(d_code.p, prog->code, prog->n_code * 4, cudaMemcpyHostToDevice, st));
    if (prog->n_locals)
        WLP_CUDA(cudaMemcpyAsync(d_init.p, prog->local_init, prog->n_locals * 8, cudaMemcpyHostToDevice, st));
    std::vector<int64_t> pbits(np, 0), alen(np, 0);
    std::vector<double*> aptr(np, nullptr);
    for (int i = 0; i < prog->n_params; ++i) {
        if (!prog->param_is_array[i]) {
            pbits[i] = prog->param_bits[i];
            continue;
        }
        alen[i] = array_len[i];
        if (arrays_on_device) {
            aptr[i] = arrays[i];
        } else if (alen[i] > 0) {
            WLP_CUDA(host_arrays[i].alloc(alen[i]));
            WLP_CUDA(cudaMemcpyAsync(host_arrays[i].p, arrays[i], alen[i] * 8, cudaMemcpyHostToDevice, st));
            aptr[i] = host_arrays[i].p;
        }
    }
    WLP_CUDA(cudaMemcpyAsync(d_params.p, pbits.data(), np * 8, cudaMemcpyHostToDevice, st));
    WLP_CUDA(cudaMemcpyAsync(d_alen.p, alen.data(), np * 8, cudaMemcpyHostToDevice, st));
    WLP_CUDA(cudaMemcpyAsync(d_arrs.p, aptr.data(), np * sizeof(double*), cudaMemcpyHostToDevice, st));
    const uint32_t* ds = streams;
    if (n_streams > 0 && !streams_on_device) {
        WLP_CUDA(d_streams.alloc(3 * n_streams));
        WLP_CUDA(cudaMemcpyAsync(d_streams.p, streams, 3 * n_streams * 4, cudaMemcpyHostToDevice, st));
        ds = d_streams.p;
    }
    WLP_CUDA(cudaMemsetAsync(d_cnt.p, 0, 5 * sizeof(unsigned long long), st));
    WLP_CUDA(cudaMemsetAsync(d_fault.p, 0, sizeof(IrFault), st));

    IrArgs a{};
    a.stmts = d_stmts.p;
    a.code = d_code.p;
    a.top_begin = prog->top_begin;
    a.top_end = prog->top_end;
    a.n_locals = prog->n_locals;
    a.local_init = d_init.p;
    a.params = d_params.p;
    a.arrays = d_arrs.p;
    a.alen = d_alen.p;
    a.streams = ds;
    a.n_streams = n_streams;
    a.bx = cfg->block_x;
    a.by = cfg->block_y;
    a.bz = cfg->block_z;
    a.gx = cfg->grid_x;
    a.gy = cfg->grid_y;
    a.ws = ws;
    a.tpb = tpb;
    a.wpb = wpb;
    a.total_warps = total_warps;
    a.mask_depth = mask_depth;
    a.max_issues = max_issues;
    a.counters = d_cnt.p;
    a.fault = d_fault.p;
    int64_t resident_blocks = static_cast<int64_t>(ir_blocks_per_sm()) * c->sms;
    void* jk = nullptr;
    if (jit) {
        std::string err;
        const int rc = ir_jit_kernel(*prog, c->dev, &jk, err);
        if (rc != WLP_OK) return fail(rc, err);
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, jk, kIrBlock, 0) != cudaSuccess || nb < 1) nb = 4;
        resident_blocks = static_cast<int64_t>(nb) * c->sms;
    }
    const int64_t need_blocks = (total_warps * 32 + kIrBlock - 1) / kIrBlock;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min(resident_blocks, need_blocks)));
    WLP_CUDA(cudaEventRecord(c->ev0, st));
    if (jit) {
        // wlp_ir_jit(P, A, AL, S, nS, bx, by, bz, gx, gy, ws, tpb, wpb, total_warps, max_iters, fault)
        const int64_t* P_ = d_params.p;
        double* const* A_ = d_arrs.p;
        const int64_t* AL_ = d_alen.p;
        const uint32_t* S_ = ds;
        long long nS = n_streams, bx = a.bx, by = a.by, bz = a.bz, gx = a.gx, gy = a.gy, wsz = ws, tp = tpb,
                  wp = wpb, tw = total_warps, mi = max_issues;
        IrFault* F_ = d_fault.p;
        void* args[] = {&P_, &A_, &AL_, &S_, &nS, &bx, &by, &bz, &gx, &gy, &wsz, &tp, &wp, &tw, &mi, &F_};
        WLP_CUDA(cudaLaunchKernel(jk, dim3(grid), dim3(kIrBlock), args, 0, st));
    } else {
        WLP_CUDA(launch_ir(a, grid, st));
    }
    WLP_CUDA(cudaEventRecord(c->ev1, st));
    if (!arrays_on_device)
        for (int i = 0; i < prog->n_params; ++i)
            if (prog->param_is_array[i] && alen[i] > 0)
                WLP_CUDA(cudaMemcpyAsync(arrays[i], aptr[i], alen[i] * 8, cudaMemcpyDeviceToHost, st));
    unsigned long long cnt[5];
    IrFault fault{};
    WLP_CUDA(cudaMemcpyAsync(cnt, d_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
    WLP_CUDA(cudaMemcpyAsync(&fault, d_fault.p, sizeof fault, cudaMemcpyDeviceToHost, st));
    WLP_CUDA(cudaStreamSynchronize(st));
    if (fault.code != 0) return fail(WLP_EFAULT, ir_fault_message(fault, mask_depth));
    if (report) {
        float ms = 0.f;
        WLP_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
        std::memset(report, 0, sizeof *report);
        report->kernel_ms = ms;
        report->total_cycles = static_cast<int64_t>(std::llround(static_cast<double>(ms) * c->clock_khz));
        const int64_t resident_warps = resident_blocks * (kIrBlock / 32);
        report->waves_executed = (total_warps + resident_warps - 1) / resident_warps;
        report->peak_resident_warps = std::min(total_warps, resident_warps);
        if (!jit) {  // the JIT has no lockstep accounting
            report->issues = cnt[0];
            report->alu_issues = cnt[1];
            report->mem_reads = cnt[2];
            report->mem_writes = cnt[3];
            report->divergence_events = cnt[4];
        }
    }
    return WLP_OK;
}

}  // namespace
}  // namespace wlp

extern "C" {

int wlp_ir_simulate(const wlp_ir_program* prog, const wlp_launch_cfg* cfg, int64_t max_threads_per_block,
                    double* const* arrays, const int64_t* array_len, int arrays_on_device,
                    const uint32_t* streams, int64_t n_streams, int streams_on_device, int mask_depth,
                    int64_t max_issues, void* stream, wlp_report* report) {
    return wlp::ir_run(prog, cfg, max_threads_per_block, arrays, array_len, arrays_on_device, streams, n_streams,
                       streams_on_device, mask_depth, max_issues, stream, report, false);
}

int wlp_ir_jit_simulate(const wlp_ir_program* prog, const wlp_launch_cfg* cfg, int64_t max_threads_per_block,
                        double* const* arrays, const int64_t* array_len, int arrays_on_device,
                        const uint32_t* streams, int64_t n_streams, int streams_on_device, int64_t max_iterations,
                        void* stream, wlp_report* report) {
    return wlp::ir_run(prog, cfg, max_threads_per_block, arrays, array_len, arrays_on_device, streams, n_streams,
                       streams_on_device, 32, max_iterations, stream, report, true);
}

int wlp_ir_jit_source(const wlp_ir_program* prog, char* out, int cap, int* need) {
    if (!prog) return fail(WLP_EDOMAIN, "ir_jit_source: null program");
    WLP_TRY(wlp::ir_check(*prog));
    const std::string src = wlp::ir_jit_source(*prog);
    if (need) *need = static_cast<int>(src.size()) + 1;
    if (out && cap > 0) {
        const size_t k = std::min<size_t>(src.size(), static_cast<size_t>(cap - 1));
        std::memcpy(out, src.data(), k);
        out[k] = 0;
    }
    return WLP_OK;
}

int wlp_shutdown(void) {
    std::lock_guard<std::mutex> g(g_ctx_mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return WLP_OK;
    auto it = g_ctx.find(dev);
    if (it == g_ctx.end()) return WLP_OK;
    DevCtx& c = *it->second;
    std::lock_guard<std::mutex> lk(c.mu);
    cudaDeviceSynchronize();
    c.powers.release();
    for (auto& kv : c.lane_tabs) kv.second.release();
    c.lane_tabs.clear();
    c.mm1_lane.release();
    c.mm1_skip.release();
    c.seeds.release();
    c.in_seeds.release();
    c.outs.release();
    c.partials.release();
    c.stats_in.release();
    c.specials.release();
    c.counter.release();
    c.rejected.release();
    if (c.ev0) cudaEventDestroy(c.ev0);
    if (c.ev1) cudaEventDestroy(c.ev1);
    if (c.done) cudaEventDestroy(c.done);
    c.ev0 = c.ev1 = c.done = nullptr;
    c.last_used = false;
    c.work.release();
    if (c.h_counter) cudaFreeHost(c.h_counter);
    c.h_counter = nullptr;
    if (c.h_mapped) cudaFreeHost(c.h_mapped);
    c.h_mapped = nullptr;
    c.seed_done.release();
    if (c.h_stage) cudaFreeHost(c.h_stage);
    c.h_stage = nullptr;
    c.h_stage_cap = 0;
    c.plan_blob.release();
    c.hw.release();
    c.jobs.release();
    c.setp.release();
    c.plan_lane.release();
    c.plan_skip.release();
    c.ready = false;
    return WLP_OK;
}

}  // extern "C"
