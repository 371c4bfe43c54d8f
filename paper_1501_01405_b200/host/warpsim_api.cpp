// C++ drop-in API (include/warpsim_b200.hpp) over the C ABI of libwlp_b200.so.
// Every model computation is a C-ABI call into the sm_100a kernels; this file holds only
// argument plumbing and the reference's error mapping (the sweep and its CSV form are in
// sweep.cpp).
#include <cstring>

#include "warpsim_b200.hpp"
#include "warpsim_ir_b200.hpp"
#include "wlp_b200.h"

namespace warpsim {
namespace {

[[noreturn]] void raise(int code) {
    const std::string msg = wlp_last_error();
    switch (code) {
        case WLP_EDOMAIN: throw DomainError(msg);
        case WLP_EPLAN: throw PlanError(msg);
        case WLP_EFAULT: throw FaultError(msg);
        default: throw Error(msg);
    }
}

void check(int code) {
    if (code != WLP_OK) raise(code);
}

wlp_params to_c(const ModelParams& p) {
    return wlp_params{p.replications, p.draws, p.clients, p.lambda, p.mu, p.steps, p.chunks};
}

int model_id(ModelKind m) { return m == ModelKind::Pi ? WLP_MODEL_PI : m == ModelKind::Mm1 ? WLP_MODEL_MM1 : WLP_MODEL_WALK; }
int mode_id(ExecutionMode m) {
    return m == ExecutionMode::Sequential ? WLP_MODE_SEQUENTIAL : m == ExecutionMode::Tlp ? WLP_MODE_TLP : WLP_MODE_WLP;
}

SimReport from_c(const wlp_report& r) {
    SimReport s;
    s.totalCycles = r.total_cycles;
    s.wavesExecuted = r.waves_executed;
    s.peakResidentWarps = r.peak_resident_warps;
    s.issues = r.issues;
    s.aluIssues = r.alu_issues;
    s.memReads = r.mem_reads;
    s.memWrites = r.mem_writes;
    s.divergenceEvents = r.divergence_events;
    s.kernelMs = r.kernel_ms;
    s.warpSplits = r.warp_splits;
    return s;
}

std::vector<std::uint32_t> soa(const RngState& s) { return {s.s1, s.s2, s.s3}; }

}  // namespace

const char* mode_name(ExecutionMode mode) {
    switch (mode) {
        case ExecutionMode::Sequential: return "sequential";
        case ExecutionMode::Tlp: return "tlp";
        case ExecutionMode::Wlp: return "wlp";
    }
    return "?";
}

ExecutionMode mode_from_name(const std::string& name) {
    if (name == "sequential") return ExecutionMode::Sequential;
    if (name == "tlp") return ExecutionMode::Tlp;
    if (name == "wlp") return ExecutionMode::Wlp;
    throw DomainError("unknown execution mode '" + name + "' (sequential|tlp|wlp)");
}

const char* model_name(ModelKind model) {
    switch (model) {
        case ModelKind::Pi: return "pi";
        case ModelKind::Mm1: return "mm1";
        case ModelKind::Walk: return "walk";
    }
    return "?";
}

ModelKind model_from_name(const std::string& name) {
    if (name == "pi") return ModelKind::Pi;
    if (name == "mm1") return ModelKind::Mm1;
    if (name == "walk") return ModelKind::Walk;
    throw DomainError("unknown model '" + name + "' (pi|mm1|walk)");
}

RngState make_rng_state(std::uint32_t s1, std::uint32_t s2, std::uint32_t s3) {
    std::uint32_t o[3];
    check(wlp_make_state(s1, s2, s3, o));
    return RngState{o[0], o[1], o[2]};
}

RngState rng_state_from_seed(std::uint64_t seed) {
    std::uint32_t o[3];
    check(wlp_master_from_seed(seed, o));
    return RngState{o[0], o[1], o[2]};
}

std::vector<RngState> random_spacing(RngState& master, std::size_t count) {
    std::vector<std::uint32_t> keys(3 * count);
    const std::uint32_t m[3] = {master.s1, master.s2, master.s3};
    std::uint32_t after[3];
    check(wlp_seed_streams_state(m, static_cast<std::int64_t>(count), count ? keys.data() : nullptr, 0, nullptr,
                                 after));
    master = RngState{after[0], after[1], after[2]};
    std::vector<RngState> out(count);
    for (std::size_t i = 0; i < count; ++i) out[i] = RngState{keys[i], keys[count + i], keys[2 * count + i]};
    return out;
}

std::vector<std::uint32_t> taus_stream(RngState& state, std::size_t n) {
    std::vector<std::uint32_t> out(n);
    // state is taken as-is (already a valid state); make_rng_state would only re-map
    check(wlp_taus_stream(state.s1, state.s2, state.s3, static_cast<std::int64_t>(n), n ? out.data() : nullptr, 0,
                          nullptr));
    const std::uint32_t s[3] = {state.s1, state.s2, state.s3};
    std::uint32_t o[3];
    check(wlp_jump_host(s, n, o));
    state = RngState{o[0], o[1], o[2]};
    return out;
}

std::uint32_t taus_next(RngState& state) {
    std::uint32_t s[3] = {state.s1, state.s2, state.s3}, out = 0;
    check(wlp_taus_next(s, &out));
    state = RngState{s[0], s[1], s[2]};
    return out;
}

double uniform01(RngState& state) { return taus_next(state) * 0x1p-32; }

double exponential_from_u(double u, double rate) {
    double out = 0.0;
    check(wlp_exponential_from_u(u, rate, &out));
    return out;
}

double exponential(RngState& state, double rate) { return exponential_from_u(uniform01(state), rate); }

int device_count() {
    int n = 0;
    check(wlp_device_count(&n));
    return n;
}

namespace detail {

void check_u(ModelKind model, std::int64_t units, std::int64_t chunks, double lambda, double mu) {
    ModelParams p;
    p.replications = 1;
    p.draws = p.clients = p.steps = units;
    p.chunks = model == ModelKind::Walk ? chunks : 2;
    p.lambda = model == ModelKind::Mm1 ? lambda : 0.5;
    p.mu = model == ModelKind::Mm1 ? mu : 1.0;
    const wlp_params c = to_c(p);
    check(wlp_validate_params(model_id(model), &c, nullptr, 0));
}

std::vector<double> run_u(ModelKind model, std::int64_t units, std::int64_t chunks, double lambda, double mu,
                          const std::vector<double>& u) {
    ModelParams p;
    p.draws = p.clients = p.steps = units;
    p.chunks = model == ModelKind::Walk ? chunks : 2;
    p.lambda = model == ModelKind::Mm1 ? lambda : 0.5;
    p.mu = model == ModelKind::Mm1 ? mu : 1.0;
    const wlp_params c = to_c(p);
    std::vector<double> o(3, 0.0);
    check(wlp_run_uniforms(model_id(model), &c, u.data(), 1, 0, &o[0], &o[1], &o[2], 0, nullptr));
    return o;
}

}  // namespace detail

LaunchPlan plan_launch(std::int64_t replications, ExecutionMode mode, const DeviceProfile& prof, int tlp_block_size,
                       std::int64_t grid_limit) {
    // the reference's order (wlp.cpp:73-76); the C layer adds CUDA's 1024-thread limit
    if (replications < 1) throw PlanError("plan_launch: need at least one replication");
    if (tlp_block_size < 1) throw PlanError("plan_launch: tlp_block_size must be >= 1");
    if (tlp_block_size > prof.maxThreadsPerBlock)
        throw PlanError("plan_launch: tlp_block_size exceeds maxThreadsPerBlock");
    wlp_launch_cfg c{};
    char warn[512];
    check(wlp_plan_launch(replications, mode_id(mode), tlp_block_size, grid_limit, &c, warn, sizeof warn));
    LaunchPlan plan;
    plan.cfg.blockDim = Dim3{c.block_x, c.block_y, c.block_z};
    plan.cfg.gridDim = Dim2{c.grid_x, c.grid_y};
    plan.cfg.warpSize = c.warp_size;
    plan.replications = replications;
    plan.mode = mode;
    if (warn[0]) plan.warning = std::string(warn);
    return plan;
}

std::optional<std::string> validate_params(ModelKind model, const ModelParams& p) {
    const wlp_params c = to_c(p);
    char warn[512];
    check(wlp_validate_params(model_id(model), &c, warn, sizeof warn));
    if (warn[0]) return std::string(warn);
    return std::nullopt;
}

namespace {
std::vector<std::vector<double>> run_one(ModelKind model, const ModelParams& p, RngState stream) {
    const auto s = soa(stream);
    const wlp_params c = to_c(p);
    const int nout = model == ModelKind::Mm1 ? 3 : 1;
    std::vector<std::vector<double>> o(3, std::vector<double>(1));
    check(wlp_run_streams(model_id(model), &c, WLP_MODE_WLP, s.data(), 1, 0, o[0].data(),
                          nout > 1 ? o[1].data() : nullptr, nout > 1 ? o[2].data() : nullptr, 0, nullptr, nullptr));
    return o;
}
}  // namespace

double pi_replication(std::int64_t draws, RngState stream) {
    ModelParams p;
    p.draws = draws;
    return run_one(ModelKind::Pi, p, stream)[0][0];
}

MM1Result mm1_replication(std::int64_t clients, double lambda, double mu, RngState stream) {
    ModelParams p;
    p.clients = clients;
    p.lambda = lambda;
    p.mu = mu;
    auto o = run_one(ModelKind::Mm1, p, stream);
    return MM1Result{o[0][0], o[1][0], o[2][0]};
}

double walk_replication(std::int64_t steps, std::int64_t chunks, RngState stream) {
    ModelParams p;
    p.steps = steps;
    p.chunks = chunks;
    return run_one(ModelKind::Walk, p, stream)[0][0];
}

double inverse_normal_cdf(double p) {
    double z = 0.0;
    check(wlp_inverse_normal_cdf(p, &z));
    return z;
}

ConfidenceInterval confidence_interval(const std::vector<double>& samples, double level) {
    wlp_ci ci{};
    check(wlp_confidence_interval(samples.empty() ? nullptr : samples.data(), static_cast<std::int64_t>(samples.size()),
                                  level, &ci));
    return ConfidenceInterval{ci.mean, ci.half_width, ci.level, ci.n, ci.warn_small_sample != 0};
}

ModelRun run_model(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                   std::uint64_t master_seed, int tlp_block_size, const SimOptions& opts) {
    struct Counters {  // scoped wlp_set_hw_counters
        bool on;
        explicit Counters(bool o) : on(o) {
            if (on) wlp_set_hw_counters(1);
        }
        ~Counters() {
            if (on) wlp_set_hw_counters(0);
        }
    } counters(opts.hardwareCounters);
    if (opts.irInterpreter)  // the reference's IR kernels (and its Sequential accounting), on the GPU
        return run_model_ir(model, p, mode, prof, master_seed, tlp_block_size, opts);
    const LaunchPlan plan = plan_launch(p.replications, mode, prof, tlp_block_size, 0x7FFFFFFF);
    const wlp_params c = to_c(p);
    const std::size_t R = static_cast<std::size_t>(p.replications);
    ModelRun run;
    run.cfg = plan.cfg;
    run.mode = mode;
    const bool mm1 = model == ModelKind::Mm1;
    std::vector<double> o0(R), o1(mm1 ? R : 0), o2(mm1 ? R : 0);
    wlp_report rep{};
    char warn[512];
    if (opts.devices > 1) {  // contiguous slices over GPUs 0..devices-1 (wlp_run_devices)
        std::vector<int> devs(static_cast<std::size_t>(opts.devices));
        for (int k = 0; k < opts.devices; ++k) devs[static_cast<std::size_t>(k)] = k;
        check(wlp_run_devices(model_id(model), &c, mode_id(mode), master_seed, tlp_block_size, devs.data(),
                              opts.devices, o0.data(), mm1 ? o1.data() : nullptr, mm1 ? o2.data() : nullptr, &rep,
                              nullptr, 0.95, warn, sizeof warn));
    } else {
        check(wlp_run(model_id(model), &c, mode_id(mode), master_seed, tlp_block_size, o0.data(),
                      mm1 ? o1.data() : nullptr, mm1 ? o2.data() : nullptr, 0, nullptr, &rep, nullptr, 0.95, warn,
                      sizeof warn));
    }
    if (warn[0]) run.warning = std::string(warn);
    run.report = from_c(rep);
    if (mm1) {
        run.outputs["outIdle"] = std::move(o0);
        run.outputs["outWait"] = std::move(o1);
        run.outputs["outSys"] = std::move(o2);
        run.primary = run.outputs["outWait"];
    } else {
        run.outputs["out"] = std::move(o0);
        run.primary = run.outputs["out"];
    }
    return run;
}

}  // namespace warpsim
