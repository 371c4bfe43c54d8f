// warpsim_b200.hpp — C++ drop-in for the reference's replication-runner API
// (namespace warpsim: proj/include/warpsim/{models,rng,wlp,sweep,error}.hpp), backed by
// the sm_100a kernels of libwlp_b200.so through its C ABI (wlp_b200.h).
//
// A caller of the reference's run_model / run_sweep / confidence_interval switches by
// including this header instead and linking libwarpsim_b200.so (which links
// libwlp_b200.so). Names, argument meaning, defaults and exception types are the
// reference's; what changes is where the replications run:
//   * Tlp / Wlp execute on the GPU (thread / warp per replication) instead of the
//     Fermi SIMT simulator; Sequential also runs on the GPU (warp per replication, the
//     engine has no host execution path) — outputs are bit-identical in every mode.
//   * SimReport carries measured GPU time (totalCycles at the device clock, waves); the
//     simulator-only counters (issues, memReads, ...) are 0 (ncu measures those).
//   * DeviceProfile / SimOptions are accepted and ignored except
//     DeviceProfile::maxThreadsPerBlock, which plan_launch still checks.
//   * run_model lifts plan_launch's 65535-block grid cap to the hardware's 2^31-1
//     (BASELINE configs need 10^6-10^7 WLP replications); plan_launch itself keeps the
//     reference default.
// The kernel IR and its text form run on the GPU through include/warpsim_ir_b200.hpp
// (an IR interpreter on the B200 in place of the reference's host simulator).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace warpsim {

// ---- error.hpp:8-36 ---------------------------------------------------------------
struct Error : std::runtime_error {
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
struct DomainError : Error {
    using Error::Error;
};
struct PlanError : Error {
    using Error::Error;
};
struct FaultError : Error {
    using Error::Error;
};
struct ParseError : Error {
    using Error::Error;
};
struct AnalysisError : Error {
    using Error::Error;
};

// ---- rng.hpp:11-45 (all of it) ----------------------------------------------------------------
struct RngState {
    std::uint32_t s1 = 2;
    std::uint32_t s2 = 8;
    std::uint32_t s3 = 16;
    bool operator==(const RngState&) const = default;
};

RngState make_rng_state(std::uint32_t s1, std::uint32_t s2, std::uint32_t s3);
RngState rng_state_from_seed(std::uint64_t seed);
// random_spacing(master, count): streams seeded on the GPU by jump-ahead; `master` is
// advanced past every draw consumed (3 per candidate), as in the reference.
std::vector<RngState> random_spacing(RngState& master, std::size_t count);
// Raw stream: n consecutive taus_next outputs from `state` (GPU), and the state after them.
std::vector<std::uint32_t> taus_stream(RngState& state, std::size_t n);

// Scalar draws (rng.hpp:22-33). These are host utilities (one value per call, the
// reference's own arithmetic: taus88 step, * 2^-32, and -log(1-u)/rate through the same
// glibc-log port the mm1 kernels run); bulk draws go through taus_stream / the kernels.
std::uint32_t taus_next(RngState& state);
double uniform01(RngState& state);
double exponential_from_u(double u, double rate);  // DomainError: rate <= 0, u outside [0,1)
double exponential(RngState& state, double rate);

// Callable uniform source over an owned state (rng.hpp:42-45).
struct TausStream {
    RngState state;
    double operator()() { return uniform01(state); }
};

// ---- kernel_ir.hpp / device.hpp records used by the API ------------------------------
struct Dim3 {
    std::int64_t x = 1, y = 1, z = 1;
    bool operator==(const Dim3&) const = default;
};
struct Dim2 {
    std::int64_t x = 1, y = 1;
    bool operator==(const Dim2&) const = default;
};
struct LaunchConfig {
    Dim3 blockDim;
    Dim2 gridDim;
    int warpSize = 32;
    std::int64_t threads_per_block() const { return blockDim.x * blockDim.y * blockDim.z; }
    std::int64_t total_blocks() const { return gridDim.x * gridDim.y; }
};
struct DeviceProfile {
    int numSMs = 14;
    int warpSchedulersPerSM = 2;
    int maxResidentBlocksPerSM = 8;
    int maxResidentWarpsPerSM = 48;
    int deviceResidentBlockCap = 64;
    std::int64_t aluIssueCycles = 1;
    std::int64_t memLatencyCycles = 400;
    int maxThreadsPerBlock = 1024;
};
struct SimOptions {
    std::optional<std::uint64_t> smPermutationSeed;  // accepted, ignored (real hardware)
    int maskStackDepth = 32;  // IR interpreter: mask-stack bound, as in the reference
    // B200 extension: fill SimReport::divergenceEvents / memReads / memWrites from
    // instrumented kernels (wlp_set_hw_counters). Off by default: costs some speed.
    bool hardwareCounters = false;
    // B200 extension: run Tlp / Wlp through the reference's IR kernels on the GPU IR
    // interpreter (warpsim_ir_b200.hpp) instead of the hand-written kernels: same
    // outputs, and the reference simulator's exact issue / divergence / memory counters.
    bool irInterpreter = false;
    // IR interpreter: statements one IR warp may issue before FaultError (guards
    // against kernels that never terminate); under irJit, loop iterations per IR thread.
    std::int64_t maxIssuesPerWarp = std::int64_t{1} << 50;
    // B200 extension: simulate() compiles the IR kernel (CUDA C++ via NVRTC) instead of
    // interpreting it. Same memory results; the report has measured time only.
    bool irJit = false;
    // B200 extension: run_model shards the replications over GPUs 0..devices-1 of this
    // process (wlp_run_devices: contiguous slices, one host thread per GPU, global
    // spacing check, statistics merged in device order). Outputs are identical.
    int devices = 1;
};
// CUDA devices visible to this process.
int device_count();
struct SimReport {
    std::int64_t totalCycles = 0;
    std::int64_t wavesExecuted = 0;
    std::int64_t peakResidentWarps = 0;
    std::uint64_t issues = 0;
    std::uint64_t aluIssues = 0;
    std::uint64_t memReads = 0;
    std::uint64_t memWrites = 0;
    std::uint64_t divergenceEvents = 0;
    double kernelMs = 0.0;  // measured model-kernel time (B200 extension)
    std::uint64_t warpSplits = 0;  // instrumented runs: all warp splits of the kernel (B200 extension)
};

// ---- wlp.hpp:16-59 ----------------------------------------------------------------
enum class ExecutionMode { Sequential, Tlp, Wlp };
const char* mode_name(ExecutionMode mode);
ExecutionMode mode_from_name(const std::string& name);

struct LaunchPlan {
    LaunchConfig cfg;
    std::int64_t replications = 0;
    ExecutionMode mode = ExecutionMode::Sequential;
    std::optional<std::string> warning;
};
LaunchPlan plan_launch(std::int64_t replications, ExecutionMode mode, const DeviceProfile& prof,
                       int tlp_block_size = 256, std::int64_t grid_limit = 65535);

// ---- models.hpp:18-175 ------------------------------------------------------------
enum class ModelKind { Pi, Mm1, Walk };
const char* model_name(ModelKind model);
ModelKind model_from_name(const std::string& name);

struct ModelParams {
    std::int64_t replications = 1;
    std::int64_t draws = 1000;
    std::int64_t clients = 1000;
    double lambda = 0.5;
    double mu = 1.0;
    std::int64_t steps = 1000;
    std::int64_t chunks = 30;
};
std::optional<std::string> validate_params(ModelKind model, const ModelParams& p);

struct MM1Result {
    double avgIdle = 0.0;
    double avgWaitQueue = 0.0;
    double avgSystem = 0.0;
};

namespace detail {
// The model body over 2 * units uniforms on the GPU (wlp_run_uniforms); checks the
// template's parameters first (check_u), as the reference throws before drawing.
void check_u(ModelKind model, std::int64_t units, std::int64_t chunks, double lambda, double mu);
std::vector<double> run_u(ModelKind model, std::int64_t units, std::int64_t chunks, double lambda, double mu,
                          const std::vector<double>& u);
template <class U>
std::vector<double> draw_u(std::int64_t units, U& next) {
    std::vector<double> u(static_cast<std::size_t>(2 * units));
    for (double& x : u) x = next();
    return u;
}
}  // namespace detail

// One replication over any uniform source (models.hpp:49-108): the source is called
// 2 * units times in the reference's order on the host, the model body runs on the GPU
// over those values (same operations, so the same result as the reference's template).
template <class U>
double pi_replication_u(std::int64_t draws, U&& next) {
    detail::check_u(ModelKind::Pi, draws, 0, 0.0, 0.0);
    return detail::run_u(ModelKind::Pi, draws, 0, 0.0, 0.0, detail::draw_u(draws, next))[0];
}

template <class U>
MM1Result mm1_replication_u(std::int64_t clients, double lambda, double mu, U&& next) {
    detail::check_u(ModelKind::Mm1, clients, 0, lambda, mu);
    const auto o = detail::run_u(ModelKind::Mm1, clients, 0, lambda, mu, detail::draw_u(clients, next));
    return MM1Result{o[0], o[1], o[2]};
}

template <class U>
double walk_replication_u(std::int64_t steps, std::int64_t chunks, U&& next) {
    detail::check_u(ModelKind::Walk, steps, chunks, 0.0, 0.0);
    return detail::run_u(ModelKind::Walk, steps, chunks, 0.0, 0.0, detail::draw_u(steps, next))[0];
}

// One replication over a given stream, computed on the GPU (models.hpp:110-112).
double pi_replication(std::int64_t draws, RngState stream);
MM1Result mm1_replication(std::int64_t clients, double lambda, double mu, RngState stream);
double walk_replication(std::int64_t steps, std::int64_t chunks, RngState stream);

struct ConfidenceInterval {
    double mean = 0.0;
    double halfWidth = 0.0;
    double level = 0.95;
    std::int64_t n = 0;
    bool warnSmallSample = false;
    double low() const { return mean - halfWidth; }
    double high() const { return mean + halfWidth; }
};
// Device two-pass reduction; bit-identical to the reference's loop for n <= 256.
ConfidenceInterval confidence_interval(const std::vector<double>& samples, double level = 0.95);
double inverse_normal_cdf(double p);

struct ModelRun {
    std::map<std::string, std::vector<double>> outputs;
    std::vector<double> primary;
    SimReport report;
    LaunchConfig cfg;
    ExecutionMode mode = ExecutionMode::Sequential;
    std::optional<std::string> warning;
};
ModelRun run_model(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                   std::uint64_t master_seed, int tlp_block_size = 256, const SimOptions& opts = {});

// ---- sweep.hpp:14-60 --------------------------------------------------------------
struct SweepSpec {
    ModelKind model = ModelKind::Pi;
    std::vector<ExecutionMode> modes;
    std::int64_t rMin = 1;
    std::int64_t rMax = 1;
    std::int64_t rStep = 1;
    ModelParams params;
    std::uint64_t masterSeed = 1;
    int tlpBlockSize = 256;
    // B200 extension: run every point through the reference's IR kernels on the GPU
    // interpreter (SimOptions::irInterpreter), so the mem_reads / mem_writes /
    // divergence_events columns are the reference simulator's and the sequential rows are
    // its unit-cost accounting; total_cycles of the tlp / wlp rows stay measured.
    bool irCounters = false;
};
struct SweepRow {
    std::int64_t replications = 0;
    ExecutionMode mode = ExecutionMode::Sequential;
    ModelKind model = ModelKind::Pi;
    std::int64_t totalCycles = 0;
    std::uint64_t memReads = 0;
    std::uint64_t memWrites = 0;
    std::uint64_t divergenceEvents = 0;
    std::int64_t waves = 0;
    double mean = 0.0;
    double ciLow = 0.0;
    double ciHigh = 0.0;
};
std::vector<SweepRow> run_sweep(const SweepSpec& spec, const DeviceProfile& prof);
std::vector<std::int64_t> detect_steps(const std::vector<std::pair<std::int64_t, std::int64_t>>& curve);
std::vector<std::pair<std::int64_t, std::int64_t>> curve_of(const std::vector<SweepRow>& rows, ExecutionMode mode);
std::string csv_string(const std::vector<SweepRow>& rows);
void emit_csv(const std::vector<SweepRow>& rows, const std::string& path);
std::vector<SweepRow> parse_csv_string(const std::string& text);
std::vector<SweepRow> parse_csv(const std::string& path);

}  // namespace warpsim
