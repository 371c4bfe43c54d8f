// The C++ drop-in (include/warpsim_b200.hpp, libwarpsim_b200.so) exercised the way the
// reference's own doctest suites exercise warpsim (test_models.cpp, test_wlp.cpp,
// test_sweep.cpp, test_rng.cpp), with the CPU oracle (oracle/liboracle.so, linked as
// test infrastructure) as the host reference.
//
//   test_dropin --cpu   host-side API only (no GPU)
//   test_dropin         everything (GPU)
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

#include "warpsim_b200.hpp"
#include "warpsim_ir_b200.hpp"

extern "C" {  // oracle/oracle.c (test infrastructure)
typedef struct {
    int64_t replications, draws, clients;
    double lambda, mu;
    int64_t steps, chunks;
} oracle_params;
int oracle_run_model(int model, const oracle_params* p, uint64_t seed, double* o0, double* o1, double* o2);
int oracle_random_spacing(uint64_t master_seed, int64_t count, uint32_t* s1, uint32_t* s2, uint32_t* s3);
int oracle_taus_stream(uint32_t a, uint32_t b, uint32_t c, int64_t n, uint32_t* out);
int oracle_master_from_seed(uint64_t seed, uint32_t s[3]);
double oracle_pi_replication(int64_t draws, const uint32_t seed[3]);
double oracle_walk_replication(int64_t steps, int64_t chunks, const uint32_t seed[3]);
void oracle_mm1_replication(int64_t clients, double lambda, double mu, const uint32_t seed[3], double out[3]);
}

using namespace warpsim;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                     \
    do {                                                                                \
        ++g_checks;                                                                     \
        if (!(cond)) {                                                                  \
            ++g_fail;                                                                   \
            std::printf("  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);               \
        }                                                                               \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                        \
    do {                                                                                \
        ++g_checks;                                                                     \
        bool ok_ = false;                                                               \
        try {                                                                           \
            (void)(expr);                                                               \
        } catch (const T&) {                                                            \
            ok_ = true;                                                                 \
        } catch (...) {                                                                 \
        }                                                                               \
        if (!ok_) {                                                                     \
            ++g_fail;                                                                   \
            std::printf("  FAIL %s:%d: %s does not throw %s\n", __FILE__, __LINE__, #expr, #T); \
        }                                                                               \
    } while (0)

static void test_case(const char* name, const std::function<void()>& body) {
    const int before = g_fail;
    try {
        body();
    } catch (const std::exception& e) {
        ++g_fail;
        std::printf("  FAIL exception: %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

static std::string root;

static std::string slurp(const std::string& path) {
    std::ifstream in(path);
    std::ostringstream s;
    s << in.rdbuf();
    return s.str();
}

static std::vector<unsigned long long> ints_after(const std::string& text, const std::string& key) {
    std::vector<unsigned long long> v;
    std::size_t i = text.find(key);
    if (i == std::string::npos) return v;
    i = text.find('[', i);
    const std::size_t end = text.find(']', i);
    std::string body = text.substr(i + 1, end - i - 1);
    std::stringstream ss(body);
    std::string tok;
    while (std::getline(ss, tok, ',')) v.push_back(std::stoull(tok));
    return v;
}

static oracle_params op(const ModelParams& p) {
    return oracle_params{p.replications, p.draws, p.clients, p.lambda, p.mu, p.steps, p.chunks};
}

static void host_tests() {
    test_case("names round trip (models.cpp:10-24, wlp.cpp:35-49)", [] {
        for (auto m : {ModelKind::Pi, ModelKind::Mm1, ModelKind::Walk}) CHECK(model_from_name(model_name(m)) == m);
        for (auto m : {ExecutionMode::Sequential, ExecutionMode::Tlp, ExecutionMode::Wlp})
            CHECK(mode_from_name(mode_name(m)) == m);
        CHECK_THROWS_AS(model_from_name("queue"), DomainError);
        CHECK_THROWS_AS(mode_from_name("simd"), DomainError);
    });
    test_case("rng state from seed and re-map (rng.cpp:29-40)", [] {
        for (std::uint64_t seed : {0ull, 42ull, 9001ull, 20260201ull}) {
            std::uint32_t s[3];
            oracle_master_from_seed(seed, s);
            CHECK((rng_state_from_seed(seed) == RngState{s[0], s[1], s[2]}));
        }
        CHECK((make_rng_state(0, 0, 0) == RngState{2, 8, 16}));
        CHECK((make_rng_state(1, 7, 15) == RngState{3, 15, 31}));
    });
    test_case("plan_launch geometry and limits (test_wlp.cpp:95-135)", [] {
        DeviceProfile prof;
        LaunchPlan w = plan_launch(10, ExecutionMode::Wlp, prof);
        CHECK(w.cfg.blockDim.x == 32 && w.cfg.gridDim.x == 10 && !w.warning);
        LaunchPlan t = plan_launch(50, ExecutionMode::Tlp, prof);
        CHECK(t.cfg.blockDim.x == 50 && t.cfg.gridDim.x == 1 && t.warning.has_value());
        LaunchPlan t2 = plan_launch(1000, ExecutionMode::Tlp, prof, 256);
        CHECK(t2.cfg.blockDim.x == 256 && t2.cfg.gridDim.x == 4);
        LaunchPlan s = plan_launch(7, ExecutionMode::Sequential, prof);
        CHECK(s.cfg.warpSize == 1 && s.cfg.blockDim.x == 1);
        CHECK_THROWS_AS(plan_launch(65536, ExecutionMode::Wlp, prof), PlanError);
        CHECK_THROWS_AS(plan_launch(0, ExecutionMode::Tlp, prof), PlanError);
        DeviceProfile small;
        small.maxThreadsPerBlock = 128;
        CHECK_THROWS_AS(plan_launch(10, ExecutionMode::Tlp, small, 256), PlanError);
    });
    test_case("validate_params (models.cpp:26-44)", [] {
        ModelParams p;
        CHECK(!validate_params(ModelKind::Pi, p));
        p.lambda = 2.0;
        CHECK(validate_params(ModelKind::Mm1, p)->find("unstable") != std::string::npos);
        p.draws = 0;
        CHECK_THROWS_AS(validate_params(ModelKind::Pi, p), DomainError);
    });
    test_case("normal quantile (test_models.cpp:152-167)", [] {
        CHECK(std::fabs(inverse_normal_cdf(0.975) - 1.9599639845400538) < 1e-14);
        CHECK_THROWS_AS(inverse_normal_cdf(0.0), DomainError);
    });
    test_case("step detection + csv round trip (test_sweep.cpp:96-218)", [] {
        CHECK((detect_steps({{1, 10}, {2, 10}, {3, 20}, {4, 20}, {5, 35}}) == std::vector<std::int64_t>{3, 5}));
        CHECK_THROWS_AS(detect_steps({{1, 10}, {2, 5}}), AnalysisError);
        CHECK_THROWS_AS(detect_steps({{2, 10}, {1, 10}}), AnalysisError);
        const std::string csv = slurp(root + "/tests/golden/sweep_pi.csv");
        auto rows = parse_csv_string(csv);
        CHECK(rows.size() == 6);
        CHECK(csv_string(rows) == csv);  // byte-stable (shortest round-trip doubles)
        CHECK_THROWS_AS(parse_csv_string("bad,header\n1,2\n"), ParseError);
        CHECK((curve_of(rows, ExecutionMode::Tlp) == std::vector<std::pair<std::int64_t, std::int64_t>>{{1, 81406}, {2, 81406}}));
    });
}

static void gpu_tests() {
    DeviceProfile prof;
    test_case("taus88.golden on the GPU (test_rng.cpp:43-57)", [] {
        const std::string g = slurp(root + "/tests/golden/taus88.json");
        auto seed = ints_after(g, "\"seed\"");
        auto want = ints_after(g, "\"outputs\"");
        RngState st = make_rng_state(seed[0], seed[1], seed[2]);
        auto got = taus_stream(st, want.size());
        bool same = got.size() == want.size();
        for (std::size_t i = 0; same && i < got.size(); ++i) same = got[i] == want[i];
        CHECK(same);
        // the state advanced exactly past the consumed draws
        std::vector<std::uint32_t> ref(101);
        oracle_taus_stream(seed[0], seed[1], seed[2], 101, ref.data());
        CHECK(taus_stream(st, 1)[0] == ref[100]);
    });
    test_case("random_spacing advances the master like the reference (rng.cpp:67-87)", [] {
        RngState master = rng_state_from_seed(42);
        auto streams = random_spacing(master, 1000);
        std::vector<std::uint32_t> a(1001), b(1001), c(1001);
        oracle_random_spacing(42, 1001, a.data(), b.data(), c.data());
        bool same = true;
        for (int i = 0; i < 1000; ++i) same = same && (streams[i] == RngState{a[i], b[i], c[i]});
        CHECK(same);
        // the next stream drawn from the advanced master is stream 1000 of one run
        auto next = random_spacing(master, 1);
        CHECK((next[0] == RngState{a[1000], b[1000], c[1000]}));
    });
    test_case("device execution is bit-identical to the host references (test_models.cpp:276-326)", [&] {
        const std::uint64_t seed = 20260201;
        ModelParams p;
        p.replications = 8;
        p.draws = 100;
        ModelRun run = run_model(ModelKind::Pi, p, ExecutionMode::Wlp, prof, seed);
        RngState master = rng_state_from_seed(seed);
        auto streams = random_spacing(master, 8);
        for (int r = 0; r < 8; ++r) {
            const std::uint32_t s[3] = {streams[r].s1, streams[r].s2, streams[r].s3};
            CHECK(run.primary[r] == oracle_pi_replication(100, s));
            CHECK(run.primary[r] == pi_replication(100, streams[r]));
        }
        p.replications = 7;
        p.clients = 90;
        ModelRun mm = run_model(ModelKind::Mm1, p, ExecutionMode::Tlp, prof, seed);
        for (int r = 0; r < 7; ++r) {
            const std::uint32_t s[3] = {streams[r].s1, streams[r].s2, streams[r].s3};
            double h[3];
            oracle_mm1_replication(90, p.lambda, p.mu, s, h);
            CHECK(mm.outputs.at("outIdle")[r] == h[0]);
            CHECK(mm.outputs.at("outWait")[r] == h[1]);
            CHECK(mm.outputs.at("outSys")[r] == h[2]);
            const MM1Result d = mm1_replication(90, p.lambda, p.mu, streams[r]);
            CHECK(d.avgWaitQueue == h[1]);
        }
        p.steps = 64;
        p.chunks = 5;
        for (auto mode : {ExecutionMode::Wlp, ExecutionMode::Tlp}) {
            ModelRun wk = run_model(ModelKind::Walk, p, mode, prof, seed);
            for (int r = 0; r < 7; ++r) {
                const std::uint32_t s[3] = {streams[r].s1, streams[r].s2, streams[r].s3};
                CHECK(wk.primary[r] == oracle_walk_replication(64, 5, s));
                CHECK(wk.primary[r] == walk_replication(64, 5, streams[r]));
            }
        }
    });
    test_case("outputs bit-identical across execution modes (acceptance criterion 9)", [&] {
        for (ModelKind model : {ModelKind::Pi, ModelKind::Mm1, ModelKind::Walk}) {
            for (std::int64_t R : {1, 7, 33}) {
                ModelParams p;
                p.replications = R;
                p.draws = 200;
                p.clients = 150;
                p.steps = 120;
                p.chunks = 7;
                std::vector<double> h0(R), h1(R), h2(R);
                const oracle_params o = op(p);
                oracle_run_model(static_cast<int>(model), &o, 9001, h0.data(), h1.data(), h2.data());
                for (auto mode : {ExecutionMode::Sequential, ExecutionMode::Tlp, ExecutionMode::Wlp}) {
                    ModelRun run = run_model(model, p, mode, prof, 9001);
                    if (model == ModelKind::Mm1) {
                        CHECK(run.outputs.at("outIdle") == h0);
                        CHECK(run.outputs.at("outWait") == h1);
                        CHECK(run.outputs.at("outSys") == h2);
                    } else {
                        CHECK(run.primary == h0);
                    }
                }
            }
        }
    });
    test_case("run_model surfaces warnings (test_models.cpp:350-366)", [&] {
        ModelParams p;
        p.replications = 50;
        p.clients = 20;
        p.lambda = 1.0;
        p.mu = 0.5;
        ModelRun run = run_model(ModelKind::Mm1, p, ExecutionMode::Tlp, prof, 1);
        CHECK(run.warning.has_value());
        CHECK(run.warning->find("unstable") != std::string::npos);
        CHECK(run.warning->find("warp") != std::string::npos);
        p.lambda = 0.5;
        p.mu = 1.0;
        p.replications = 64;
        CHECK(!run_model(ModelKind::Mm1, p, ExecutionMode::Tlp, prof, 1).warning.has_value());
        CHECK(run.report.totalCycles > 0 && run.report.kernelMs > 0.0);
    });
    test_case("confidence intervals (test_models.cpp:169-198)", [] {
        ConfidenceInterval ci = confidence_interval({1.0, 2.0, 3.0, 4.0, 5.0});
        CHECK(ci.mean == 3.0);
        CHECK(std::fabs(ci.halfWidth - 1.3859038243496777) < 1e-14 * 1.386);
        CHECK(ci.n == 5 && ci.warnSmallSample);
        CHECK(confidence_interval({2.5, 2.5, 2.5, 2.5}).halfWidth == 0.0);
        CHECK_THROWS_AS(confidence_interval({1.0}), DomainError);
        CHECK_THROWS_AS(confidence_interval({1.0, 2.0}, 1.0), DomainError);
        std::vector<double> thirty(30);
        for (int i = 0; i < 30; ++i) thirty[i] = i % 2;
        CHECK(!confidence_interval(thirty).warnSmallSample);
    });
    test_case("sweep_pi.golden mean / CI columns (test_sweep.cpp:40-47)", [&] {
        SweepSpec spec;
        spec.model = ModelKind::Pi;
        spec.modes = {ExecutionMode::Sequential, ExecutionMode::Tlp, ExecutionMode::Wlp};
        spec.rMin = 1;
        spec.rMax = 2;
        spec.params.draws = 100;
        spec.masterSeed = 42;
        auto rows = run_sweep(spec, prof);
        auto want = parse_csv_string(slurp(root + "/tests/golden/sweep_pi.csv"));
        CHECK(rows.size() == want.size());
        for (std::size_t i = 0; i < rows.size() && i < want.size(); ++i) {
            CHECK(rows[i].replications == want[i].replications && rows[i].mode == want[i].mode);
            CHECK(rows[i].mean == want[i].mean && rows[i].ciLow == want[i].ciLow && rows[i].ciHigh == want[i].ciHigh);
            CHECK(rows[i].totalCycles > 0);
        }
        CHECK_THROWS_AS(run_sweep(SweepSpec{}, prof), DomainError);  // no modes
    });
    test_case("SimReport hardware counters via SimOptions (TLP walk diverges, WLP does not)", [&] {
        ModelParams p;
        p.replications = 64;
        p.steps = 100;
        SimOptions opts;
        opts.hardwareCounters = true;
        ModelRun tlp = run_model(ModelKind::Walk, p, ExecutionMode::Tlp, prof, 42, 256, opts);
        ModelRun wlp = run_model(ModelKind::Walk, p, ExecutionMode::Wlp, prof, 42, 256, opts);
        CHECK(tlp.report.divergenceEvents > 0 && tlp.report.memReads == 6 && tlp.report.memWrites == 2);
        CHECK(wlp.report.divergenceEvents == 0 && wlp.report.memReads > 0);
        CHECK(run_model(ModelKind::Walk, p, ExecutionMode::Tlp, prof, 42).report.divergenceEvents == 0);  // off
    });
    test_case("errors map onto the reference's exception types", [&] {
        ModelParams p;
        p.draws = 0;
        CHECK_THROWS_AS(run_model(ModelKind::Pi, p, ExecutionMode::Wlp, prof, 1), DomainError);
        p.draws = 10;
        CHECK_THROWS_AS(run_model(ModelKind::Pi, p, ExecutionMode::Tlp, prof, 1, 4096), PlanError);
    });
}

static void ir_host_tests() {
    test_case("IR values: promotion, truncation, comparisons, faults (kernel_ir.cpp:46-107)", [&] {
        CHECK(apply_bin(BinOp::Div, Value::integer(-7), Value::integer(2), "t").bit_equal(Value::integer(-3)));
        CHECK(apply_bin(BinOp::Mod, Value::integer(-7), Value::integer(2), "t").bit_equal(Value::integer(-1)));
        CHECK(apply_bin(BinOp::Add, Value::integer(1), Value::real(0.5), "t").bit_equal(Value::real(1.5)));
        const Value nan = Value::real(std::nan(""));
        CHECK(apply_bin(BinOp::Le, nan, Value::real(1.0), "t").bit_equal(Value::integer(1)));
        CHECK(apply_bin(BinOp::Lt, nan, Value::real(1.0), "t").bit_equal(Value::integer(0)));
        CHECK(apply_un(UnOp::Floor, Value::real(-2.5), "t").bit_equal(Value::integer(-3)));
        CHECK(!Value::real(0.0).bit_equal(Value::real(-0.0)) && nan.bit_equal(nan));
        CHECK_THROWS_AS(apply_bin(BinOp::Div, Value::integer(1), Value::integer(0), "t"), FaultError);
        CHECK_THROWS_AS(apply_un(UnOp::Log, Value::real(0.0), "t"), FaultError);
    });
    test_case("IR builder validation and kernel text round trip (kernel_text.hpp)", [&] {
        KernelProgram p;
        p.add_param("n", ParamKind::Int);
        p.add_param("out", ParamKind::Array);
        p.add_local("x", ValueType::Int);
        CHECK_THROWS_AS(p.add_local("n", ValueType::Real), DomainError);
        CHECK_THROWS_AS(p.param("out"), DomainError);
        CHECK_THROWS_AS(p.load("x", "out", p.ci(0)), DomainError);  // load target must be real
        p.body.push_back(p.assign("x", p.sreg(Sreg::TidX)));
        p.body.push_back(KernelProgram::if_(p.bin(BinOp::Lt, p.local("x"), p.param("n")),
                                            {p.store("out", p.local("x"), p.bin(BinOp::Mul, p.local("x"), p.cr(0.5)))}));
        p.finalize();
        const std::string text = dump_kernel(p);
        CHECK(dump_kernel(parse_kernel(text)) == text);
        CHECK_THROWS_AS(parse_kernel("(kernel (body (frob)))"), ParseError);
        for (auto m : {ModelKind::Pi, ModelKind::Mm1, ModelKind::Walk}) {
            const KernelProgram body = build_model_body(m);
            CHECK(dump_kernel(parse_kernel(dump_kernel(wrap_wlp(body)))) == dump_kernel(wrap_wlp(body)));
            CHECK_THROWS_AS(wrap_tlp(wrap_tlp(body)), DomainError);  // double wrap
        }
        const std::string names[] = {"pi", "mm1", "walk"};
        for (int m = 0; m < 3; ++m)  // the reference's own dumps (tests/golden/ir)
            CHECK(dump_kernel(wrap_tlp(build_model_body(static_cast<ModelKind>(m)))) ==
                  slurp(root + "/tests/golden/ir/" + names[m] + "_tlp.sexp"));
    });
}

static void ir_gpu_tests() {
    DeviceProfile prof;
    test_case("IR on the GPU: divergent branch, then before else, halts (test_kernel_ir.cpp:225-278)", [&] {
        KernelProgram p;
        p.add_param("out", ParamKind::Array);
        p.add_local("x", ValueType::Int);
        p.body.push_back(p.assign("x", p.sreg(Sreg::TidX)));
        std::vector<Statement> inner{p.assign("x", p.bin(BinOp::Mul, p.local("x"), p.ci(2)))};
        std::vector<Statement> then_body{p.assign("x", p.bin(BinOp::Add, p.local("x"), p.ci(10))),
                                         KernelProgram::if_(p.bin(BinOp::Lt, p.local("x"), p.ci(12)), inner),
                                         p.assign("x", p.bin(BinOp::Add, p.local("x"), p.ci(1)))};
        p.body.push_back(KernelProgram::if_(p.bin(BinOp::Lt, p.local("x"), p.ci(4)), then_body, {KernelProgram::halt()}));
        p.body.push_back(p.assign("x", p.bin(BinOp::Add, p.local("x"), p.ci(100))));
        p.body.push_back(p.store("out", p.sreg(Sreg::TidX), p.local("x")));
        p.finalize();
        LaunchConfig cfg;
        cfg.blockDim = {8, 1, 1};
        cfg.warpSize = 8;
        GlobalMemory mem;
        mem.arrays["out"] = std::vector<double>(8, -1.0);
        const SimReport rep = simulate(p, cfg, prof, mem, {}, {});
        const double want[8] = {121, 123, 113, 114, -1, -1, -1, -1};
        for (int l = 0; l < 8; ++l) CHECK(mem.arrays["out"][l] == want[l]);
        CHECK(rep.issues == 9 && rep.divergenceEvents == 1 && rep.memWrites == 1 && rep.aluIssues == 8);
    });
    test_case("IR on the GPU: run_model via SimOptions::irInterpreter equals the engine", [&] {
        ModelParams p;
        p.replications = 40;
        p.clients = 50;
        p.steps = 50;
        p.draws = 50;
        SimOptions opts;
        opts.irInterpreter = true;
        for (auto m : {ModelKind::Pi, ModelKind::Mm1, ModelKind::Walk})
            for (auto mode : {ExecutionMode::Tlp, ExecutionMode::Wlp}) {
                const ModelRun a = run_model(m, p, mode, prof, 7, 256, opts);
                const ModelRun b = run_model(m, p, ExecutionMode::Sequential, prof, 7);
                CHECK(a.outputs == b.outputs);
                CHECK(a.report.issues > 0 && a.report.memWrites > 0);
            }
        const ModelRun seq = run_model_ir(ModelKind::Pi, p, ExecutionMode::Sequential, prof, 7);
        CHECK(seq.outputs == run_model(ModelKind::Pi, p, ExecutionMode::Sequential, prof, 7).outputs);
        CHECK(seq.report.issues > 0 && seq.report.totalCycles == static_cast<std::int64_t>(seq.report.issues));
    });
    test_case("IR on the GPU: faults are FaultError", [&] {
        GlobalMemory mem;
        mem.arrays["o"] = std::vector<double>(4, 0.0);
        LaunchConfig cfg;
        cfg.blockDim = {32, 1, 1};
        CHECK_THROWS_AS(simulate(parse_kernel("(kernel (param o array) (body (store o tid.x 1.0)))"), cfg, prof, mem, {}, {}),
                        FaultError);
        CHECK_THROWS_AS(simulate(parse_kernel("(kernel (local a int) (body (assign a (div 1 (sub tid.x 5)))))"), cfg, prof,
                                 mem, {}, {}),
                        FaultError);
    });
}

int main(int argc, char** argv) {
    root = argc > 2 ? argv[2] : ".";
    const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
    host_tests();
    ir_host_tests();
    if (!cpu_only) {
        gpu_tests();
        ir_gpu_tests();
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
