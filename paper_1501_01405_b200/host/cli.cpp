// warpsim CLI on the B200 engine: `sweep`, `steps`, `ci` with the reference's flags and
// exit codes (tools/warpsim_main.cpp:175-222: 0 ok, 2 usage / DomainError, 1 Error).
// Built as paper_1501_01405_b200/warpsim; the replications run on the GPU.
//
//   warpsim sweep --model pi --modes sequential,tlp,wlp --r-min 1 --r-max 130 --draws 1000 --seed 42
//   warpsim steps pi.csv
//   warpsim ci --model mm1 --replications 30 --clients 100000 --seed 42
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <vector>

#include "warpsim_b200.hpp"
#include "warpsim_ir_b200.hpp"

using namespace warpsim;

namespace {

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Args {
    std::string cmd;
    std::vector<std::string> positional;
    std::map<std::string, std::string> opt;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    std::string str(const std::string& k, const std::string& d) const { return has(k) ? opt.at(k) : d; }
    long long integer(const std::string& k, long long d) const {
        if (!has(k)) return d;
        char* end = nullptr;
        const long long v = std::strtoll(opt.at(k).c_str(), &end, 10);
        if (!end || *end) throw Usage("--" + k + ": not an integer: " + opt.at(k));
        return v;
    }
    unsigned long long uinteger(const std::string& k, unsigned long long d) const {
        if (!has(k)) return d;
        char* end = nullptr;
        const unsigned long long v = std::strtoull(opt.at(k).c_str(), &end, 10);
        if (!end || *end) throw Usage("--" + k + ": not an integer: " + opt.at(k));
        return v;
    }
    double real(const std::string& k, double d) const {
        if (!has(k)) return d;
        char* end = nullptr;
        const double v = std::strtod(opt.at(k).c_str(), &end);
        if (!end || *end) throw Usage("--" + k + ": not a number: " + opt.at(k));
        return v;
    }
};

const char* kUsage =
    "usage: warpsim <sweep|steps|ci> [options]\n"
    "  common:  --model pi|mm1|walk --seed N --tlp-block-size N --profile FILE (ignored)\n"
    "           --draws N --clients N --lambda X --mu X --steps N --chunks N\n"
    "  sweep:   --modes sequential,tlp,wlp --r-min N --r-max N --r-step N [--out FILE] [--wallclock] [--dump-kernel]\n"
    "           [--ir-counters]  (the reference's IR kernels on the GPU interpreter: its counters)\n"
    "  steps:   CSV_FILE\n"
    "  ci:      --mode wlp --replications N --level 0.95\n";

Args parse(int argc, char** argv) {
    if (argc < 2) throw Usage("missing subcommand");
    Args a;
    a.cmd = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string s = argv[i];
        if (s.rfind("--", 0) == 0) {
            std::string key = s.substr(2), val;
            const auto eq = key.find('=');
            if (eq != std::string::npos) {
                val = key.substr(eq + 1);
                key = key.substr(0, eq);
            } else if (key == "wallclock" || key == "help" || key == "dump-kernel" || key == "ir-counters") {
                val = "1";
            } else {
                if (i + 1 >= argc) throw Usage("--" + key + " needs a value");
                val = argv[++i];
            }
            a.opt[key] = val;
        } else {
            a.positional.push_back(s);
        }
    }
    return a;
}

ModelParams model_params(const Args& a) {
    ModelParams p;
    p.draws = a.integer("draws", p.draws);
    p.clients = a.integer("clients", p.clients);
    p.lambda = a.real("lambda", p.lambda);
    p.mu = a.real("mu", p.mu);
    p.steps = a.integer("steps", p.steps);
    p.chunks = a.integer("chunks", p.chunks);
    return p;
}

std::vector<ExecutionMode> parse_modes(const std::string& csv) {
    std::vector<ExecutionMode> modes;
    std::size_t start = 0;
    while (start <= csv.size()) {
        const std::size_t comma = csv.find(',', start);
        const std::string item = csv.substr(start, comma == std::string::npos ? comma : comma - start);
        if (!item.empty()) modes.push_back(mode_from_name(item));
        if (comma == std::string::npos) break;
        start = comma + 1;
    }
    if (modes.empty()) throw DomainError("no execution modes given");
    return modes;
}

int cmd_sweep(const Args& a) {
    SweepSpec spec;
    spec.model = model_from_name(a.str("model", "pi"));
    spec.modes = parse_modes(a.str("modes", "sequential,tlp,wlp"));
    spec.rMin = a.integer("r-min", 1);
    spec.rMax = a.integer("r-max", 1);
    spec.rStep = a.integer("r-step", 1);
    spec.params = model_params(a);
    spec.masterSeed = a.uinteger("seed", 1);
    spec.tlpBlockSize = static_cast<int>(a.integer("tlp-block-size", 256));
    spec.irCounters = a.has("ir-counters");
    if (a.has("dump-kernel")) {  // the IR kernel each mode would run (warpsim_main.cpp:101-110)
        ModelParams p = spec.params;
        p.replications = spec.rMax;
        for (ExecutionMode mode : spec.modes) {
            const KernelBundle b = build_kernel(spec.model, p, mode, DeviceProfile{}, spec.tlpBlockSize);
            std::printf("; %s, %s, R=%lld\n%s\n", model_name(spec.model), mode_name(mode),
                        static_cast<long long>(spec.rMax), dump_kernel(b.program).c_str());
        }
        return 0;
    }
    const auto t0 = std::chrono::steady_clock::now();
    const std::vector<SweepRow> rows = run_sweep(spec, DeviceProfile{});
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (a.has("out")) {
        emit_csv(rows, a.str("out", ""));
        std::fprintf(stderr, "wrote %zu rows to %s\n", rows.size(), a.str("out", "").c_str());
    } else {
        std::fputs(csv_string(rows).c_str(), stdout);
    }
    if (a.has("wallclock")) std::fprintf(stderr, "host wall clock: %.3fs (GPU; cycles are measured)\n", secs);
    return 0;
}

int cmd_steps(const Args& a) {
    if (a.positional.empty()) throw Usage("steps: missing CSV file");
    const std::vector<SweepRow> rows = parse_csv(a.positional[0]);
    for (ExecutionMode mode : {ExecutionMode::Sequential, ExecutionMode::Tlp, ExecutionMode::Wlp}) {
        const auto curve = curve_of(rows, mode);
        if (curve.empty()) continue;
        const auto steps = detect_steps(curve);
        std::printf("%-10s points=%zu plateau=%lld cycles", mode_name(mode), curve.size(),
                    static_cast<long long>(curve.front().second));
        if (steps.empty()) {
            std::printf(" steps=none\n");
        } else {
            std::printf(" steps=");
            for (std::size_t i = 0; i < steps.size(); ++i)
                std::printf("%s%lld", i ? "," : "", static_cast<long long>(steps[i]));
            std::printf("\n");
        }
    }
    return 0;
}

int cmd_ci(const Args& a) {
    const ModelKind model = model_from_name(a.str("model", "pi"));
    const ExecutionMode mode = mode_from_name(a.str("mode", "wlp"));
    ModelParams p = model_params(a);
    p.replications = a.integer("replications", 30);
    const double level = a.real("level", 0.95);
    const ModelRun run = run_model(model, p, mode, DeviceProfile{}, a.uinteger("seed", 1),
                                   static_cast<int>(a.integer("tlp-block-size", 256)));
    if (run.warning) std::fprintf(stderr, "warning: %s\n", run.warning->c_str());
    auto one = [&](const char* name, const std::vector<double>& x) {
        if (x.size() < 2) {
            std::printf("%-8s n=%zu mean=%.10g (need >= 2 replications for an interval)\n", name, x.size(),
                        x.empty() ? 0.0 : x[0]);
            return;
        }
        const ConfidenceInterval ci = confidence_interval(x, level);
        std::printf("%-8s n=%lld mean=%.10g ci%.0f=[%.10g, %.10g] half=%.4g%s\n", name,
                    static_cast<long long>(ci.n), ci.mean, level * 100.0, ci.low(), ci.high(), ci.halfWidth,
                    ci.warnSmallSample ? "  (small sample: n < 30)" : "");
    };
    if (model == ModelKind::Mm1) {
        one("idle", run.outputs.at("outIdle"));
        one("wait", run.outputs.at("outWait"));
        one("system", run.outputs.at("outSys"));
    } else {
        one("estimate", run.primary);
    }
    std::printf("cycles=%lld waves=%lld kernel_ms=%.4f (measured on the GPU)\n",
                static_cast<long long>(run.report.totalCycles), static_cast<long long>(run.report.wavesExecuted),
                run.report.kernelMs);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Args a = parse(argc, argv);
        if (a.has("help")) {
            std::fputs(kUsage, stdout);
            return 0;
        }
        if (a.cmd == "sweep") return cmd_sweep(a);
        if (a.cmd == "steps") return cmd_steps(a);
        if (a.cmd == "ci") return cmd_ci(a);
        throw Usage("unknown subcommand '" + a.cmd + "'");
    } catch (const Usage& e) {
        std::fprintf(stderr, "error: %s\n%s", e.what(), kUsage);
        return 2;
    } catch (const DomainError& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const Error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
