// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference sources (/root/reference/proj/src/*.cpp),
// compiled in place by oracle/Makefile into oracle/_ref/libwarpsim_ref.so with the
// reference's own flags (-std=c++20 -O2 -ffp-contract=off, proj/CMakeLists.txt:3,12-13).
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
// load this library; it is the checker and the CPU baseline, never the thing measured.
//
// Every entry point wraps one public reference function and maps the reference's
// exception taxonomy (proj/include/warpsim/error.hpp:8-36) onto the status codes the
// product C-ABI uses (include/wlp_b200.h), so parity tests can compare errors too.

#include <algorithm>
#include <cstdint>
#include <map>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "warpsim/device.hpp"
#include "warpsim/error.hpp"
#include "warpsim/kernel_text.hpp"
#include "warpsim/models.hpp"
#include "warpsim/rng.hpp"
#include "warpsim/sweep.hpp"
#include "warpsim/wlp.hpp"

namespace {

thread_local std::string g_err;

// Same layout as wlp_params in include/wlp_b200.h.
struct RefParams {
    std::int64_t replications, draws, clients;
    double lambda, mu;
    std::int64_t steps, chunks;
};

warpsim::ModelParams to_params(const RefParams* p) {
    warpsim::ModelParams mp;
    mp.replications = p->replications;
    mp.draws = p->draws;
    mp.clients = p->clients;
    mp.lambda = p->lambda;
    mp.mu = p->mu;
    mp.steps = p->steps;
    mp.chunks = p->chunks;
    return mp;
}

warpsim::ModelKind to_model(int m) {
    switch (m) {
        case 0: return warpsim::ModelKind::Pi;
        case 1: return warpsim::ModelKind::Mm1;
        case 2: return warpsim::ModelKind::Walk;
    }
    throw warpsim::DomainError("unknown model id");
}

warpsim::ExecutionMode to_mode(int m) {
    switch (m) {
        case 0: return warpsim::ExecutionMode::Sequential;
        case 1: return warpsim::ExecutionMode::Tlp;
        case 2: return warpsim::ExecutionMode::Wlp;
    }
    throw warpsim::DomainError("unknown mode id");
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const warpsim::DomainError& e) {
        g_err = e.what();
        return 1;
    } catch (const warpsim::PlanError& e) {
        g_err = e.what();
        return 2;
    } catch (const warpsim::FaultError& e) {
        g_err = e.what();
        return 3;
    } catch (const warpsim::ParseError& e) {
        g_err = e.what();
        return 8;
    } catch (const warpsim::AnalysisError& e) {
        g_err = e.what();
        return 9;
    } catch (const warpsim::Error& e) {
        g_err = e.what();
        // random_spacing's exhaustion error (rng.cpp:81-82) is the only plain Error
        // on this path; report it as the spacing status.
        return std::string(e.what()).find("random_spacing") != std::string::npos ? 4 : 7;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 7;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// make_rng_state(s1,s2,s3) then n × taus_next (rng.cpp:29-51).
int ref_taus_stream(std::uint32_t s1, std::uint32_t s2, std::uint32_t s3, std::int64_t n,
                    std::uint32_t* out) {
    return guarded([&] {
        warpsim::RngState st = warpsim::make_rng_state(s1, s2, s3);
        for (std::int64_t i = 0; i < n; ++i) out[i] = warpsim::taus_next(st);
    });
}

// rng_state_from_seed (rng.cpp:36-40) → 3 words.
int ref_master_from_seed(std::uint64_t seed, std::uint32_t* s) {
    return guarded([&] {
        warpsim::RngState st = warpsim::rng_state_from_seed(seed);
        s[0] = st.s1;
        s[1] = st.s2;
        s[2] = st.s3;
    });
}

// random_spacing(rng_state_from_seed(seed), count) (rng.cpp:67-87), SoA out.
int ref_random_spacing(std::uint64_t master_seed, std::int64_t count, std::uint32_t* s1,
                       std::uint32_t* s2, std::uint32_t* s3) {
    return guarded([&] {
        warpsim::RngState master = warpsim::rng_state_from_seed(master_seed);
        auto v = warpsim::random_spacing(master, static_cast<std::size_t>(count));
        for (std::int64_t i = 0; i < count; ++i) {
            s1[i] = v[i].s1;
            s2[i] = v[i].s2;
            s3[i] = v[i].s3;
        }
    });
}

// run_model (models.cpp:329-397) in any mode; outputs in the bundle's order
// (pi: out; mm1: outIdle,outWait,outSys; walk: out).
int ref_run_model(int model, const RefParams* p, int mode, std::uint64_t seed, int tlp_block,
                  double* o0, double* o1, double* o2, char* warn, int warn_cap,
                  std::int64_t* total_cycles) {
    return guarded([&] {
        warpsim::DeviceProfile prof;
        warpsim::ModelKind mk = to_model(model);
        warpsim::ModelRun run =
            warpsim::run_model(mk, to_params(p), to_mode(mode), prof, seed, tlp_block);
        const std::size_t R = run.primary.size();
        auto put = [&](const char* name, double* dst) {
            if (!dst) return;
            const auto& v = run.outputs.at(name);
            std::memcpy(dst, v.data(), R * sizeof(double));
        };
        if (mk == warpsim::ModelKind::Mm1) {
            put("outIdle", o0);
            put("outWait", o1);
            put("outSys", o2);
        } else {
            put("out", o0);
        }
        if (warn && warn_cap > 0) {
            std::string w = run.warning.value_or("");
            std::strncpy(warn, w.c_str(), static_cast<std::size_t>(warn_cap - 1));
            warn[warn_cap - 1] = 0;
        }
        if (total_cycles) *total_cycles = run.report.totalCycles;
    });
}

// SimReport of run_model (device.hpp:62-71): [totalCycles, wavesExecuted,
// peakResidentWarps, issues, aluIssues, memReads, memWrites, divergenceEvents].
int ref_run_model_report(int model, const RefParams* p, int mode, std::uint64_t seed, int tlp_block,
                         std::int64_t* out8) {
    return guarded([&] {
        warpsim::DeviceProfile prof;
        warpsim::ModelRun run = warpsim::run_model(to_model(model), to_params(p), to_mode(mode), prof, seed,
                                                   tlp_block);
        const warpsim::SimReport& r = run.report;
        const std::int64_t v[8] = {r.totalCycles,
                                   r.wavesExecuted,
                                   r.peakResidentWarps,
                                   static_cast<std::int64_t>(r.issues),
                                   static_cast<std::int64_t>(r.aluIssues),
                                   static_cast<std::int64_t>(r.memReads),
                                   static_cast<std::int64_t>(r.memWrites),
                                   static_cast<std::int64_t>(r.divergenceEvents)};
        std::memcpy(out8, v, sizeof v);
    });
}

// The reference's host replication loop (models.cpp:345-376) over caller-given streams,
// split into contiguous slices over `nthreads` host threads. The per-replication
// functions are pure, so slicing changes nothing but wall time. This is the
// CPU baseline ("kind": "reference") timed by bench.py.
int ref_replications(int model, const RefParams* p, const std::uint32_t* s1,
                     const std::uint32_t* s2, const std::uint32_t* s3, std::int64_t count,
                     double* o0, double* o1, double* o2, int nthreads) {
    return guarded([&] {
        warpsim::ModelKind mk = to_model(model);
        warpsim::validate_params(mk, to_params(p));
        if (nthreads < 1) nthreads = 1;
        std::vector<std::thread> pool;
        std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nthreads));
        for (int t = 0; t < nthreads; ++t) {
            const std::int64_t lo = count * t / nthreads, hi = count * (t + 1) / nthreads;
            pool.emplace_back([&, t, lo, hi] {
                try {
                    for (std::int64_t r = lo; r < hi; ++r) {
                        warpsim::RngState st{s1[r], s2[r], s3[r]};
                        switch (mk) {
                            case warpsim::ModelKind::Pi:
                                o0[r] = warpsim::pi_replication(p->draws, st);
                                break;
                            case warpsim::ModelKind::Mm1: {
                                warpsim::MM1Result m =
                                    warpsim::mm1_replication(p->clients, p->lambda, p->mu, st);
                                o0[r] = m.avgIdle;
                                o1[r] = m.avgWaitQueue;
                                o2[r] = m.avgSystem;
                                break;
                            }
                            case warpsim::ModelKind::Walk:
                                o0[r] = warpsim::walk_replication(p->steps, p->chunks, st);
                                break;
                        }
                    }
                } catch (...) {
                    errs[static_cast<std::size_t>(t)] = std::current_exception();
                }
            });
        }
        for (auto& th : pool) th.join();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
    });
}

// The reference's *_replication_u templates (models.hpp:49-108) over explicit uniforms:
// replication r's source yields u[r*2n ...] in order (pins wlp_run_uniforms).
int ref_replications_u(int model, const RefParams* p, const double* u, std::int64_t count, double* o0,
                       double* o1, double* o2) {
    return guarded([&] {
        warpsim::ModelKind mk = to_model(model);
        const std::int64_t n = mk == warpsim::ModelKind::Pi ? p->draws
                               : mk == warpsim::ModelKind::Mm1 ? p->clients : p->steps;
        for (std::int64_t r = 0; r < count; ++r) {
            const double* src = u + r * 2 * n;
            std::int64_t i = 0;
            auto next = [&] { return src[i++]; };
            switch (mk) {
                case warpsim::ModelKind::Pi: o0[r] = warpsim::pi_replication_u(p->draws, next); break;
                case warpsim::ModelKind::Mm1: {
                    warpsim::MM1Result m = warpsim::mm1_replication_u(p->clients, p->lambda, p->mu, next);
                    o0[r] = m.avgIdle;
                    o1[r] = m.avgWaitQueue;
                    o2[r] = m.avgSystem;
                    break;
                }
                case warpsim::ModelKind::Walk: o0[r] = warpsim::walk_replication_u(p->steps, p->chunks, next); break;
            }
        }
    });
}

// confidence_interval (models.cpp:99-119).
int ref_confidence_interval(const double* x, std::int64_t n, double level, double* mean,
                            double* half_width, std::int64_t* n_out, int* warn_small) {
    return guarded([&] {
        std::vector<double> v(x, x + n);
        warpsim::ConfidenceInterval ci = warpsim::confidence_interval(v, level);
        *mean = ci.mean;
        *half_width = ci.halfWidth;
        *n_out = ci.n;
        *warn_small = ci.warnSmallSample ? 1 : 0;
    });
}

// inverse_normal_cdf (models.cpp:61-97).
int ref_inverse_normal_cdf(double p, double* out) {
    return guarded([&] { *out = warpsim::inverse_normal_cdf(p); });
}

// -log(1-u)/rate through the reference's exponential_from_u (rng.cpp:57-61): the glibc
// log call mm1 depends on (models.hpp:67,75 perform the same expression inline).
int ref_exponential_from_u(const double* u, std::int64_t n, double rate, double* out) {
    return guarded([&] {
        for (std::int64_t i = 0; i < n; ++i) out[i] = warpsim::exponential_from_u(u[i], rate);
    });
}

// plan_launch (wlp.cpp:71-105) geometry + warning.
int ref_plan_launch(std::int64_t replications, int mode, int tlp_block, std::int64_t* dims,
                    char* warn, int warn_cap) {
    return guarded([&] {
        warpsim::DeviceProfile prof;
        warpsim::LaunchPlan plan = warpsim::plan_launch(replications, to_mode(mode), prof, tlp_block);
        dims[0] = plan.cfg.blockDim.x;
        dims[1] = plan.cfg.gridDim.x;
        dims[2] = plan.cfg.warpSize;
        if (warn && warn_cap > 0) {
            std::string w = plan.warning.value_or("");
            std::strncpy(warn, w.c_str(), static_cast<std::size_t>(warn_cap - 1));
            warn[warn_cap - 1] = 0;
        }
    });
}

// run_sweep + csv_string (sweep.cpp:57-94, 119-129). modes: bitmask 1=seq 2=tlp 4=wlp.
int ref_sweep_csv(int model, int modes_mask, std::int64_t r_min, std::int64_t r_max,
                  std::int64_t r_step, const RefParams* p, std::uint64_t seed, int tlp_block,
                  char* buf, std::int64_t cap) {
    return guarded([&] {
        warpsim::SweepSpec spec;
        spec.model = to_model(model);
        if (modes_mask & 1) spec.modes.push_back(warpsim::ExecutionMode::Sequential);
        if (modes_mask & 2) spec.modes.push_back(warpsim::ExecutionMode::Tlp);
        if (modes_mask & 4) spec.modes.push_back(warpsim::ExecutionMode::Wlp);
        spec.rMin = r_min;
        spec.rMax = r_max;
        spec.rStep = r_step;
        spec.params = to_params(p);
        spec.masterSeed = seed;
        spec.tlpBlockSize = tlp_block;
        warpsim::DeviceProfile prof;
        std::string s = warpsim::csv_string(warpsim::run_sweep(spec, prof));
        if (static_cast<std::int64_t>(s.size()) + 1 > cap) throw warpsim::Error("csv buffer too small");
        std::memcpy(buf, s.c_str(), s.size() + 1);
    });
}


// ---- kernel IR (the checker of the GPU IR interpreter) -----------------------------------

namespace {
int put_text(const std::string& s, char* out, int cap, int* need) {
    if (need) *need = static_cast<int>(s.size()) + 1;
    if (out && cap > 0) {
        const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = 0;
    }
    return 0;
}
}  // namespace

// dump_kernel (kernel_text.cpp:344-366) of build_model_body (mode 0) or its wrap_tlp (1) /
// wrap_wlp (2) form (wlp.cpp:107-138).
int ref_ir_model_text(int model, int mode, char* out, int cap, int* need) {
    return guarded([&] {
        warpsim::KernelProgram body = warpsim::build_model_body(to_model(model));
        warpsim::KernelProgram prog = mode == 0 ? body : mode == 1 ? warpsim::wrap_tlp(body) : warpsim::wrap_wlp(body);
        put_text(warpsim::dump_kernel(prog), out, cap, need);
    });
}

// dump_kernel(parse_kernel(text)).
int ref_ir_canonical(const char* text, char* out, int cap, int* need) {
    return guarded([&] { put_text(warpsim::dump_kernel(warpsim::parse_kernel(text)), out, cap, need); });
}

// simulate (device.cpp:140-226) of a kernel text: scalars by name, arrays by name (updated
// in place), lane streams SoA[3*n_streams]; report8 as ref_run_model_report.
int ref_ir_simulate_text(const char* text, const std::int64_t* cfg6, int max_threads_per_block, int n_scalars,
                         const char* const* names, const int* is_int, const std::int64_t* ivals,
                         const double* rvals, int n_arrays, const char* const* anames, double* const* arrays,
                         const std::int64_t* alen, const std::uint32_t* streams, std::int64_t n_streams,
                         int mask_depth, std::int64_t* report8) {
    return guarded([&] {
        warpsim::KernelProgram prog = warpsim::parse_kernel(text);
        warpsim::LaunchConfig cfg;
        cfg.blockDim = {cfg6[0], cfg6[1], cfg6[2]};
        cfg.gridDim = {cfg6[3], cfg6[4]};
        cfg.warpSize = static_cast<int>(cfg6[5]);
        std::map<std::string, warpsim::Value> scalars;
        for (int k = 0; k < n_scalars; ++k)
            scalars[names[k]] = is_int[k] ? warpsim::Value::integer(ivals[k]) : warpsim::Value::real(rvals[k]);
        warpsim::GlobalMemory mem;
        for (int k = 0; k < n_arrays; ++k) mem.arrays[anames[k]].assign(arrays[k], arrays[k] + alen[k]);
        std::vector<warpsim::RngState> st(static_cast<std::size_t>(n_streams));
        for (std::int64_t t = 0; t < n_streams; ++t)
            st[t] = warpsim::RngState{streams[t], streams[n_streams + t], streams[2 * n_streams + t]};
        warpsim::DeviceProfile prof;
        prof.maxThreadsPerBlock = max_threads_per_block;
        warpsim::SimOptions opts;
        opts.maskStackDepth = mask_depth;
        const warpsim::SimReport r = warpsim::simulate(prog, cfg, prof, mem, scalars, st, opts);
        for (int k = 0; k < n_arrays; ++k) std::copy(mem.arrays[anames[k]].begin(), mem.arrays[anames[k]].end(), arrays[k]);
        const std::int64_t v[8] = {r.totalCycles, r.wavesExecuted, r.peakResidentWarps,
                                   static_cast<std::int64_t>(r.issues), static_cast<std::int64_t>(r.aluIssues),
                                   static_cast<std::int64_t>(r.memReads), static_cast<std::int64_t>(r.memWrites),
                                   static_cast<std::int64_t>(r.divergenceEvents)};
        std::memcpy(report8, v, sizeof v);
    });
}

}  // extern "C"
