// warpsim_ir_b200.hpp — the reference's kernel IR and its text form, executed on the
// B200 ("a GPU-hosted interpreter for the kernel IR").
//
// Drop-in for proj/include/warpsim/{value,kernel_ir,kernel_text}.hpp and the IR half of
// wlp.hpp / device.hpp / models.hpp: the same types, builder methods, validation,
// s-expression dump/parse, WLP/TLP wrappers and model bodies. What changes is where a
// kernel runs: `simulate` executes it on the GPU (libwlp_b200.so, wlp_ir_simulate), one IR
// warp per hardware warp, with the reference simulator's mask-stack semantics — so memory
// contents and the SimReport counters issues / aluIssues / memReads / memWrites /
// divergenceEvents are the reference's exactly (tests/test_ir_gpu.py). totalCycles,
// wavesExecuted and peakResidentWarps are measured on the hardware instead of the Fermi
// cost model (DeviceProfile is accepted; only maxThreadsPerBlock is used).
//
// User-defined models therefore run on the B200 without recompiling: write the kernel
// in the text form, parse_kernel, simulate.
//
// Not provided: the host simulator itself (WarpState / run_warp, warp_exec.hpp;
// simulate_single_thread stands in for run_single_thread) and the Fermi dispatch model (plan_dispatch, load_profile,
// report_mem_ratio) — the hardware replaces them. warpSize must be <= 32 (one hardware
// warp per IR warp); the reference accepts up to 64.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "warpsim_b200.hpp"

namespace warpsim {

// ---- value.hpp --------------------------------------------------------------------
enum class ValueType { Int, Real };

struct Value {
    ValueType type = ValueType::Int;
    std::int64_t i = 0;
    double r = 0.0;

    static Value integer(std::int64_t v) { return Value{ValueType::Int, v, 0.0}; }
    static Value real(double v) { return Value{ValueType::Real, 0, v}; }
    bool is_int() const { return type == ValueType::Int; }
    double as_real() const { return is_int() ? static_cast<double>(i) : r; }
    bool truthy() const { return is_int() ? i != 0 : r != 0.0; }
    bool bit_equal(const Value& o) const;  // representation equality (-0.0 != 0.0, NaN == NaN)
    std::string str() const;
};

enum class BinOp { Add, Sub, Mul, Div, Mod, Lt, Le, Gt, Ge, Eq, Ne, And, Or };
enum class UnOp { Neg, Log, Floor };

// Host evaluation with the reference's promotion rules and faults (FaultError).
Value apply_bin(BinOp op, const Value& a, const Value& b, const char* where);
Value apply_un(UnOp op, const Value& a, const char* where);
const char* bin_op_name(BinOp op);
const char* un_op_name(UnOp op);

// ---- kernel_ir.hpp: launch geometry -------------------------------------------------
struct ThreadCoord {
    std::int64_t x = 0, y = 0, z = 0;
};
struct BlockCoord {
    std::int64_t x = 0, y = 0;
};
inline std::int64_t warps_per_block(const LaunchConfig& cfg) {
    return (cfg.threads_per_block() + cfg.warpSize - 1) / cfg.warpSize;
}
void validate_launch(const LaunchConfig& cfg);
std::optional<std::string> launch_warning(const LaunchConfig& cfg);
std::int64_t linear_thread_id(const ThreadCoord& t, const BlockCoord& b, const LaunchConfig& cfg);
std::int64_t intra_block_thread_id(const ThreadCoord& t, const LaunchConfig& cfg);

// ---- kernel_ir.hpp: programs --------------------------------------------------------
enum class Sreg { TidX, TidY, TidZ, BidX, BidY, BDimX, BDimY, BDimZ, GDimX, GDimY, WarpSize };
enum class ParamKind { Int, Real, Array };

struct ParamDecl {
    std::string name;
    ParamKind kind;
};
struct LocalDecl {
    std::string name;
    ValueType type;
};

using ExprId = std::int32_t;

struct Expr {
    enum class Kind { Const, Local, Param, Special, Draw, Bin, Un };
    Kind kind = Kind::Const;
    Value konst;
    int slot = -1;
    Sreg sreg{};
    BinOp bop{};
    UnOp uop{};
    ExprId a = -1, b = -1;
};

enum class StmtKind { Assign, Load, Store, If, While, Halt };

struct Statement {
    StmtKind kind;
    int slot = -1;       // Assign / Load target local; Store array param
    ExprId expr_a = -1;  // Assign value, Load / Store index, If / While condition
    ExprId expr_b = -1;  // Store value; Load: the array param slot
    std::vector<Statement> body1;
    std::vector<Statement> body2;
};

struct KernelProgram {
    std::vector<ParamDecl> params;
    std::vector<LocalDecl> locals;
    std::vector<Expr> exprs;
    std::vector<Statement> body;

    int add_param(const std::string& name, ParamKind kind);
    int add_local(const std::string& name, ValueType type);
    int param_slot(const std::string& name) const;
    int local_slot(const std::string& name) const;

    ExprId ci(std::int64_t v);
    ExprId cr(double v);
    ExprId local(const std::string& name);
    ExprId param(const std::string& name);
    ExprId sreg(Sreg r);
    ExprId draw();
    ExprId bin(BinOp op, ExprId a, ExprId b);
    ExprId un(UnOp op, ExprId a);

    Statement assign(const std::string& local, ExprId value) const;
    Statement load(const std::string& local, const std::string& array, ExprId index) const;
    Statement store(const std::string& array, ExprId index, ExprId value) const;
    static Statement if_(ExprId cond, std::vector<Statement> then_body, std::vector<Statement> else_body = {});
    static Statement while_(ExprId cond, std::vector<Statement> loop_body);
    static Statement halt();

    void finalize() const;  // structural validation, DomainError
};

struct GlobalMemory {
    std::map<std::string, std::vector<double>> arrays;
};
struct ParamEnv {
    std::vector<Value> scalars;
    std::vector<std::vector<double>*> arrays;
};
ParamEnv bind_params(const KernelProgram& prog, const std::map<std::string, Value>& scalars, GlobalMemory& memory);

// ---- kernel_text.hpp ----------------------------------------------------------------
std::string dump_kernel(const KernelProgram& prog);
KernelProgram parse_kernel(const std::string& text);  // ParseError with a line reference

// ---- wlp.hpp (IR half) --------------------------------------------------------------
std::int64_t warp_index(const ThreadCoord& t, const BlockCoord& b, const LaunchConfig& cfg);
bool is_warp_leader(const ThreadCoord& t, const LaunchConfig& cfg);
KernelProgram wrap_wlp(const KernelProgram& body);
KernelProgram wrap_tlp(const KernelProgram& body);
std::vector<RngState> assign_lane_streams(ExecutionMode mode, const LaunchConfig& cfg,
                                          const std::vector<RngState>& replication_streams);

// ---- models.hpp (IR half) -----------------------------------------------------------
KernelProgram build_model_body(ModelKind model);

struct KernelBundle {
    KernelProgram program;
    LaunchConfig cfg;
    std::map<std::string, Value> scalars;
    std::vector<std::pair<std::string, std::int64_t>> arrays;
    std::vector<std::string> outputs;
    std::string primary;
    std::optional<std::string> warning;
};
KernelBundle build_kernel(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                          int tlp_block_size = 256);

// ---- device.hpp: simulate, on the B200 ------------------------------------------------
// Runs every warp of the launch on the GPU interpreter. Lane streams by global linear
// thread id (default state past the end of `streams`). SimOptions::maskStackDepth bounds
// nesting as in the reference; SimOptions::maxIssuesPerWarp guards against kernels that
// never terminate (FaultError when exceeded).
SimReport simulate(const KernelProgram& prog, const LaunchConfig& cfg, const DeviceProfile& prof,
                   GlobalMemory& memory, const std::map<std::string, Value>& scalars,
                   const std::vector<RngState>& streams, const SimOptions& opts = {});

// run_single_thread (warp_exec.hpp:95-98) on the GPU interpreter: one thread, warpSize 1,
// the given stream and initial locals; the report holds that run's counters.
SimReport simulate_single_thread(const KernelProgram& prog, GlobalMemory& memory,
                                 const std::map<std::string, Value>& scalars, RngState stream,
                                 const std::map<std::string, Value>& initial_locals = {},
                                 const SimOptions& opts = {});

// run_model through the IR path of the reference (build_kernel -> random_spacing ->
// assign_lane_streams -> simulate), on the GPU interpreter. Same outputs as run_model
// (bit-identical to Sequential) and the reference simulator's counters; for Sequential,
// the reference's unit-cost report (one body execution times R, models.cpp:377-389).
// run_model itself does this when SimOptions::irInterpreter is set.
ModelRun run_model_ir(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                      std::uint64_t master_seed, int tlp_block_size = 256, const SimOptions& opts = {});

}  // namespace warpsim
