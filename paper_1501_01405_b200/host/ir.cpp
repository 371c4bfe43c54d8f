// Kernel IR front end for the B200 interpreter (include/warpsim_ir_b200.hpp): the
// reference's IR types and builder (kernel_ir.hpp:67-141, kernel_ir.cpp), value
// arithmetic (value.hpp, kernel_ir.cpp:46-107), the s-expression text form
// (kernel_text.hpp), the WLP/TLP wrappers (wlp.hpp:43-59), the model bodies
// (models.cpp:124-268, written here as kernel text), and `simulate` — which flattens a
// program into typed stack bytecode (include/wlp_b200.h) and runs it on the GPU through
// wlp_ir_simulate. A small extern "C" surface at the end serves the Python mirror.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstring>
#include <limits>
#include <utility>

#include "warpsim_ir_b200.hpp"
#include "wlp_b200.h"

namespace warpsim {
namespace {

[[noreturn]] void raise_status(int code) {
    const std::string msg = wlp_last_error();
    switch (code) {
        case WLP_EDOMAIN: throw DomainError(msg);
        case WLP_EPLAN: throw PlanError(msg);
        case WLP_EFAULT: throw FaultError(msg);
        default: throw Error(msg);
    }
}

[[noreturn]] void lane_fault(const char* where, const std::string& what) {
    throw FaultError(std::string(where) + ": " + what);
}

bool lt(const Value& a, const Value& b) { return a.is_int() && b.is_int() ? a.i < b.i : a.as_real() < b.as_real(); }
bool eq(const Value& a, const Value& b) { return a.is_int() && b.is_int() ? a.i == b.i : a.as_real() == b.as_real(); }

std::uint64_t bits_of(double x) {
    std::uint64_t u;
    std::memcpy(&u, &x, sizeof u);
    return u;
}

}  // namespace

// ---- values --------------------------------------------------------------------------

bool Value::bit_equal(const Value& o) const {
    if (type != o.type) return false;
    return is_int() ? i == o.i : bits_of(r) == bits_of(o.r);
}

std::string Value::str() const { return is_int() ? std::to_string(i) : std::to_string(r); }

Value apply_bin(BinOp op, const Value& a, const Value& b, const char* where) {
    const bool ints = a.is_int() && b.is_int();
    const double x = a.as_real(), y = b.as_real();
    switch (op) {
        case BinOp::Add: return ints ? Value::integer(a.i + b.i) : Value::real(x + y);
        case BinOp::Sub: return ints ? Value::integer(a.i - b.i) : Value::real(x - y);
        case BinOp::Mul: return ints ? Value::integer(a.i * b.i) : Value::real(x * y);
        case BinOp::Div:
            if (ints) {
                if (b.i == 0) lane_fault(where, "integer division by zero");
                return Value::integer(a.i / b.i);
            }
            if (y == 0.0) lane_fault(where, "division by zero");
            return Value::real(x / y);
        case BinOp::Mod:
            if (ints) {
                if (b.i == 0) lane_fault(where, "integer modulo by zero");
                return Value::integer(a.i % b.i);
            }
            if (y == 0.0) lane_fault(where, "modulo by zero");
            return Value::real(std::fmod(x, y));
        case BinOp::Lt: return Value::integer(lt(a, b));
        case BinOp::Le: return Value::integer(!lt(b, a));
        case BinOp::Gt: return Value::integer(lt(b, a));
        case BinOp::Ge: return Value::integer(!lt(a, b));
        case BinOp::Eq: return Value::integer(eq(a, b));
        case BinOp::Ne: return Value::integer(!eq(a, b));
        case BinOp::And: return Value::integer(a.truthy() && b.truthy());
        case BinOp::Or: return Value::integer(a.truthy() || b.truthy());
    }
    lane_fault(where, "unknown binary op");
}

Value apply_un(UnOp op, const Value& a, const char* where) {
    switch (op) {
        case UnOp::Neg: return a.is_int() ? Value::integer(-a.i) : Value::real(-a.r);
        case UnOp::Log: {
            const double x = a.as_real();
            if (!(x > 0.0)) lane_fault(where, "log of a non-positive value");
            return Value::real(std::log(x));
        }
        case UnOp::Floor: {
            if (a.is_int()) return a;
            const double f = std::floor(a.r);
            if (!(f >= -9.2233720368547758e18 && f <= 9.2233720368547758e18))
                lane_fault(where, "floor result outside the integer range");
            return Value::integer(f >= 9.2233720368547758e18 ? std::numeric_limits<std::int64_t>::min()
                                                              : static_cast<std::int64_t>(f));
        }
    }
    lane_fault(where, "unknown unary op");
}

namespace {
constexpr const char* kBinNames[] = {"add", "sub", "mul", "div", "mod", "lt", "le",
                                     "gt",  "ge",  "eq",  "ne",  "and", "or"};
constexpr const char* kUnNames[] = {"neg", "log", "floor"};
constexpr const char* kSregNames[] = {"tid.x",  "tid.y",  "tid.z",  "bid.x",  "bid.y",   "bdim.x",
                                      "bdim.y", "bdim.z", "gdim.x", "gdim.y", "warpsize"};
}  // namespace

const char* bin_op_name(BinOp op) { return kBinNames[static_cast<int>(op)]; }
const char* un_op_name(UnOp op) { return kUnNames[static_cast<int>(op)]; }

// ---- launch geometry (kernel_ir.hpp:47-63) -----------------------------------------------

void validate_launch(const LaunchConfig& c) {
    if (c.blockDim.x < 1 || c.blockDim.y < 1 || c.blockDim.z < 1)
        throw DomainError("launch: blockDim components must be >= 1");
    if (c.gridDim.x < 1 || c.gridDim.y < 1) throw DomainError("launch: gridDim components must be >= 1");
    if (c.warpSize < 1 || c.warpSize > 64) throw DomainError("launch: warpSize must be in [1,64]");
}

std::optional<std::string> launch_warning(const LaunchConfig& c) {
    const std::int64_t tpb = c.threads_per_block();
    if (tpb % c.warpSize == 0) return std::nullopt;
    return "block size " + std::to_string(tpb) + " is not a multiple of warpSize " + std::to_string(c.warpSize) +
           "; trailing warp runs partially populated";
}

namespace {
void check_thread(const ThreadCoord& t, const LaunchConfig& c) {
    if (t.x < 0 || t.y < 0 || t.z < 0 || t.x >= c.blockDim.x || t.y >= c.blockDim.y || t.z >= c.blockDim.z)
        throw DomainError("thread coordinate outside blockDim");
}
}  // namespace

std::int64_t intra_block_thread_id(const ThreadCoord& t, const LaunchConfig& c) {
    check_thread(t, c);
    return t.x + c.blockDim.x * (t.y + c.blockDim.y * t.z);
}

std::int64_t linear_thread_id(const ThreadCoord& t, const BlockCoord& b, const LaunchConfig& c) {
    if (b.x < 0 || b.y < 0 || b.x >= c.gridDim.x || b.y >= c.gridDim.y)
        throw DomainError("block coordinate outside gridDim");
    check_thread(t, c);
    const std::int64_t block = b.x + c.gridDim.x * b.y;
    return t.x + c.blockDim.x * (t.y + c.blockDim.y * (t.z + c.blockDim.z * block));
}

std::int64_t warp_index(const ThreadCoord& t, const BlockCoord& b, const LaunchConfig& c) {
    return linear_thread_id(t, b, c) / c.warpSize;
}

bool is_warp_leader(const ThreadCoord& t, const LaunchConfig& c) { return intra_block_thread_id(t, c) % c.warpSize == 0; }

// ---- program builder (kernel_ir.cpp) --------------------------------------------------

int KernelProgram::param_slot(const std::string& name) const {
    for (std::size_t k = 0; k < params.size(); ++k)
        if (params[k].name == name) return static_cast<int>(k);
    return -1;
}

int KernelProgram::local_slot(const std::string& name) const {
    for (std::size_t k = 0; k < locals.size(); ++k)
        if (locals[k].name == name) return static_cast<int>(k);
    return -1;
}

int KernelProgram::add_param(const std::string& name, ParamKind kind) {
    if (param_slot(name) >= 0 || local_slot(name) >= 0) throw DomainError("duplicate declaration: " + name);
    params.push_back(ParamDecl{name, kind});
    return static_cast<int>(params.size()) - 1;
}

int KernelProgram::add_local(const std::string& name, ValueType type) {
    if (param_slot(name) >= 0 || local_slot(name) >= 0) throw DomainError("duplicate declaration: " + name);
    locals.push_back(LocalDecl{name, type});
    return static_cast<int>(locals.size()) - 1;
}

namespace {
ExprId push_expr(KernelProgram& p, Expr e) {
    p.exprs.push_back(std::move(e));
    return static_cast<ExprId>(p.exprs.size()) - 1;
}
}  // namespace

ExprId KernelProgram::ci(std::int64_t v) {
    Expr e;
    e.konst = Value::integer(v);
    return push_expr(*this, e);
}

ExprId KernelProgram::cr(double v) {
    Expr e;
    e.konst = Value::real(v);
    return push_expr(*this, e);
}

ExprId KernelProgram::local(const std::string& name) {
    const int s = local_slot(name);
    if (s < 0) throw DomainError("reference to undeclared local: " + name);
    Expr e;
    e.kind = Expr::Kind::Local;
    e.slot = s;
    return push_expr(*this, e);
}

ExprId KernelProgram::param(const std::string& name) {
    const int s = param_slot(name);
    if (s < 0) throw DomainError("reference to undeclared param: " + name);
    if (params[s].kind == ParamKind::Array) throw DomainError("array param used as a scalar: " + name);
    Expr e;
    e.kind = Expr::Kind::Param;
    e.slot = s;
    return push_expr(*this, e);
}

ExprId KernelProgram::sreg(Sreg r) {
    Expr e;
    e.kind = Expr::Kind::Special;
    e.sreg = r;
    return push_expr(*this, e);
}

ExprId KernelProgram::draw() {
    Expr e;
    e.kind = Expr::Kind::Draw;
    return push_expr(*this, e);
}

ExprId KernelProgram::bin(BinOp op, ExprId a, ExprId b) {
    Expr e;
    e.kind = Expr::Kind::Bin;
    e.bop = op;
    e.a = a;
    e.b = b;
    return push_expr(*this, e);
}

ExprId KernelProgram::un(UnOp op, ExprId a) {
    Expr e;
    e.kind = Expr::Kind::Un;
    e.uop = op;
    e.a = a;
    return push_expr(*this, e);
}

Statement KernelProgram::assign(const std::string& name, ExprId value) const {
    const int s = local_slot(name);
    if (s < 0) throw DomainError("assign to undeclared local: " + name);
    return Statement{StmtKind::Assign, s, value, -1, {}, {}};
}

Statement KernelProgram::load(const std::string& name, const std::string& array, ExprId index) const {
    const int s = local_slot(name);
    const int a = param_slot(array);
    if (s < 0) throw DomainError("load into undeclared local: " + name);
    if (a < 0 || params[a].kind != ParamKind::Array) throw DomainError("load from undeclared array: " + array);
    if (locals[s].type != ValueType::Real) throw DomainError("load target must be a real local: " + name);
    return Statement{StmtKind::Load, s, index, a, {}, {}};
}

Statement KernelProgram::store(const std::string& array, ExprId index, ExprId value) const {
    const int a = param_slot(array);
    if (a < 0 || params[a].kind != ParamKind::Array) throw DomainError("store to undeclared array: " + array);
    return Statement{StmtKind::Store, a, index, value, {}, {}};
}

Statement KernelProgram::if_(ExprId cond, std::vector<Statement> then_body, std::vector<Statement> else_body) {
    return Statement{StmtKind::If, -1, cond, -1, std::move(then_body), std::move(else_body)};
}

Statement KernelProgram::while_(ExprId cond, std::vector<Statement> loop_body) {
    return Statement{StmtKind::While, -1, cond, -1, std::move(loop_body), {}};
}

Statement KernelProgram::halt() { return Statement{StmtKind::Halt, -1, -1, -1, {}, {}}; }

namespace {

void check_expr(const KernelProgram& p, ExprId id) {
    if (id < 0 || id >= static_cast<ExprId>(p.exprs.size())) throw DomainError("expression reference out of range");
    const Expr& e = p.exprs[id];
    switch (e.kind) {
        case Expr::Kind::Local:
            if (e.slot < 0 || e.slot >= static_cast<int>(p.locals.size()))
                throw DomainError("local reference out of range");
            break;
        case Expr::Kind::Param:
            if (e.slot < 0 || e.slot >= static_cast<int>(p.params.size()))
                throw DomainError("param reference out of range");
            if (p.params[e.slot].kind == ParamKind::Array)
                throw DomainError("array param used as a scalar: " + p.params[e.slot].name);
            break;
        case Expr::Kind::Bin:
            check_expr(p, e.a);
            check_expr(p, e.b);
            break;
        case Expr::Kind::Un: check_expr(p, e.a); break;
        default: break;
    }
}

bool is_array(const KernelProgram& p, int slot) {
    return slot >= 0 && slot < static_cast<int>(p.params.size()) && p.params[slot].kind == ParamKind::Array;
}

void check_list(const KernelProgram& p, const std::vector<Statement>& list) {
    const int nl = static_cast<int>(p.locals.size());
    for (const Statement& st : list) {
        switch (st.kind) {
            case StmtKind::Assign:
                if (st.slot < 0 || st.slot >= nl) throw DomainError("assign target out of range");
                check_expr(p, st.expr_a);
                break;
            case StmtKind::Load:
                if (st.slot < 0 || st.slot >= nl) throw DomainError("load target out of range");
                if (!is_array(p, st.expr_b)) throw DomainError("load source is not an array param");
                check_expr(p, st.expr_a);
                break;
            case StmtKind::Store:
                if (!is_array(p, st.slot)) throw DomainError("store target is not an array param");
                check_expr(p, st.expr_a);
                check_expr(p, st.expr_b);
                break;
            case StmtKind::If:
                check_expr(p, st.expr_a);
                check_list(p, st.body1);
                check_list(p, st.body2);
                break;
            case StmtKind::While:
                check_expr(p, st.expr_a);
                if (!st.body2.empty()) throw DomainError("while carries no else body");
                check_list(p, st.body1);
                break;
            case StmtKind::Halt: break;
        }
    }
}

}  // namespace

void KernelProgram::finalize() const { check_list(*this, body); }

ParamEnv bind_params(const KernelProgram& prog, const std::map<std::string, Value>& scalars, GlobalMemory& memory) {
    ParamEnv env;
    env.scalars.assign(prog.params.size(), Value{});
    env.arrays.assign(prog.params.size(), nullptr);
    for (std::size_t k = 0; k < prog.params.size(); ++k) {
        const ParamDecl& d = prog.params[k];
        if (d.kind == ParamKind::Array) {
            auto it = memory.arrays.find(d.name);
            if (it == memory.arrays.end()) throw DomainError("no array bound for param: " + d.name);
            env.arrays[k] = &it->second;
            continue;
        }
        auto it = scalars.find(d.name);
        if (it == scalars.end()) throw DomainError("no value bound for param: " + d.name);
        if (d.kind == ParamKind::Int && !it->second.is_int()) throw DomainError("param expects an integer: " + d.name);
        env.scalars[k] = d.kind == ParamKind::Real ? Value::real(it->second.as_real()) : it->second;
    }
    return env;
}

// ---- text form (kernel_text.hpp) ------------------------------------------------------

namespace {

bool sreg_of(const std::string& s, Sreg& out) {
    for (int k = 0; k < 11; ++k)
        if (s == kSregNames[k]) {
            out = static_cast<Sreg>(k);
            return true;
        }
    return false;
}

bool ident(const std::string& s) {
    if (s.empty() || !(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_')) return false;
    for (char ch : s)
        if (!(std::isalnum(static_cast<unsigned char>(ch)) || ch == '_')) return false;
    Sreg r;
    return !sreg_of(s, r);
}

// Shortest round-trip form; a real literal always shows a '.', an exponent, or inf/nan.
std::string real_literal(double v) {
    char buf[64];
    const auto res = std::to_chars(buf, buf + sizeof buf, v);
    std::string s(buf, res.ptr);
    if (s.find_first_of(".eEni") == std::string::npos) s += ".0";
    return s;
}

struct Writer {
    const KernelProgram& p;
    std::string out;

    void expr(ExprId id) {
        const Expr& e = p.exprs[id];
        switch (e.kind) {
            case Expr::Kind::Const: out += e.konst.is_int() ? std::to_string(e.konst.i) : real_literal(e.konst.r); break;
            case Expr::Kind::Local: out += p.locals[e.slot].name; break;
            case Expr::Kind::Param: out += p.params[e.slot].name; break;
            case Expr::Kind::Special: out += kSregNames[static_cast<int>(e.sreg)]; break;
            case Expr::Kind::Draw: out += "(draw)"; break;
            case Expr::Kind::Bin:
                out += std::string("(") + bin_op_name(e.bop) + " ";
                expr(e.a);
                out += " ";
                expr(e.b);
                out += ")";
                break;
            case Expr::Kind::Un:
                out += std::string("(") + un_op_name(e.uop) + " ";
                expr(e.a);
                out += ")";
                break;
        }
    }

    void list(const std::vector<Statement>& stmts, int indent) {
        for (const Statement& st : stmts) {
            out += "\n";
            stmt(st, indent);
        }
    }

    void stmt(const Statement& st, int indent) {
        const std::string pad(static_cast<std::size_t>(indent), ' ');
        out += pad;
        switch (st.kind) {
            case StmtKind::Assign:
                out += "(assign " + p.locals[st.slot].name + " ";
                expr(st.expr_a);
                out += ")";
                break;
            case StmtKind::Load:
                out += "(load " + p.locals[st.slot].name + " " + p.params[st.expr_b].name + " ";
                expr(st.expr_a);
                out += ")";
                break;
            case StmtKind::Store:
                out += "(store " + p.params[st.slot].name + " ";
                expr(st.expr_a);
                out += " ";
                expr(st.expr_b);
                out += ")";
                break;
            case StmtKind::Halt: out += "(halt)"; break;
            case StmtKind::If:
                out += "(if ";
                expr(st.expr_a);
                out += "\n" + pad + "  (then";
                list(st.body1, indent + 4);
                out += ")";
                if (!st.body2.empty()) {
                    out += "\n" + pad + "  (else";
                    list(st.body2, indent + 4);
                    out += ")";
                }
                out += ")";
                break;
            case StmtKind::While:
                out += "(while ";
                expr(st.expr_a);
                list(st.body1, indent + 2);
                out += ")";
                break;
        }
    }
};

// S-expression tree with line numbers.
struct Node {
    bool atom = false;
    std::string text;
    std::vector<Node> kids;
    int line = 0;
    const std::string& head() const {
        static const std::string none;
        return (!atom && !kids.empty() && kids[0].atom) ? kids[0].text : none;
    }
};

[[noreturn]] void syntax(int line, const std::string& what) {
    throw ParseError("line " + std::to_string(line) + ": " + what);
}

std::vector<Node> read_forms(const std::string& text) {
    std::vector<Node> open(1);
    int line = 1;
    for (std::size_t k = 0; k < text.size();) {
        const char ch = text[k];
        if (ch == '\n') {
            ++line;
            ++k;
        } else if (std::isspace(static_cast<unsigned char>(ch))) {
            ++k;
        } else if (ch == ';') {
            while (k < text.size() && text[k] != '\n') ++k;
        } else if (ch == '(') {
            Node n;
            n.line = line;
            open.push_back(std::move(n));
            ++k;
        } else if (ch == ')') {
            if (open.size() < 2) syntax(line, "unmatched ')'");
            Node n = std::move(open.back());
            open.pop_back();
            open.back().kids.push_back(std::move(n));
            ++k;
        } else {
            const std::size_t b = k;
            while (k < text.size() && !std::isspace(static_cast<unsigned char>(text[k])) && text[k] != '(' &&
                   text[k] != ')' && text[k] != ';')
                ++k;
            Node n;
            n.atom = true;
            n.text = text.substr(b, k - b);
            n.line = line;
            open.back().kids.push_back(std::move(n));
        }
    }
    if (open.size() != 1) syntax(line, "unterminated '('");
    return std::move(open[0].kids);
}

template <class T>
bool number(const std::string& s, T& v) {
    const auto res = std::from_chars(s.data(), s.data() + s.size(), v);
    return res.ec == std::errc{} && res.ptr == s.data() + s.size();
}

struct Reader {
    KernelProgram& p;

    ExprId expr(const Node& n) {
        if (n.atom) {
            Sreg r;
            std::int64_t iv;
            double rv;
            if (sreg_of(n.text, r)) return p.sreg(r);
            if (number(n.text, iv)) return p.ci(iv);
            if (number(n.text, rv)) return p.cr(rv);
            if (p.local_slot(n.text) >= 0) return p.local(n.text);
            const int ps = p.param_slot(n.text);
            if (ps >= 0) {
                if (p.params[ps].kind == ParamKind::Array) syntax(n.line, "array '" + n.text + "' used as a scalar");
                return p.param(n.text);
            }
            syntax(n.line, "unknown name '" + n.text + "'");
        }
        const std::string& h = n.head();
        if (h.empty()) syntax(n.line, "expected an expression");
        const std::size_t argc = n.kids.size() - 1;
        if (h == "draw") {
            if (argc != 0) syntax(n.line, "(draw) takes no arguments");
            return p.draw();
        }
        for (int k = 0; k < 3; ++k)
            if (h == kUnNames[k]) {
                if (argc != 1) syntax(n.line, "(" + h + " ...) takes one argument");
                return p.un(static_cast<UnOp>(k), expr(n.kids[1]));
            }
        for (int k = 0; k < 13; ++k)
            if (h == kBinNames[k]) {
                if (argc != 2) syntax(n.line, "(" + h + " ...) takes two arguments");
                const ExprId a = expr(n.kids[1]);
                const ExprId b = expr(n.kids[2]);
                return p.bin(static_cast<BinOp>(k), a, b);
            }
        syntax(n.line, "unknown operator '" + h + "'");
    }

    std::vector<Statement> list(const Node& parent, std::size_t from) {
        std::vector<Statement> out;
        for (std::size_t k = from; k < parent.kids.size(); ++k) out.push_back(stmt(parent.kids[k]));
        return out;
    }

    Statement stmt(const Node& n) {
        if (n.atom) syntax(n.line, "expected a statement list, got '" + n.text + "'");
        const std::string& h = n.head();
        const std::size_t argc = n.kids.size() - 1;
        try {
            if (h == "assign") {
                if (argc != 2 || !n.kids[1].atom) syntax(n.line, "(assign name expr)");
                return p.assign(n.kids[1].text, expr(n.kids[2]));
            }
            if (h == "load") {
                if (argc != 3 || !n.kids[1].atom || !n.kids[2].atom) syntax(n.line, "(load local array index)");
                return p.load(n.kids[1].text, n.kids[2].text, expr(n.kids[3]));
            }
            if (h == "store") {
                if (argc != 3 || !n.kids[1].atom) syntax(n.line, "(store array index value)");
                const ExprId idx = expr(n.kids[2]);
                const ExprId val = expr(n.kids[3]);
                return p.store(n.kids[1].text, idx, val);
            }
            if (h == "halt") {
                if (argc != 0) syntax(n.line, "(halt) takes no arguments");
                return KernelProgram::halt();
            }
            if (h == "if") {
                if (argc < 2 || argc > 3) syntax(n.line, "(if cond (then ...) [(else ...)])");
                const ExprId cond = expr(n.kids[1]);
                const Node& t = n.kids[2];
                if (t.atom || t.head() != "then") syntax(t.line, "expected (then ...)");
                std::vector<Statement> tb = list(t, 1), eb;
                if (argc == 3) {
                    const Node& e = n.kids[3];
                    if (e.atom || e.head() != "else") syntax(e.line, "expected (else ...)");
                    eb = list(e, 1);
                }
                return KernelProgram::if_(cond, std::move(tb), std::move(eb));
            }
            if (h == "while") {
                if (argc < 1) syntax(n.line, "(while cond stmts...)");
                const ExprId cond = expr(n.kids[1]);
                return KernelProgram::while_(cond, list(n, 2));
            }
        } catch (const DomainError& e) {
            syntax(n.line, e.what());
        }
        syntax(n.line, h.empty() ? "expected a statement" : "unknown statement '" + h + "'");
    }
};

}  // namespace

std::string dump_kernel(const KernelProgram& prog) {
    prog.finalize();
    for (const ParamDecl& d : prog.params)
        if (!ident(d.name)) throw DomainError("unprintable param name: " + d.name);
    for (const LocalDecl& d : prog.locals)
        if (!ident(d.name)) throw DomainError("unprintable local name: " + d.name);
    Writer w{prog, "(kernel"};
    static const char* pk[] = {"int", "real", "array"};
    for (const ParamDecl& d : prog.params) w.out += "\n  (param " + d.name + " " + pk[static_cast<int>(d.kind)] + ")";
    for (const LocalDecl& d : prog.locals)
        w.out += "\n  (local " + d.name + " " + (d.type == ValueType::Int ? "int" : "real") + ")";
    w.out += "\n  (body";
    w.list(prog.body, 4);
    w.out += "))\n";
    return w.out;
}

KernelProgram parse_kernel(const std::string& text) {
    const std::vector<Node> top = read_forms(text);
    if (top.size() != 1 || top[0].atom || top[0].head() != "kernel")
        throw ParseError("line 1: expected a single (kernel ...) form");
    const Node& k = top[0];
    KernelProgram p;
    std::size_t at = 1;
    for (; at < k.kids.size() && k.kids[at].head() != "body"; ++at) {
        const Node& d = k.kids[at];
        const std::string& h = d.head();
        if (h != "param" && h != "local") syntax(d.line, "expected (param ...), (local ...) or (body ...)");
        if (d.kids.size() != 3 || !d.kids[1].atom || !d.kids[2].atom) syntax(d.line, "(" + h + " name kind)");
        const std::string& name = d.kids[1].text;
        const std::string& kind = d.kids[2].text;
        if (!ident(name)) syntax(d.kids[1].line, "bad name '" + name + "'");
        try {
            if (h == "param") {
                if (kind == "int")
                    p.add_param(name, ParamKind::Int);
                else if (kind == "real")
                    p.add_param(name, ParamKind::Real);
                else if (kind == "array")
                    p.add_param(name, ParamKind::Array);
                else
                    syntax(d.kids[2].line, "param kind must be int, real or array");
            } else {
                if (kind == "int")
                    p.add_local(name, ValueType::Int);
                else if (kind == "real")
                    p.add_local(name, ValueType::Real);
                else
                    syntax(d.kids[2].line, "local kind must be int or real");
            }
        } catch (const DomainError& e) {
            syntax(d.line, e.what());
        }
    }
    if (at >= k.kids.size()) throw ParseError("line " + std::to_string(k.line) + ": missing (body ...)");
    Reader r{p};
    p.body = r.list(k.kids[at], 1);
    if (at + 1 != k.kids.size()) syntax(k.kids[at + 1].line, "unexpected form after (body ...)");
    p.finalize();
    return p;
}

// ---- WLP / TLP wrappers (wlp.hpp:43-59) --------------------------------------------------

namespace {

// tid.x + bdim.x*(tid.y + bdim.y*(tid.z + bdim.z*(bid.x + gdim.x*bid.y)))
ExprId global_tid(KernelProgram& p) {
    const ExprId block = p.bin(BinOp::Add, p.sreg(Sreg::BidX), p.bin(BinOp::Mul, p.sreg(Sreg::GDimX), p.sreg(Sreg::BidY)));
    const ExprId z = p.bin(BinOp::Add, p.sreg(Sreg::TidZ), p.bin(BinOp::Mul, p.sreg(Sreg::BDimZ), block));
    const ExprId y = p.bin(BinOp::Add, p.sreg(Sreg::TidY), p.bin(BinOp::Mul, p.sreg(Sreg::BDimY), z));
    return p.bin(BinOp::Add, p.sreg(Sreg::TidX), p.bin(BinOp::Mul, p.sreg(Sreg::BDimX), y));
}

// tid.x + bdim.x*(tid.y + bdim.y*tid.z)
ExprId block_tid(KernelProgram& p) {
    const ExprId y = p.bin(BinOp::Add, p.sreg(Sreg::TidY), p.bin(BinOp::Mul, p.sreg(Sreg::BDimY), p.sreg(Sreg::TidZ)));
    return p.bin(BinOp::Add, p.sreg(Sreg::TidX), p.bin(BinOp::Mul, p.sreg(Sreg::BDimX), y));
}

void require_wrappable(const KernelProgram& body) {
    const int rid = body.local_slot("rid");
    if (rid < 0 || body.locals[rid].type != ValueType::Int)
        throw DomainError("wrap: body must declare an Int local 'rid'");
    const int reps = body.param_slot("replications");
    if (reps < 0 || body.params[reps].kind != ParamKind::Int)
        throw DomainError("wrap: body must declare an Int param 'replications'");
    if (!body.body.empty() && body.body.front().kind == StmtKind::Assign && body.body.front().slot == rid)
        throw DomainError("wrap: body already initializes 'rid' — double wrap");
}

KernelProgram wrap(const KernelProgram& body, bool wlp) {
    require_wrappable(body);
    KernelProgram p = body;
    std::vector<Statement> inner = std::move(p.body);
    p.body.clear();
    if (wlp) {  // rid := warpIdx; lanes other than the warp's first halt
        p.body.push_back(p.assign("rid", p.bin(BinOp::Div, global_tid(p), p.sreg(Sreg::WarpSize))));
        const ExprId lane = p.bin(BinOp::Mod, block_tid(p), p.sreg(Sreg::WarpSize));
        p.body.push_back(KernelProgram::if_(p.bin(BinOp::Ne, lane, p.ci(0)), {KernelProgram::halt()}));
    } else {
        p.body.push_back(p.assign("rid", global_tid(p)));
    }
    p.body.push_back(KernelProgram::if_(p.bin(BinOp::Lt, p.local("rid"), p.param("replications")), std::move(inner)));
    p.finalize();
    return p;
}

}  // namespace

KernelProgram wrap_wlp(const KernelProgram& body) { return wrap(body, true); }
KernelProgram wrap_tlp(const KernelProgram& body) { return wrap(body, false); }

std::vector<RngState> assign_lane_streams(ExecutionMode mode, const LaunchConfig& cfg,
                                          const std::vector<RngState>& streams) {
    if (mode != ExecutionMode::Wlp || streams.empty()) return streams;
    std::vector<RngState> lanes((streams.size() - 1) * static_cast<std::size_t>(cfg.warpSize) + 1);
    for (std::size_t r = 0; r < streams.size(); ++r) lanes[r * static_cast<std::size_t>(cfg.warpSize)] = streams[r];
    return lanes;
}

// ---- model bodies (models.cpp:124-268), as kernel text ---------------------------------

namespace {

// pi: the hit count lives in global memory (cnt[rid]), loaded and stored per point.
constexpr const char* kPiBody = R"((kernel
  (param replications int) (param draws int) (param cnt array) (param out array)
  (local rid int) (local i int) (local x real) (local y real) (local c real)
  (body
    (assign i 0)
    (while (lt i draws)
      (assign x (draw))
      (assign y (draw))
      (load c cnt rid)
      (store cnt rid (add c (le (add (mul x x) (mul y y)) 1.0)))
      (assign i (add i 1)))
    (load c cnt rid)
    (store out rid (div (mul 4.0 c) draws))))
)";

// mm1: Lindley recursion with exponential draws -log(1 - u)/rate.
constexpr const char* kMm1Body = R"((kernel
  (param replications int) (param clients int) (param lambda real) (param mu real)
  (param outIdle array) (param outWait array) (param outSys array)
  (local rid int) (local i int) (local a real) (local s real) (local t real) (local w real)
  (local idle real) (local sumw real) (local sums real)
  (body
    (assign i 0)
    (while (lt i clients)
      (assign a (div (neg (log (sub 1.0 (draw)))) lambda))
      (assign t (sub (add w s) a))
      (if (lt t 0.0)
        (then (assign idle (sub idle t)) (assign w 0.0))
        (else (assign w t)))
      (assign s (div (neg (log (sub 1.0 (draw)))) mu))
      (assign sumw (add sumw w))
      (assign sums (add sums (add w s)))
      (assign i (add i 1)))
    (store outIdle rid (div idle clients))
    (store outWait rid (div sumw clients))
    (store outSys rid (div sums clients))))
)";

// walk: positions in global memory, a 4-way nested branch per step.
constexpr const char* kWalkBody = R"((kernel
  (param replications int) (param steps int) (param chunks int)
  (param posX array) (param posY array) (param out array)
  (local rid int) (local i int) (local u real) (local v real) (local d int) (local px real) (local py real)
  (body
    (assign i 0)
    (while (lt i steps)
      (assign u (draw))
      (assign v (draw))
      (assign d (floor (mul 4.0 u)))
      (if (eq d 0)
        (then (load px posX rid) (store posX rid (add px 1.0)))
        (else
          (if (eq d 1)
            (then (load px posX rid) (store posX rid (sub px 1.0)))
            (else
              (if (eq d 2)
                (then (load py posY rid) (store posY rid (add py 1.0)))
                (else (load py posY rid) (store posY rid (sub py 1.0))))))))
      (assign i (add i 1)))
    (load px posX rid)
    (store out rid (mod (add (mod px chunks) chunks) chunks))))
)";

}  // namespace

KernelProgram build_model_body(ModelKind model) {
    switch (model) {
        case ModelKind::Pi: return parse_kernel(kPiBody);
        case ModelKind::Mm1: return parse_kernel(kMm1Body);
        case ModelKind::Walk: return parse_kernel(kWalkBody);
    }
    throw DomainError("unknown model");
}

KernelBundle build_kernel(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                          int tlp_block_size) {
    const std::optional<std::string> pw = validate_params(model, p);
    KernelProgram body = build_model_body(model);
    const LaunchPlan plan = plan_launch(p.replications, mode, prof, tlp_block_size);
    KernelBundle b;
    b.program = mode == ExecutionMode::Sequential ? std::move(body)
                : mode == ExecutionMode::Tlp      ? wrap_tlp(body)
                                                  : wrap_wlp(body);
    b.cfg = plan.cfg;
    if (pw && plan.warning)
        b.warning = *pw + "; " + *plan.warning;
    else
        b.warning = pw ? pw : plan.warning;
    const std::int64_t R = p.replications;
    b.scalars["replications"] = Value::integer(R);
    switch (model) {
        case ModelKind::Pi:
            b.scalars["draws"] = Value::integer(p.draws);
            b.arrays = {{"cnt", R}, {"out", R}};
            b.outputs = {"out"};
            b.primary = "out";
            break;
        case ModelKind::Mm1:
            b.scalars["clients"] = Value::integer(p.clients);
            b.scalars["lambda"] = Value::real(p.lambda);
            b.scalars["mu"] = Value::real(p.mu);
            b.arrays = {{"outIdle", R}, {"outWait", R}, {"outSys", R}};
            b.outputs = {"outIdle", "outWait", "outSys"};
            b.primary = "outWait";
            break;
        case ModelKind::Walk:
            b.scalars["steps"] = Value::integer(p.steps);
            b.scalars["chunks"] = Value::integer(p.chunks);
            b.arrays = {{"posX", R}, {"posY", R}, {"out", R}};
            b.outputs = {"out"};
            b.primary = "out";
            break;
    }
    return b;
}

// ---- flattening to the device form (include/wlp_b200.h) ----------------------------------

struct Flat {
    std::vector<wlp_ir_stmt> stmts;
    std::vector<std::int32_t> code;
    std::vector<std::int64_t> local_init, param_bits;
    std::vector<std::int32_t> param_is_array;
    std::int32_t top_begin = 0, top_end = 0;
};

struct Compiler {
    const KernelProgram& p;
    Flat& f;

    void op(int o) { f.code.push_back(o); }

    ValueType expr(ExprId id) {
        const Expr& e = p.exprs[id];
        switch (e.kind) {
            case Expr::Kind::Const: {
                const std::uint64_t u = e.konst.is_int() ? static_cast<std::uint64_t>(e.konst.i) : bits_of(e.konst.r);
                op(WLP_IR_OP_CONST);
                op(static_cast<std::int32_t>(u & 0xFFFFFFFFu));
                op(static_cast<std::int32_t>(u >> 32));
                return e.konst.type;
            }
            case Expr::Kind::Local:
                op(WLP_IR_OP_LOCAL);
                op(e.slot);
                return p.locals[e.slot].type;
            case Expr::Kind::Param:
                op(WLP_IR_OP_PARAM);
                op(e.slot);
                return p.params[e.slot].kind == ParamKind::Int ? ValueType::Int : ValueType::Real;
            case Expr::Kind::Special:
                op(WLP_IR_OP_SREG);
                op(static_cast<int>(e.sreg));
                return ValueType::Int;
            case Expr::Kind::Draw: op(WLP_IR_OP_DRAW); return ValueType::Real;
            case Expr::Kind::Un: {
                const ValueType t = expr(e.a);
                switch (e.uop) {
                    case UnOp::Neg: op(t == ValueType::Int ? WLP_IR_OP_NEG_I : WLP_IR_OP_NEG_R); return t;
                    case UnOp::Log:
                        if (t == ValueType::Int) op(WLP_IR_OP_I2R_0);
                        op(WLP_IR_OP_LOG);
                        return ValueType::Real;
                    case UnOp::Floor:
                        if (t == ValueType::Real) op(WLP_IR_OP_FLOOR);  // floor of an int is the int
                        return ValueType::Int;
                }
                break;
            }
            case Expr::Kind::Bin: {
                const ValueType ta = expr(e.a), tb = expr(e.b);
                const bool ints = ta == ValueType::Int && tb == ValueType::Int;
                const int k = static_cast<int>(e.bop);
                if (e.bop == BinOp::And || e.bop == BinOp::Or) {
                    if (ta == ValueType::Real) op(WLP_IR_OP_TRUTH_1);
                    if (tb == ValueType::Real) op(WLP_IR_OP_TRUTH_0);
                    op(e.bop == BinOp::And ? WLP_IR_OP_AND : WLP_IR_OP_OR);
                    return ValueType::Int;
                }
                if (!ints) {
                    if (ta == ValueType::Int) op(WLP_IR_OP_I2R_1);
                    if (tb == ValueType::Int) op(WLP_IR_OP_I2R_0);
                }
                if (k <= static_cast<int>(BinOp::Mod)) {  // arithmetic
                    op((ints ? WLP_IR_OP_ADD_I : WLP_IR_OP_ADD_R) + k);
                    return ints ? ValueType::Int : ValueType::Real;
                }
                op((ints ? WLP_IR_OP_LT_I : WLP_IR_OP_LT_R) + (k - static_cast<int>(BinOp::Lt)));
                return ValueType::Int;
            }
        }
        throw DomainError("ir: unknown expression kind");
    }

    // Emits a whole expression; returns its code offset.
    std::int32_t root(ExprId id, ValueType* type = nullptr, bool truth = false, bool as_real = false) {
        const std::int32_t at = static_cast<std::int32_t>(f.code.size());
        const ValueType t = expr(id);
        if (truth && t == ValueType::Real) op(WLP_IR_OP_TRUTH_0);
        if (as_real && t == ValueType::Int) op(WLP_IR_OP_I2R_0);
        op(WLP_IR_OP_END);
        if (type) *type = t;
        return at;
    }

    // Lays out one statement list as a contiguous range, children after it.
    std::pair<std::int32_t, std::int32_t> place(const std::vector<Statement>& list) {
        const std::int32_t begin = static_cast<std::int32_t>(f.stmts.size());
        f.stmts.resize(f.stmts.size() + list.size());
        for (std::size_t k = 0; k < list.size(); ++k) {
            const Statement& st = list[k];
            wlp_ir_stmt s{};
            s.kind = static_cast<std::int32_t>(st.kind);
            s.slot = st.slot;
            s.arr = -1;
            s.code_a = s.code_b = -1;
            ValueType t;
            switch (st.kind) {
                case StmtKind::Assign:
                    s.code_a = root(st.expr_a, &t);
                    if (p.locals[st.slot].type == ValueType::Int && t == ValueType::Real) s.flags |= WLP_IR_F_REAL_INTO_INT;
                    if (p.locals[st.slot].type == ValueType::Real && t == ValueType::Int) s.flags |= WLP_IR_F_INT_TO_REAL;
                    break;
                case StmtKind::Load:
                    s.arr = st.expr_b;
                    s.code_a = root(st.expr_a, &t);
                    if (t == ValueType::Real) s.flags |= WLP_IR_F_REAL_INDEX;
                    break;
                case StmtKind::Store:
                    s.code_a = root(st.expr_a, &t);
                    if (t == ValueType::Real) s.flags |= WLP_IR_F_REAL_INDEX;
                    s.code_b = root(st.expr_b, nullptr, false, true);
                    break;
                case StmtKind::If:
                case StmtKind::While: s.code_a = root(st.expr_a, nullptr, true); break;
                case StmtKind::Halt: break;
            }
            if (st.kind == StmtKind::If || st.kind == StmtKind::While) {
                const auto b1 = place(st.body1);
                const auto b2 = place(st.body2);
                s.b1_begin = b1.first;
                s.b1_end = b1.second;
                s.b2_begin = b2.first;
                s.b2_end = b2.second;
            }
            f.stmts[begin + k] = s;
        }
        return {begin, begin + static_cast<std::int32_t>(list.size())};
    }
};

Flat flatten(const KernelProgram& prog, const ParamEnv* env) {
    prog.finalize();
    if (prog.locals.size() > WLP_IR_MAX_LOCALS)
        throw DomainError("ir: the B200 interpreter holds at most " + std::to_string(WLP_IR_MAX_LOCALS) + " locals");
    Flat f;
    Compiler c{prog, f};
    const auto top = c.place(prog.body);
    f.top_begin = top.first;
    f.top_end = top.second;
    if (f.code.empty()) f.code.push_back(WLP_IR_OP_END);  // no expression at all (still a valid table)
    for (const LocalDecl& d : prog.locals) f.local_init.push_back(d.type == ValueType::Int ? 0 : static_cast<std::int64_t>(bits_of(0.0)));
    for (std::size_t k = 0; k < prog.params.size(); ++k) {
        const bool arr = prog.params[k].kind == ParamKind::Array;
        f.param_is_array.push_back(arr ? 1 : 0);
        std::int64_t bits = 0;
        if (env && !arr) {
            const Value& v = env->scalars[k];
            bits = v.is_int() ? v.i : static_cast<std::int64_t>(bits_of(v.r));
        }
        f.param_bits.push_back(bits);
    }
    return f;
}

wlp_ir_program view(const Flat& f) {
    wlp_ir_program v{};
    v.stmts = f.stmts.data();
    v.n_stmts = static_cast<std::int32_t>(f.stmts.size());
    v.top_begin = f.top_begin;
    v.top_end = f.top_end;
    v.code = f.code.data();
    v.n_code = static_cast<std::int32_t>(f.code.size());
    v.n_locals = static_cast<std::int32_t>(f.local_init.size());
    v.local_init = f.local_init.data();
    v.n_params = static_cast<std::int32_t>(f.param_bits.size());
    v.param_bits = f.param_bits.data();
    v.param_is_array = f.param_is_array.data();
    return v;
}

namespace {

SimReport report_of(const wlp_report& r) {
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
    return s;
}

}  // namespace

namespace {

SimReport simulate_impl(const KernelProgram& prog, const LaunchConfig& cfg, const DeviceProfile& prof,
                        GlobalMemory& memory, const std::map<std::string, Value>& scalars,
                        const std::vector<RngState>& streams, const SimOptions& opts,
                        const std::map<std::string, Value>& initial_locals) {
    validate_launch(cfg);
    prog.finalize();
    if (cfg.threads_per_block() > prof.maxThreadsPerBlock)
        throw PlanError("block of " + std::to_string(cfg.threads_per_block()) + " threads exceeds maxThreadsPerBlock " +
                        std::to_string(prof.maxThreadsPerBlock));
    ParamEnv env = bind_params(prog, scalars, memory);
    Flat f = flatten(prog, &env);
    for (const auto& [name, v] : initial_locals) {  // WarpState's initial_locals (warp_exec.cpp:79-86)
        const int slot = prog.local_slot(name);
        if (slot < 0) throw DomainError("initial value for undeclared local '" + name + "'");
        if (prog.locals[slot].type == ValueType::Int) {
            if (!v.is_int()) throw FaultError("assign: real value into int local '" + name + "'");
            f.local_init[slot] = v.i;
        } else {
            f.local_init[slot] = static_cast<std::int64_t>(bits_of(v.as_real()));
        }
    }
    const wlp_ir_program v = view(f);
    std::vector<double*> arrays(prog.params.size(), nullptr);
    std::vector<std::int64_t> lens(prog.params.size(), 0);
    for (std::size_t k = 0; k < prog.params.size(); ++k)
        if (env.arrays[k]) {
            arrays[k] = env.arrays[k]->data();
            lens[k] = static_cast<std::int64_t>(env.arrays[k]->size());
        }
    // streams needed: those of real threads only
    const std::int64_t threads = cfg.threads_per_block() * cfg.total_blocks();
    const std::int64_t n = std::min<std::int64_t>(static_cast<std::int64_t>(streams.size()), threads);
    std::vector<std::uint32_t> soa(static_cast<std::size_t>(3 * n));
    for (std::int64_t t = 0; t < n; ++t) {
        soa[t] = streams[t].s1;
        soa[n + t] = streams[t].s2;
        soa[2 * n + t] = streams[t].s3;
    }
    const wlp_launch_cfg c{cfg.blockDim.x, cfg.blockDim.y, cfg.blockDim.z, cfg.gridDim.x, cfg.gridDim.y, cfg.warpSize};
    wlp_report rep{};
    const int st = opts.irJit ? wlp_ir_jit_simulate(&v, &c, prof.maxThreadsPerBlock, arrays.data(), lens.data(), 0,
                                                    soa.data(), n, 0, opts.maxIssuesPerWarp, nullptr, &rep)
                              : wlp_ir_simulate(&v, &c, prof.maxThreadsPerBlock, arrays.data(), lens.data(), 0,
                                                soa.data(), n, 0, opts.maskStackDepth, opts.maxIssuesPerWarp, nullptr,
                                                &rep);
    if (st == WLP_EFAULT) {  // name the local of a typed-assign fault, as warp_exec.cpp does
        std::string msg = wlp_last_error();
        const std::string tag = "assign: real value into int local #";
        if (msg.rfind(tag, 0) == 0) {
            const std::size_t slot = std::stoul(msg.substr(tag.size()));
            if (slot < prog.locals.size()) msg = "assign: real value into int local '" + prog.locals[slot].name + "'";
        }
        throw FaultError(msg);
    }
    if (st != WLP_OK) raise_status(st);
    return report_of(rep);
}

}  // namespace

SimReport simulate(const KernelProgram& prog, const LaunchConfig& cfg, const DeviceProfile& prof, GlobalMemory& memory,
                   const std::map<std::string, Value>& scalars, const std::vector<RngState>& streams,
                   const SimOptions& opts) {
    return simulate_impl(prog, cfg, prof, memory, scalars, streams, opts, {});
}

SimReport simulate_single_thread(const KernelProgram& prog, GlobalMemory& memory,
                                 const std::map<std::string, Value>& scalars, RngState stream,
                                 const std::map<std::string, Value>& initial_locals, const SimOptions& opts) {
    LaunchConfig cfg;  // run_single_thread (warp_exec.cpp:308-316): one thread, warpSize 1
    cfg.blockDim = {1, 1, 1};
    cfg.gridDim = {1, 1};
    cfg.warpSize = 1;
    return simulate_impl(prog, cfg, DeviceProfile{}, memory, scalars, {stream}, opts, initial_locals);
}

ModelRun run_model_ir(ModelKind model, const ModelParams& p, ExecutionMode mode, const DeviceProfile& prof,
                      std::uint64_t master_seed, int tlp_block_size, const SimOptions& opts) {
    KernelBundle b = build_kernel(model, p, mode, prof, tlp_block_size);
    RngState master = rng_state_from_seed(master_seed);
    const std::vector<RngState> streams = random_spacing(master, static_cast<std::size_t>(p.replications));
    if (mode == ExecutionMode::Sequential) {
        // models.cpp:345-389: the outputs of the host loop (here the engine, bit-identical)
        // and the unit-cost report of ONE body execution (rid = 0, stream 0) times R
        ModelRun run = run_model(model, p, mode, prof, master_seed, tlp_block_size);
        GlobalMemory mem;
        for (const auto& [name, size] : b.arrays) mem.arrays[name].assign(static_cast<std::size_t>(size), 0.0);
        SimOptions one = opts;
        one.irJit = false;  // the accounting needs the interpreter
        const SimReport st = simulate_single_thread(b.program, mem, b.scalars, streams[0], {{"rid", Value::integer(0)}},
                                                    one);
        const auto R = static_cast<std::uint64_t>(p.replications);
        run.report = SimReport{};
        run.report.totalCycles = static_cast<std::int64_t>(st.issues * R);
        run.report.peakResidentWarps = 1;
        run.report.issues = st.issues * R;
        run.report.aluIssues = st.aluIssues * R;
        run.report.memReads = st.memReads * R;
        run.report.memWrites = st.memWrites * R;
        run.report.kernelMs = st.kernelMs;
        return run;
    }
    ModelRun run;
    run.cfg = b.cfg;
    run.mode = mode;
    run.warning = b.warning;
    GlobalMemory mem;
    for (const auto& [name, size] : b.arrays) mem.arrays[name].assign(static_cast<std::size_t>(size), 0.0);
    run.report = simulate(b.program, b.cfg, prof, mem, b.scalars, assign_lane_streams(mode, b.cfg, streams), opts);
    for (const std::string& name : b.outputs) run.outputs[name] = mem.arrays[name];
    run.primary = run.outputs[b.primary];
    return run;
}

}  // namespace warpsim

// ---- extern "C" surface for the Python mirror -------------------------------------------

namespace {

thread_local std::string g_ir_err;

int map_exception() {
    try {
        throw;
    } catch (const warpsim::ParseError& e) {
        g_ir_err = e.what();
        return WLP_EPARSE;
    } catch (const warpsim::DomainError& e) {
        g_ir_err = e.what();
        return WLP_EDOMAIN;
    } catch (const warpsim::PlanError& e) {
        g_ir_err = e.what();
        return WLP_EPLAN;
    } catch (const warpsim::FaultError& e) {
        g_ir_err = e.what();
        return WLP_EFAULT;
    } catch (const std::exception& e) {
        g_ir_err = e.what();
        return WLP_EINTERNAL;
    }
}

int copy_text(const std::string& s, char* out, int cap, int* need) {
    if (need) *need = static_cast<int>(s.size()) + 1;
    if (out && cap > 0) {
        const std::size_t n = std::min<std::size_t>(s.size(), static_cast<std::size_t>(cap - 1));
        std::memcpy(out, s.data(), n);
        out[n] = '\0';
    }
    return WLP_OK;
}

void to_report(const warpsim::SimReport& s, wlp_report* r) {
    if (!r) return;
    r->total_cycles = s.totalCycles;
    r->waves_executed = s.wavesExecuted;
    r->peak_resident_warps = s.peakResidentWarps;
    r->issues = s.issues;
    r->alu_issues = s.aluIssues;
    r->mem_reads = s.memReads;
    r->mem_writes = s.memWrites;
    r->divergence_events = s.divergenceEvents;
    r->kernel_ms = s.kernelMs;
}

}  // namespace

extern "C" {

const char* warpsim_ir_last_error(void) { return g_ir_err.c_str(); }

// parse_kernel then dump_kernel (the canonical text), or the error.
int warpsim_ir_canonical(const char* text, char* out, int cap, int* need) {
    try {
        return copy_text(warpsim::dump_kernel(warpsim::parse_kernel(text)), out, cap, need);
    } catch (...) {
        return map_exception();
    }
}

// The CUDA C++ the JIT generates for a kernel text (parse, flatten, translate).
int warpsim_ir_jit_source_text(const char* text, char* out, int cap, int* need) {
    try {
        const warpsim::KernelProgram prog = warpsim::parse_kernel(text);
        const warpsim::Flat f = warpsim::flatten(prog, nullptr);
        const wlp_ir_program v = warpsim::view(f);
        int n = 0;
        int st = wlp_ir_jit_source(&v, nullptr, 0, &n);
        if (st != WLP_OK) {
            g_ir_err = wlp_last_error();
            return st;
        }
        std::string src(static_cast<std::size_t>(n), '\0');
        st = wlp_ir_jit_source(&v, src.data(), n, nullptr);
        src.resize(std::strlen(src.c_str()));
        return copy_text(src, out, cap, need);
    } catch (...) {
        return map_exception();
    }
}

// dump_kernel of a model body (mode 0) or its Tlp (1) / Wlp (2) wrapping.
int warpsim_ir_model_text(int model, int mode, char* out, int cap, int* need) {
    try {
        if (model < 0 || model > 2 || mode < 0 || mode > 2) throw warpsim::DomainError("model / mode id");
        const warpsim::KernelProgram body = warpsim::build_model_body(static_cast<warpsim::ModelKind>(model));
        const warpsim::KernelProgram prog = mode == 0 ? body : mode == 1 ? warpsim::wrap_tlp(body) : warpsim::wrap_wlp(body);
        return copy_text(warpsim::dump_kernel(prog), out, cap, need);
    } catch (...) {
        return map_exception();
    }
}

// simulate (device.hpp) of a kernel given as text. Scalars by name (is_int selects ivals
// or rvals); arrays by name, updated in place; streams SoA[3*n_streams].
int warpsim_ir_simulate_text(const char* text, const wlp_launch_cfg* cfg, int max_threads_per_block, int n_scalars,
                             const char* const* names, const int* is_int, const int64_t* ivals, const double* rvals,
                             int n_arrays, const char* const* anames, double* const* arrays, const int64_t* alen,
                             const uint32_t* streams, int64_t n_streams, int mask_depth, int64_t max_issues,
                             int jit, wlp_report* report) {
    try {
        const warpsim::KernelProgram prog = warpsim::parse_kernel(text);
        warpsim::LaunchConfig lc;
        lc.blockDim = {cfg->block_x, cfg->block_y, cfg->block_z};
        lc.gridDim = {cfg->grid_x, cfg->grid_y};
        lc.warpSize = cfg->warp_size;
        std::map<std::string, warpsim::Value> scalars;
        for (int k = 0; k < n_scalars; ++k)
            scalars[names[k]] = is_int[k] ? warpsim::Value::integer(ivals[k]) : warpsim::Value::real(rvals[k]);
        warpsim::GlobalMemory mem;
        for (int k = 0; k < n_arrays; ++k) mem.arrays[anames[k]].assign(arrays[k], arrays[k] + alen[k]);
        std::vector<warpsim::RngState> st(static_cast<std::size_t>(n_streams));
        for (int64_t t = 0; t < n_streams; ++t) st[t] = warpsim::RngState{streams[t], streams[n_streams + t], streams[2 * n_streams + t]};
        warpsim::DeviceProfile prof;
        prof.maxThreadsPerBlock = max_threads_per_block;
        warpsim::SimOptions opts;
        opts.maskStackDepth = mask_depth;
        opts.maxIssuesPerWarp = max_issues;
        opts.irJit = jit != 0;
        const warpsim::SimReport rep = warpsim::simulate(prog, lc, prof, mem, scalars, st, opts);
        for (int k = 0; k < n_arrays; ++k) std::copy(mem.arrays[anames[k]].begin(), mem.arrays[anames[k]].end(), arrays[k]);
        to_report(rep, report);
        return WLP_OK;
    } catch (...) {
        return map_exception();
    }
}

// run_model through the IR path on the GPU interpreter (mode Tlp / Wlp).
int warpsim_ir_run_model(int model, const wlp_params* p, int mode, uint64_t seed, int tlp_block, double* out0,
                         double* out1, double* out2, wlp_report* report, char* warn, int warn_cap, int jit) {
    try {
        if (model < 0 || model > 2 || mode < 0 || mode > 2) throw warpsim::DomainError("model / mode id");
        warpsim::ModelParams mp;
        mp.replications = p->replications;
        mp.draws = p->draws;
        mp.clients = p->clients;
        mp.lambda = p->lambda;
        mp.mu = p->mu;
        mp.steps = p->steps;
        mp.chunks = p->chunks;
        warpsim::SimOptions opts;
        opts.irJit = jit != 0;
        const warpsim::ModelRun run =
            warpsim::run_model_ir(static_cast<warpsim::ModelKind>(model), mp, static_cast<warpsim::ExecutionMode>(mode),
                                  warpsim::DeviceProfile{}, seed, tlp_block, opts);
        const bool mm1 = model == 1;
        const auto put = [&](const char* name, double* dst) {
            if (dst) std::copy(run.outputs.at(name).begin(), run.outputs.at(name).end(), dst);
        };
        if (mm1) {
            put("outIdle", out0);
            put("outWait", out1);
            put("outSys", out2);
        } else {
            put("out", out0);
        }
        to_report(run.report, report);
        copy_text(run.warning.value_or(""), warn, warn_cap, nullptr);
        return WLP_OK;
    } catch (...) {
        return map_exception();
    }
}

}  // extern "C"
