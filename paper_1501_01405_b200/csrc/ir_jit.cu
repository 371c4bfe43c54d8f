// Kernel IR → CUDA C++ → NVRTC → sm_100a: user-defined models at native speed
// (beside the interpreter in ir_interp.cu).
//
// The flattened program (include/wlp_b200.h: statement ranges + typed stack bytecode) is
// translated into one __global__ function. Each IR statement becomes structured C++:
// locals are registers, expressions become typed temporaries in the bytecode's
// evaluation order (so draws are consumed as in the reference), IF / WHILE are real
// branches and loops (the hardware serialises divergent paths), HALT ends the IR thread,
// and every fault of apply_bin / apply_un (kernel_ir.cpp:46-107) and of loads / stores is
// checked. Stores resolve same-element conflicts in ascending lane order
// (__match_any_sync) as the reference does. IR warps map onto hardware warps as in the
// interpreter, and special registers have the same values.
//
// What the JIT does not give: the simulator's issue / divergence counters. Those need
// the reference's lockstep mask semantics, which the interpreter implements. Kernels
// whose lanes communicate through memory across the two sides of a divergent branch
// may also order differently.
//
// NVRTC is loaded with dlopen on first use, so the library works without it (JIT calls
// then fail with WLP_ECUDA). Compiled kernels are cached by source text.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/wlp_b200.h"
#include "jit_headers.inc"

namespace wlp {
namespace {

// ---- NVRTC, loaded lazily -------------------------------------------------------------

typedef int nvrtcResult_;
typedef struct _nvrtcProgram* nvrtcProgram_;
struct Nvrtc {
    nvrtcResult_ (*create)(nvrtcProgram_*, const char*, const char*, int, const char* const*, const char* const*);
    nvrtcResult_ (*compile)(nvrtcProgram_, int, const char* const*);
    nvrtcResult_ (*log_size)(nvrtcProgram_, size_t*);
    nvrtcResult_ (*log)(nvrtcProgram_, char*);
    nvrtcResult_ (*cubin_size)(nvrtcProgram_, size_t*);
    nvrtcResult_ (*cubin)(nvrtcProgram_, char*);
    nvrtcResult_ (*destroy)(nvrtcProgram_*);
    bool ok = false;
    std::string why;
};

const Nvrtc& nvrtc() {
    static const Nvrtc n = [] {
        Nvrtc r{};
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            r.why = std::string("NVRTC not found: ") + dlerror();
            return r;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
        r.create = reinterpret_cast<decltype(r.create)>(sym("nvrtcCreateProgram"));
        r.compile = reinterpret_cast<decltype(r.compile)>(sym("nvrtcCompileProgram"));
        r.log_size = reinterpret_cast<decltype(r.log_size)>(sym("nvrtcGetProgramLogSize"));
        r.log = reinterpret_cast<decltype(r.log)>(sym("nvrtcGetProgramLog"));
        r.cubin_size = reinterpret_cast<decltype(r.cubin_size)>(sym("nvrtcGetCUBINSize"));
        r.cubin = reinterpret_cast<decltype(r.cubin)>(sym("nvrtcGetCUBIN"));
        r.destroy = reinterpret_cast<decltype(r.destroy)>(sym("nvrtcDestroyProgram"));
        r.ok = r.create && r.compile && r.log_size && r.log && r.cubin_size && r.cubin && r.destroy;
        if (!r.ok) r.why = "NVRTC lacks an expected entry point";
        return r;
    }();
    return n;
}

// ---- code generation -------------------------------------------------------------------

const char* const kPrelude = R"SRC(
#include "taus88.cuh"
#include "glibc_log.cuh"
struct IrFault { int code; int pad; long long a, b, warp; };
__device__ __forceinline__ double R_(long long v) { return __longlong_as_double(v); }
__device__ __forceinline__ long long B_(double x) { return __double_as_longlong(x); }
#define FAULT(c, x, y) do { if (atomicCAS(&fault->code, 0, (c)) == 0) { fault->a = (x); fault->b = (y); \
    fault->warp = g; } goto done; } while (0)
)SRC";

struct Gen {
    const wlp_ir_program& p;
    std::string out;
    int tmp = 0;

    std::string t() { return "t" + std::to_string(tmp++); }
    static std::string hex64(uint64_t v) {
        char b[32];
        std::snprintf(b, sizeof b, "0x%016llxULL", static_cast<unsigned long long>(v));
        return b;
    }

    // Emits the expression at code[pc]; returns the temporary holding its bits.
    std::string expr(int pc, const std::string& ind) {
        std::vector<std::string> st;
        auto emit = [&](const std::string& rhs) {
            const std::string v = t();
            out += ind + "const long long " + v + " = " + rhs + ";\n";
            st.push_back(v);
        };
        for (;;) {
            const int op = p.code[pc++];
            if (op == WLP_IR_OP_END) return st.back();
            switch (op) {
                case WLP_IR_OP_CONST: {
                    const uint64_t v = static_cast<uint32_t>(p.code[pc]) |
                                       (static_cast<uint64_t>(static_cast<uint32_t>(p.code[pc + 1])) << 32);
                    pc += 2;
                    emit("(long long)" + hex64(v));
                    break;
                }
                case WLP_IR_OP_LOCAL: emit("L" + std::to_string(p.code[pc++])); break;
                case WLP_IR_OP_PARAM: emit("__ldg(P + " + std::to_string(p.code[pc++]) + ")"); break;
                case WLP_IR_OP_SREG: {
                    static const char* names[] = {"tx", "ty", "tz", "bidx", "bidy", "bx", "by", "bz", "gx", "gy", "ws"};
                    emit(std::string(names[p.code[pc++]]));
                    break;
                }
                case WLP_IR_OP_DRAW: emit("B_(wlp::u01(wlp::taus_next(rng)))"); break;
                case WLP_IR_OP_I2R_0: {
                    const std::string a = st.back();
                    st.pop_back();
                    emit("B_((double)" + a + ")");
                    break;
                }
                case WLP_IR_OP_I2R_1: {
                    const std::string b = st.back();
                    st.pop_back();
                    const std::string a = st.back();
                    st.pop_back();
                    emit("B_((double)" + a + ")");
                    st.push_back(b);
                    break;
                }
                case WLP_IR_OP_TRUTH_0: {
                    const std::string a = st.back();
                    st.pop_back();
                    emit("(R_(" + a + ") != 0.0 ? 1LL : 0LL)");
                    break;
                }
                case WLP_IR_OP_TRUTH_1: {
                    const std::string b = st.back();
                    st.pop_back();
                    const std::string a = st.back();
                    st.pop_back();
                    emit("(R_(" + a + ") != 0.0 ? 1LL : 0LL)");
                    st.push_back(b);
                    break;
                }
                case WLP_IR_OP_NEG_I: {
                    const std::string a = st.back();
                    st.pop_back();
                    emit("(long long)(0ULL - (unsigned long long)" + a + ")");
                    break;
                }
                case WLP_IR_OP_NEG_R: {
                    const std::string a = st.back();
                    st.pop_back();
                    emit("B_(-R_(" + a + "))");
                    break;
                }
                case WLP_IR_OP_LOG: {
                    const std::string a = st.back();
                    st.pop_back();
                    out += ind + "if (!(R_(" + a + ") > 0.0)) FAULT(5, 0, 0);\n";
                    emit("B_(wlp::glibc_log_tab(R_(" + a + "), wlp::kLogTabDev))");
                    break;
                }
                case WLP_IR_OP_FLOOR: {
                    const std::string a = st.back();
                    st.pop_back();
                    const std::string f = t();
                    out += ind + "const double " + f + " = floor(R_(" + a + "));\n";
                    out += ind + "if (!(" + f + " >= -9.2233720368547758e18 && " + f +
                           " <= 9.2233720368547758e18)) FAULT(6, 0, 0);\n";
                    emit("(" + f + " >= 9.2233720368547758e18 ? (long long)0x8000000000000000ULL : (long long)" + f +
                         ")");
                    break;
                }
                default: {
                    const std::string b = st.back();
                    st.pop_back();
                    const std::string a = st.back();
                    st.pop_back();
                    const std::string ua = "(unsigned long long)" + a, ub = "(unsigned long long)" + b;
                    const std::string ra = "R_(" + a + ")", rb = "R_(" + b + ")";
                    switch (op) {
                        case WLP_IR_OP_ADD_I: emit("(long long)(" + ua + " + " + ub + ")"); break;
                        case WLP_IR_OP_SUB_I: emit("(long long)(" + ua + " - " + ub + ")"); break;
                        case WLP_IR_OP_MUL_I: emit("(long long)(" + ua + " * " + ub + ")"); break;
                        case WLP_IR_OP_DIV_I:
                            out += ind + "if (" + b + " == 0) FAULT(1, 0, 0);\n";
                            emit("(" + b + " == -1 ? (long long)(0ULL - " + ua + ") : " + a + " / " + b + ")");
                            break;
                        case WLP_IR_OP_MOD_I:
                            out += ind + "if (" + b + " == 0) FAULT(3, 0, 0);\n";
                            emit("(" + b + " == -1 ? 0LL : " + a + " % " + b + ")");
                            break;
                        case WLP_IR_OP_ADD_R: emit("B_(__dadd_rn(" + ra + ", " + rb + "))"); break;
                        case WLP_IR_OP_SUB_R: emit("B_(__dsub_rn(" + ra + ", " + rb + "))"); break;
                        case WLP_IR_OP_MUL_R: emit("B_(__dmul_rn(" + ra + ", " + rb + "))"); break;
                        case WLP_IR_OP_DIV_R:
                            out += ind + "if (" + rb + " == 0.0) FAULT(2, 0, 0);\n";
                            emit("B_(__ddiv_rn(" + ra + ", " + rb + "))");
                            break;
                        case WLP_IR_OP_MOD_R:
                            out += ind + "if (" + rb + " == 0.0) FAULT(4, 0, 0);\n";
                            emit("B_(fmod(" + ra + ", " + rb + "))");
                            break;
                        case WLP_IR_OP_LT_I: emit("(long long)(" + a + " < " + b + ")"); break;
                        case WLP_IR_OP_LE_I: emit("(long long)!(" + b + " < " + a + ")"); break;
                        case WLP_IR_OP_GT_I: emit("(long long)(" + b + " < " + a + ")"); break;
                        case WLP_IR_OP_GE_I: emit("(long long)!(" + a + " < " + b + ")"); break;
                        case WLP_IR_OP_EQ_I: emit("(long long)(" + a + " == " + b + ")"); break;
                        case WLP_IR_OP_NE_I: emit("(long long)(" + a + " != " + b + ")"); break;
                        case WLP_IR_OP_LT_R: emit("(long long)(" + ra + " < " + rb + ")"); break;
                        case WLP_IR_OP_LE_R: emit("(long long)!(" + rb + " < " + ra + ")"); break;
                        case WLP_IR_OP_GT_R: emit("(long long)(" + rb + " < " + ra + ")"); break;
                        case WLP_IR_OP_GE_R: emit("(long long)!(" + ra + " < " + rb + ")"); break;
                        case WLP_IR_OP_EQ_R: emit("(long long)(" + ra + " == " + rb + ")"); break;
                        case WLP_IR_OP_NE_R: emit("(long long)!(" + ra + " == " + rb + ")"); break;
                        case WLP_IR_OP_AND: emit("(long long)(" + a + " != 0 && " + b + " != 0)"); break;
                        case WLP_IR_OP_OR: emit("(long long)(" + a + " != 0 || " + b + " != 0)"); break;
                        default: emit("0LL"); break;
                    }
                    break;
                }
            }
        }
    }

    void list(int begin, int end, const std::string& ind) {
        for (int i = begin; i < end; ++i) stmt(p.stmts[i], ind);
    }

    void stmt(const wlp_ir_stmt& s, const std::string& ind) {
        const std::string in2 = ind + "  ";
        out += ind + "{\n";
        switch (s.kind) {
            case WLP_IR_ASSIGN: {
                const std::string v = expr(s.code_a, in2);
                if (s.flags & WLP_IR_F_REAL_INTO_INT) out += in2 + "FAULT(11, " + std::to_string(s.slot) + ", 0);\n";
                out += in2 + "L" + std::to_string(s.slot) + " = " +
                       ((s.flags & WLP_IR_F_INT_TO_REAL) ? "B_((double)" + v + ")" : v) + ";\n";
                break;
            }
            case WLP_IR_LOAD: {
                const std::string i = expr(s.code_a, in2);
                const std::string len = "__ldg(AL + " + std::to_string(s.arr) + ")";
                if (s.flags & WLP_IR_F_REAL_INDEX) out += in2 + "FAULT(7, 0, 0);\n";
                out += in2 + "if (" + i + " < 0 || " + i + " >= " + len + ") FAULT(8, " + i + ", " + len + ");\n";
                out += in2 + "L" + std::to_string(s.slot) + " = B_(A[" + std::to_string(s.arr) + "][" + i + "]);\n";
                break;
            }
            case WLP_IR_STORE: {
                const std::string i = expr(s.code_a, in2);
                const std::string len = "__ldg(AL + " + std::to_string(s.slot) + ")";
                if (s.flags & WLP_IR_F_REAL_INDEX) out += in2 + "FAULT(9, 0, 0);\n";
                out += in2 + "if (" + i + " < 0 || " + i + " >= " + len + ") FAULT(10, " + i + ", " + len + ");\n";
                const std::string v = expr(s.code_b, in2);
                out += in2 + "{ const unsigned m_ = __activemask();\n";
                out += in2 + "  const unsigned grp_ = __match_any_sync(m_, (unsigned long long)" + i + ");\n";
                out += in2 + "  if (lane == 31 - __clz((int)grp_)) A[" + std::to_string(s.slot) + "][" + i + "] = R_(" + v +
                       ");\n";
                out += in2 + "  __syncwarp(m_); }\n";
                break;
            }
            case WLP_IR_IF: {
                const std::string c = expr(s.code_a, in2);
                out += in2 + "if (" + c + " != 0) {\n";
                list(s.b1_begin, s.b1_end, in2 + "  ");
                out += in2 + "} else {\n";
                list(s.b2_begin, s.b2_end, in2 + "  ");
                out += in2 + "}\n";
                break;
            }
            case WLP_IR_WHILE: {
                out += in2 + "for (;;) {\n";
                const std::string c = expr(s.code_a, in2 + "  ");
                out += in2 + "  if (" + c + " == 0) break;\n";
                out += in2 + "  if (++iters > max_iters) FAULT(13, max_iters, 0);\n";
                list(s.b1_begin, s.b1_end, in2 + "  ");
                out += in2 + "}\n";
                break;
            }
            default:  // HALT
                out += in2 + "goto done;\n";
                break;
        }
        out += ind + "}\n";
    }

    std::string kernel() {
        out = kPrelude;
        out += "extern \"C\" __global__ void __launch_bounds__(128) wlp_ir_jit(\n"
               "    const long long* __restrict__ P, double* const* __restrict__ A, const long long* __restrict__ AL,\n"
               "    const unsigned* __restrict__ S, long long nS, long long bx, long long by, long long bz,\n"
               "    long long gx, long long gy, long long ws, long long tpb, long long wpb, long long total_warps,\n"
               "    long long max_iters, IrFault* fault) {\n"
               "  const int lane = threadIdx.x & 31;\n"
               "  const long long hw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;\n"
               "  const long long nhw = ((long long)gridDim.x * blockDim.x) >> 5;\n"
               "  for (long long g = hw; g < total_warps; g += nhw) {\n"
               "    if (*(volatile int*)&fault->code) return;\n"
               "    const long long blk = g / wpb, w = g % wpb, bidx = blk % gx, bidy = blk / gx;\n"
               "    const long long tib = w * ws + lane;\n"
               "    if (lane >= ws || tib >= tpb) continue;\n"
               "    long long rem = tib;\n"
               "    const long long tx = rem % bx; rem /= bx;\n"
               "    const long long ty = rem % by, tz = rem / by;\n"
               "    const long long tid = tib + tpb * (bidx + gx * bidy);\n"
               "    wlp::Taus rng{wlp::kMin1, wlp::kMin2, wlp::kMin3};\n"
               "    if (tid < nS) rng = wlp::Taus{__ldg(S + tid), __ldg(S + nS + tid), __ldg(S + 2 * nS + tid)};\n"
               "    long long iters = 0;\n";
        for (int i = 0; i < p.n_locals; ++i)
            out += "    long long L" + std::to_string(i) + " = (long long)" + hex64(static_cast<uint64_t>(p.local_init[i])) +
                   ";\n";
        out += "    (void)tx; (void)ty; (void)tz; (void)iters;\n";
        list(p.top_begin, p.top_end, "    ");
        out += "  done:;\n  }\n}\n";
        return out;
    }
};

// ---- compile cache -----------------------------------------------------------------------

struct Compiled {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t kernel = nullptr;
};

std::mutex g_jit_mu;
std::map<std::pair<int, std::string>, Compiled> g_cache;  // (device, source)

int compile(const std::string& src, Compiled& out, std::string& err) {
    const Nvrtc& n = nvrtc();
    if (!n.ok) {
        err = n.why;
        return WLP_ECUDA;
    }
    const char* names[wlp_jit::kNumHeaders + 1];
    const char* srcs[wlp_jit::kNumHeaders + 1];
    for (int i = 0; i < wlp_jit::kNumHeaders; ++i) {
        names[i] = wlp_jit::kHeaderNames[i];
        srcs[i] = wlp_jit::kHeaderSrcs[i];
    }
    names[wlp_jit::kNumHeaders] = "stdint.h";  // NVRTC ships no C library headers
    srcs[wlp_jit::kNumHeaders] =
        "#pragma once\ntypedef unsigned int uint32_t; typedef int int32_t; typedef unsigned long long uint64_t;\n"
        "typedef long long int64_t;\n";
    nvrtcProgram_ prog = nullptr;
    if (n.create(&prog, src.c_str(), "wlp_ir_jit.cu", wlp_jit::kNumHeaders + 1, srcs, names) != 0) {
        err = "nvrtcCreateProgram failed";
        return WLP_ECUDA;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--std=c++17", "-default-device"};
    const int rc = n.compile(prog, 4, opts);
    if (rc != 0) {
        size_t ls = 0;
        n.log_size(prog, &ls);
        std::string log(ls, '\0');
        n.log(prog, log.data());
        n.destroy(&prog);
        err = "NVRTC compile failed: " + log;
        return WLP_EINTERNAL;
    }
    size_t cs = 0;
    n.cubin_size(prog, &cs);
    std::vector<char> cubin(cs);
    n.cubin(prog, cubin.data());
    n.destroy(&prog);
    cudaError_t e = cudaLibraryLoadData(&out.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (e == cudaSuccess) e = cudaLibraryGetKernel(&out.kernel, out.lib, "wlp_ir_jit");
    if (e != cudaSuccess) {
        err = std::string("loading the JIT cubin: ") + cudaGetErrorString(e);
        return WLP_ECUDA;
    }
    return WLP_OK;
}

}  // namespace

std::string ir_jit_source(const wlp_ir_program& p) { return Gen{p}.kernel(); }

int ir_jit_kernel(const wlp_ir_program& p, int device, void** kernel, std::string& err) {
    const std::string src = ir_jit_source(p);
    std::lock_guard<std::mutex> g(g_jit_mu);
    auto it = g_cache.find({device, src});
    if (it == g_cache.end()) {
        Compiled c;
        const int rc = compile(src, c, err);
        if (rc != WLP_OK) return rc;
        it = g_cache.emplace(std::make_pair(device, src), c).first;
    }
    *kernel = reinterpret_cast<void*>(it->second.kernel);
    return WLP_OK;
}

}  // namespace wlp
