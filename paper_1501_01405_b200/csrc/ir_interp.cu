// SIMT interpreter of the reference's kernel IR, running on the B200.
//
// The reference executes its IR kernels (kernel_ir.hpp:67-141) in a host simulator:
// simulate (device.cpp:140-226) runs every warp through WarpState::step
// (warp_exec.cpp:178-298), a lockstep interpreter with a divergence mask stack. Here each
// IR warp runs on one hardware warp, IR lane l on lane l, and the warp walks the
// statement tree with the same mask-stack rules: then-side before else-side, loop
// re-tests under the shrinking mask, permanent halts, reconvergence into the parent,
// one "issue" per statement or loop re-test. Lanes evaluate their own expressions
// (typed stack bytecode, include/wlp_b200.h); branch masks come from __ballot_sync, and
// conflicting stores resolve in ascending lane order with __match_any_sync. So values,
// memory and the issue / divergence / memory counters are the simulator's exactly, but
// the lanes are real hardware lanes: a divergent IF really serialises the warp.
//
// Arithmetic follows apply_bin / apply_un (kernel_ir.cpp:46-107) including every fault
// and the no-FMA rounding (--fmad=false); log is the bit-exact glibc port.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/wlp_b200.h"
#include "glibc_log.cuh"
#include "ir_interp.cuh"
#include "taus88.cuh"

namespace wlp {
namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kMaxFrames = 64;

enum FrameKind : int32_t { kTop = 0, kThen = 1, kElse = 2, kLoop = 3 };

struct Frame {
    int32_t begin, end, next, owner;
    uint32_t mask, else_mask;
    int32_t kind, else_pending;
};

__device__ __forceinline__ double as_f(int64_t v) { return __longlong_as_double(static_cast<long long>(v)); }
__device__ __forceinline__ int64_t as_i(double x) { return static_cast<int64_t>(__double_as_longlong(x)); }

// Lane context for expression evaluation.
struct Lane {
    Taus rng;
    int64_t tx, ty, tz;
    int fault;      // first fault code of this lane (0: none)
    int64_t fa, fb;  // fault details
};

__device__ __forceinline__ int64_t sreg_value(int r, const IrArgs& a, const Lane& L, int64_t bx, int64_t by) {
    switch (r) {
        case 0: return L.tx;
        case 1: return L.ty;
        case 2: return L.tz;
        case 3: return bx;
        case 4: return by;
        case 5: return a.bx;
        case 6: return a.by;
        case 7: return a.bz;
        case 8: return a.gx;
        case 9: return a.gy;
        default: return a.ws;
    }
}

__device__ __forceinline__ void lane_fault(Lane& L, int code, int64_t x = 0, int64_t y = 0) {
    if (!L.fault) {
        L.fault = code;
        L.fa = x;
        L.fb = y;
    }
}

// Evaluates the expression at code[pc]; returns its 64-bit pattern (type static).
__device__ int64_t eval(const IrArgs& a, int pc, int64_t* stk, const int64_t* loc, Lane& L, int64_t bx,
                        int64_t by) {
    const int32_t* code = a.code;
    int sp = 0;
    for (;;) {
        const int op = __ldg(code + pc++);
        switch (op) {
            case WLP_IR_OP_END:
                return stk[0];
            case WLP_IR_OP_CONST: {
                const uint32_t lo = static_cast<uint32_t>(__ldg(code + pc));
                const uint32_t hi = static_cast<uint32_t>(__ldg(code + pc + 1));
                pc += 2;
                stk[sp++] = static_cast<int64_t>((static_cast<uint64_t>(hi) << 32) | lo);
                break;
            }
            case WLP_IR_OP_LOCAL: stk[sp++] = loc[__ldg(code + pc++)]; break;
            case WLP_IR_OP_PARAM: stk[sp++] = __ldg(reinterpret_cast<const long long*>(a.params) + __ldg(code + pc++)); break;
            case WLP_IR_OP_SREG: stk[sp++] = sreg_value(__ldg(code + pc++), a, L, bx, by); break;
            case WLP_IR_OP_DRAW: stk[sp++] = as_i(u01(taus_next(L.rng))); break;
            case WLP_IR_OP_I2R_0: stk[sp - 1] = as_i(static_cast<double>(stk[sp - 1])); break;
            case WLP_IR_OP_I2R_1: stk[sp - 2] = as_i(static_cast<double>(stk[sp - 2])); break;
            case WLP_IR_OP_TRUTH_0: stk[sp - 1] = as_f(stk[sp - 1]) != 0.0 ? 1 : 0; break;
            case WLP_IR_OP_TRUTH_1: stk[sp - 2] = as_f(stk[sp - 2]) != 0.0 ? 1 : 0; break;
            case WLP_IR_OP_NEG_I: stk[sp - 1] = static_cast<int64_t>(0ull - static_cast<uint64_t>(stk[sp - 1])); break;
            case WLP_IR_OP_NEG_R: stk[sp - 1] = as_i(-as_f(stk[sp - 1])); break;
            case WLP_IR_OP_LOG: {
                const double x = as_f(stk[sp - 1]);
                if (!(x > 0.0)) lane_fault(L, 5);
                stk[sp - 1] = as_i(glibc_log_tab(x, kLogTabDev));
                break;
            }
            case WLP_IR_OP_FLOOR: {
                const double f = floor(as_f(stk[sp - 1]));
                if (!(f >= -9.2233720368547758e18 && f <= 9.2233720368547758e18)) lane_fault(L, 6);
                // x86-64 cvttsd2si gives INT64_MIN for 2^63, which the range check admits
                stk[sp - 1] = f >= 9.2233720368547758e18 ? INT64_MIN : static_cast<int64_t>(f);
                break;
            }
            default: {  // binary
                const int64_t y = stk[--sp];
                const int64_t x = stk[sp - 1];
                const double xr = as_f(x), yr = as_f(y);
                int64_t r = 0;
                switch (op) {
                    case WLP_IR_OP_ADD_I: r = static_cast<int64_t>(static_cast<uint64_t>(x) + static_cast<uint64_t>(y)); break;
                    case WLP_IR_OP_SUB_I: r = static_cast<int64_t>(static_cast<uint64_t>(x) - static_cast<uint64_t>(y)); break;
                    case WLP_IR_OP_MUL_I: r = static_cast<int64_t>(static_cast<uint64_t>(x) * static_cast<uint64_t>(y)); break;
                    case WLP_IR_OP_DIV_I:
                        if (y == 0) lane_fault(L, 1);
                        r = (y == 0 || (y == -1 && x == INT64_MIN)) ? (y == -1 ? x : 0) : x / y;
                        break;
                    case WLP_IR_OP_MOD_I:
                        if (y == 0) lane_fault(L, 3);
                        r = (y == 0 || y == -1) ? 0 : x % y;
                        break;
                    case WLP_IR_OP_ADD_R: r = as_i(__dadd_rn(xr, yr)); break;
                    case WLP_IR_OP_SUB_R: r = as_i(__dsub_rn(xr, yr)); break;
                    case WLP_IR_OP_MUL_R: r = as_i(__dmul_rn(xr, yr)); break;
                    case WLP_IR_OP_DIV_R:
                        if (yr == 0.0) lane_fault(L, 2);
                        r = as_i(__ddiv_rn(xr, yr));
                        break;
                    case WLP_IR_OP_MOD_R:
                        if (yr == 0.0) lane_fault(L, 4);
                        r = as_i(fmod(xr, yr));
                        break;
                    // comparisons exactly as numeric_lt / numeric_eq (kernel_ir.cpp:35-43):
                    // le = !(b < a), ge = !(a < b), so NaN compares le/ge true
                    case WLP_IR_OP_LT_I: r = x < y; break;
                    case WLP_IR_OP_LE_I: r = !(y < x); break;
                    case WLP_IR_OP_GT_I: r = y < x; break;
                    case WLP_IR_OP_GE_I: r = !(x < y); break;
                    case WLP_IR_OP_EQ_I: r = x == y; break;
                    case WLP_IR_OP_NE_I: r = x != y; break;
                    case WLP_IR_OP_LT_R: r = xr < yr; break;
                    case WLP_IR_OP_LE_R: r = !(yr < xr); break;
                    case WLP_IR_OP_GT_R: r = yr < xr; break;
                    case WLP_IR_OP_GE_R: r = !(xr < yr); break;
                    case WLP_IR_OP_EQ_R: r = xr == yr; break;
                    case WLP_IR_OP_NE_R: r = !(xr == yr); break;
                    case WLP_IR_OP_AND: r = (x != 0 && y != 0); break;
                    case WLP_IR_OP_OR: r = (x != 0 || y != 0); break;
                    default: lane_fault(L, 99); break;
                }
                stk[sp - 1] = r;
                break;
            }
        }
    }
}

__device__ __forceinline__ void count_issue(unsigned long long (&c)[5], int kind, bool event) {
    c[0] += 1;                   // issues
    if (kind == WLP_IR_LOAD)
        c[2] += 1;               // mem reads
    else if (kind == WLP_IR_STORE)
        c[3] += 1;               // mem writes
    else
        c[1] += 1;               // alu issues
    if (event) c[4] += 1;        // divergence events
}

// Runs one IR warp to completion (or to the first lane fault, recorded in *a.fault).
__device__ void run_ir_warp(const IrArgs& a, int64_t g, int lane, unsigned long long (&cnt)[5]) {
    const int64_t block_id = g / a.wpb;
    const int64_t w = g % a.wpb;
    const int64_t bx = block_id % a.gx, by = block_id / a.gx;
    Lane L;
    L.fault = 0;
    L.fa = L.fb = 0;
    const int64_t tib = w * a.ws + lane;  // thread id within the block
    const bool valid = lane < a.ws && tib < a.tpb;
    L.tx = L.ty = L.tz = 0;
    L.rng = Taus{kMin1, kMin2, kMin3};  // RngState{} (rng.hpp:11-17)
    if (valid) {
        int64_t rem = tib;
        L.tx = rem % a.bx;
        rem /= a.bx;
        L.ty = rem % a.by;
        L.tz = rem / a.by;
        const int64_t tid = tib + a.tpb * (bx + a.gx * by);
        if (tid < a.n_streams)
            L.rng = Taus{__ldg(a.streams + tid), __ldg(a.streams + a.n_streams + tid),
                         __ldg(a.streams + 2 * a.n_streams + tid)};
    }
    int64_t loc[WLP_IR_MAX_LOCALS];
    int64_t stk[WLP_IR_MAX_STACK];
    for (int s = 0; s < a.n_locals; ++s) loc[s] = __ldg(reinterpret_cast<const long long*>(a.local_init) + s);

    Frame fr[kMaxFrames];
    int depth = 0;
    const uint32_t entry = __ballot_sync(kFull, valid);
    if (entry == 0) return;
    fr[depth++] = Frame{a.top_begin, a.top_end, a.top_begin, -1, entry, 0u, kTop, 0};
    uint32_t halted = 0;
    int64_t issued = 0;
    const uint32_t me = 1u << lane;

    while (depth > 0) {
        Frame& f = fr[depth - 1];
        f.mask &= ~halted;
        if (f.mask == 0 || f.next >= f.end) {
            if (f.kind == kThen && f.else_pending) {
                f.else_pending = 0;
                const uint32_t em = f.else_mask & ~halted;
                if (em != 0) {
                    const wlp_ir_stmt* o = a.stmts + f.owner;
                    f.begin = __ldg(&o->b2_begin);
                    f.end = __ldg(&o->b2_end);
                    f.next = f.begin;
                    f.mask = em;
                    f.kind = kElse;
                    continue;
                }
            }
            if (f.kind == kLoop && f.mask != 0 && f.next >= f.end) {  // loop re-test
                const wlp_ir_stmt* ws = a.stmts + f.owner;
                const bool in = (f.mask & me) != 0;
                bool t = false;
                if (in) t = eval(a, __ldg(&ws->code_a), stk, loc, L, bx, by) != 0;
                const uint32_t again = __ballot_sync(kFull, in && t);
                const uint32_t leave = f.mask & ~again;
                count_issue(cnt, WLP_IR_WHILE, again != 0 && leave != 0 && __ldg(&ws->b1_end) > __ldg(&ws->b1_begin));
                if (again == 0) {
                    --depth;
                } else {
                    f.mask = again;
                    f.next = f.begin;
                }
            } else {
                --depth;
                continue;
            }
        } else {
            const int32_t si = f.next;
            const wlp_ir_stmt* sp = a.stmts + si;
            const int kind = __ldg(&sp->kind);
            const int flags = __ldg(&sp->flags);
            const bool in = (f.mask & me) != 0;
            f.next += 1;
            switch (kind) {
                case WLP_IR_ASSIGN: {
                    if (in) {
                        int64_t v = eval(a, __ldg(&sp->code_a), stk, loc, L, bx, by);
                        if (flags & WLP_IR_F_REAL_INTO_INT) lane_fault(L, 11, __ldg(&sp->slot));
                        if (flags & WLP_IR_F_INT_TO_REAL) v = as_i(static_cast<double>(v));
                        loc[__ldg(&sp->slot)] = v;
                    }
                    count_issue(cnt, kind, false);
                    break;
                }
                case WLP_IR_LOAD: {
                    if (in) {
                        const int64_t idx = eval(a, __ldg(&sp->code_a), stk, loc, L, bx, by);
                        const int arr = __ldg(&sp->arr);
                        const int64_t len = __ldg(reinterpret_cast<const long long*>(a.alen) + arr);
                        if (flags & WLP_IR_F_REAL_INDEX)
                            lane_fault(L, 7);
                        else if (idx < 0 || idx >= len)
                            lane_fault(L, 8, idx, len);
                        else
                            loc[__ldg(&sp->slot)] = as_i(a.arrays[arr][idx]);
                    }
                    count_issue(cnt, kind, false);
                    break;
                }
                case WLP_IR_STORE: {
                    const int arr = __ldg(&sp->slot);
                    int64_t idx = -1;
                    double val = 0.0;
                    bool ok = false;
                    if (in) {
                        idx = eval(a, __ldg(&sp->code_a), stk, loc, L, bx, by);
                        const int64_t len = __ldg(reinterpret_cast<const long long*>(a.alen) + arr);
                        if (flags & WLP_IR_F_REAL_INDEX) {
                            lane_fault(L, 9);
                        } else if (idx < 0 || idx >= len) {
                            lane_fault(L, 10, idx, len);
                        } else {
                            val = as_f(eval(a, __ldg(&sp->code_b), stk, loc, L, bx, by));
                            ok = L.fault == 0;
                        }
                    }
                    // the reference stores lane by lane in ascending order and throws at the
                    // first faulting lane (warp_exec.cpp:255-265): lanes above it never store
                    const uint32_t faulted = __ballot_sync(kFull, in && L.fault != 0);
                    if (faulted && lane >= __ffs(static_cast<int>(faulted)) - 1) ok = false;
                    // lanes storing to one element: the highest lane's value lands last
                    // (the reference stores in ascending lane order)
                    const unsigned long long key = ok ? static_cast<unsigned long long>(idx)
                                                      : (0xFFFFFFFF00000000ull | static_cast<unsigned>(lane));
                    const unsigned grp = __match_any_sync(kFull, key);
                    if (ok && lane == 31 - __clz(static_cast<int>(grp))) a.arrays[arr][idx] = val;
                    __syncwarp();
                    count_issue(cnt, kind, false);
                    break;
                }
                case WLP_IR_HALT:
                    halted |= f.mask;
                    count_issue(cnt, kind, false);
                    break;
                case WLP_IR_IF: {
                    bool t = false;
                    if (in) t = eval(a, __ldg(&sp->code_a), stk, loc, L, bx, by) != 0;
                    const uint32_t taken = __ballot_sync(kFull, in && t);
                    const uint32_t other = f.mask & ~taken;
                    const int b1b = __ldg(&sp->b1_begin), b1e = __ldg(&sp->b1_end);
                    const int b2b = __ldg(&sp->b2_begin), b2e = __ldg(&sp->b2_end);
                    const bool then_work = b1e > b1b, else_work = b2e > b2b;
                    count_issue(cnt, kind, taken != 0 && other != 0 && then_work && else_work);
                    Frame nf;
                    bool push = false;
                    if (taken != 0 && then_work) {
                        nf = Frame{b1b, b1e, b1b, si, taken, other, kThen, (other != 0 && else_work) ? 1 : 0};
                        push = true;
                    } else if (other != 0 && else_work) {
                        nf = Frame{b2b, b2e, b2b, si, other, 0u, kElse, 0};
                        push = true;
                    }
                    if (push) {
                        if (depth >= a.mask_depth) {
                            lane_fault(L, 12, a.mask_depth);
                        } else {
                            fr[depth++] = nf;
                        }
                    }
                    break;
                }
                default: {  // WHILE
                    bool t = false;
                    if (in) t = eval(a, __ldg(&sp->code_a), stk, loc, L, bx, by) != 0;
                    const uint32_t enter = __ballot_sync(kFull, in && t);
                    const uint32_t skip = f.mask & ~enter;
                    const int b1b = __ldg(&sp->b1_begin), b1e = __ldg(&sp->b1_end);
                    count_issue(cnt, kind, enter != 0 && skip != 0 && b1e > b1b);
                    if (enter != 0 && b1e > b1b) {
                        if (depth >= a.mask_depth)
                            lane_fault(L, 12, a.mask_depth);
                        else
                            fr[depth++] = Frame{b1b, b1e, b1b, si, enter, 0u, kLoop, 0};
                    }
                    break;
                }
            }
        }
        // faults: the lowest faulting lane's record wins (the reference stops at the
        // first lane, in ascending order, that faults)
        const uint32_t bad = __ballot_sync(kFull, L.fault != 0);
        if (bad) {
            const int first = __ffs(static_cast<int>(bad)) - 1;
            if (lane == first && atomicCAS(&a.fault->code, 0, L.fault) == 0) {
                a.fault->a = L.fa;
                a.fault->b = L.fb;
                a.fault->warp = g;
            }
            return;
        }
        if (++issued >= a.max_issues) {
            if (lane == 0 && atomicCAS(&a.fault->code, 0, 13) == 0) {
                a.fault->a = a.max_issues;
                a.fault->warp = g;
            }
            return;
        }
        if ((issued & 255) == 0 && *reinterpret_cast<volatile int*>(&a.fault->code) != 0) return;  // another warp faulted
    }
}

__global__ void __launch_bounds__(kIrBlock) k_ir(IrArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t hw_warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t n_hw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    unsigned long long cnt[5] = {0, 0, 0, 0, 0};
    for (int64_t g = hw_warp; g < a.total_warps; g += n_hw) {
        if (*reinterpret_cast<volatile int*>(&a.fault->code) != 0) break;
        run_ir_warp(a, g, lane, cnt);
    }
    if (lane == 0) {
        for (int k = 0; k < 5; ++k)
            if (cnt[k]) atomicAdd(a.counters + k, cnt[k]);
    }
}

}  // namespace

int ir_blocks_per_sm() {
    int nb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ir, kIrBlock, 0);
    return nb < 1 ? 1 : nb;
}

cudaError_t launch_ir(const IrArgs& a, int grid, cudaStream_t st) {
    k_ir<<<grid, kIrBlock, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace wlp
