// Launch interface of the kernel-IR interpreter (ir_interp.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/wlp_b200.h"

namespace wlp {

constexpr int kIrBlock = 128;

// First lane fault of a launch (codes: ir_fault_message in runtime.cu).
struct IrFault {
    int code;
    int pad;
    long long a, b, warp;
};

struct IrArgs {
    const wlp_ir_stmt* stmts;
    const int32_t* code;
    int32_t top_begin, top_end;
    int32_t n_locals;
    const int64_t* local_init;
    const int64_t* params;   // scalar param bits by slot
    double* const* arrays;   // device pointers by param slot
    const int64_t* alen;     // element counts by param slot
    const uint32_t* streams;  // SoA [3][n_streams]
    int64_t n_streams;
    int64_t bx, by, bz, gx, gy;  // LaunchConfig
    int64_t ws, tpb, wpb, total_warps;
    int mask_depth;
    int64_t max_issues;
    unsigned long long* counters;  // issues, alu, mem reads, mem writes, divergence events
    IrFault* fault;
};

int ir_blocks_per_sm();
cudaError_t launch_ir(const IrArgs& a, int grid, cudaStream_t st);

}  // namespace wlp
