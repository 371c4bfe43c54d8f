/*
 * wlp_b200.h — C ABI of the B200 Multiple-Replications-in-Parallel engine
 * (Warp-Level Parallelism, arXiv 1501.01405), libwlp_b200.so.
 *
 * Plain C: pointers, sizes, status codes; no C++ or torch types. Every entry point
 * names the reference interface it replaces (paths relative to /root/reference/proj).
 * The C++ drop-in (include/warpsim_b200.hpp) and the Python mirror
 * (paper_1501_01405_b200/__init__.py) are thin layers over these calls.
 *
 * Execution: all model work runs in hand-written sm_100a kernels on the calling
 * thread's current CUDA device (cudaSetDevice), on `stream` (a cudaStream_t, or NULL for
 * the legacy default stream). There is no CPU fallback: without a usable GPU every
 * compute call returns WLP_ECUDA.
 *
 * Buffers are caller-owned. `*_on_device` = 1 means the pointer is device memory on the
 * current device and the call is asynchronous on `stream` unless stated otherwise;
 * 0 means host memory (pageable or pinned) and the call returns with results written.
 * The library owns its device scratch (released by wlp_shutdown).
 *
 * Thread safety: calls are serialised per device by an internal lock.
 */
#ifndef WLP_B200_H
#define WLP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the C++ layer rethrows them as the reference's exception types
 * (include/warpsim/error.hpp:8-36). */
#define WLP_OK 0
#define WLP_EDOMAIN 1   /* DomainError: invalid params (models.cpp:26-44, rng.cpp:58-59)   */
#define WLP_EPLAN 2     /* PlanError: launch planning (wlp.cpp:71-105)                     */
#define WLP_EFAULT 3    /* FaultError: a device lane fault                                 */
#define WLP_ESPACING 4  /* Error: random_spacing found no distinct seed (rng.cpp:81-82)    */
#define WLP_ECUDA 5     /* Error: CUDA runtime failure / no device                         */
#define WLP_EPARSE 6    /* ParseError: kernel text (kernel_text.hpp; libwarpsim_b200.so)    */
#define WLP_EINTERNAL 7 /* Error: anything else                                            */

/* ModelKind (models.hpp:18) and ExecutionMode (wlp.hpp:16). */
#define WLP_MODEL_PI 0
#define WLP_MODEL_MM1 1
#define WLP_MODEL_WALK 2
#define WLP_MODE_SEQUENTIAL 0
#define WLP_MODE_TLP 1
#define WLP_MODE_WLP 2

/* ModelParams (models.hpp:23-31); defaults 1, 1000, 1000, 0.5, 1.0, 1000, 30. */
typedef struct wlp_params {
    int64_t replications;
    int64_t draws;   /* pi: points per replication   */
    int64_t clients; /* mm1                          */
    double lambda;   /* mm1 arrival rate             */
    double mu;       /* mm1 service rate             */
    int64_t steps;   /* walk                         */
    int64_t chunks;  /* walk                         */
} wlp_params;

/* LaunchConfig (kernel_ir.hpp:35-45), 1-D/2-D as the reference uses it. */
typedef struct wlp_launch_cfg {
    int64_t block_x, block_y, block_z;
    int64_t grid_x, grid_y;
    int32_t warp_size;
} wlp_launch_cfg;

/* SimReport (device.hpp:62-71). On the GPU: total_cycles = measured kernel time in SM
 * cycles at the device's clock, waves_executed = ceil(blocks / resident capacity),
 * peak_resident_warps = min(launch warps, resident capacity); the simulator-only
 * counters (issues, memReads, ...) are 0 — ncu measures those. */
typedef struct wlp_report {
    int64_t total_cycles;
    int64_t waves_executed;
    int64_t peak_resident_warps;
    uint64_t issues, alu_issues, mem_reads, mem_writes, divergence_events;
    double kernel_ms; /* model-kernel time from CUDA events (0 when not timed) */
    uint64_t warp_splits; /* instrumented runs: every warp split of the kernel (see below) */
} wlp_report;

/* ConfidenceInterval (models.hpp:118-127). */
typedef struct wlp_ci {
    double mean;
    double half_width;
    double level;
    int64_t n;
    int32_t warn_small_sample; /* n < 30 */
} wlp_ci;

/* Sufficient statistics of one output array over a replication range: count, sum as an
 * unevaluated double-double (hi + lo), and, after the second pass, the centred sum of
 * squares about `center` (hi + lo). Shards combine these exactly (wlp_stats_merge). */
typedef struct wlp_stats {
    int64_t n;
    double sum_hi, sum_lo;
    double center;
    double ss_hi, ss_lo;
} wlp_stats;

/* A seeding candidate whose stream key could collide with another's (some component
 * below twice its minimum). `index` is the global candidate
 * index (candidate i = remap(master draws 3i+1..3i+3)). */
typedef struct wlp_special {
    int64_t index;
    uint32_t s1, s2, s3, pad;
} wlp_special;

/* ---- host-only utilities (no GPU needed) -------------------------------------- */

const char* wlp_last_error(void);   /* message of the last failing call on this thread */
int wlp_version(void);              /* ABI version (1)                                  */

/* Hardware counters for the SimReport of later calls on this thread (enable != 0): the
 * replication kernels run instrumented variants and wlp_report gets
 *   divergence_events — warp-level splits of the model's data-dependent `if`s, counted
 *                       with the reference's event definition (warp_exec.cpp:272-284):
 *                       the TLP walk's 3 nested direction ifs, the TLP mm1 `t < 0`;
 *                       WLP has none (no lane runs a model branch against another);
 *   mem_reads / mem_writes — global load / store warp-instructions of the model kernel
 *                       (the analogue of the paper's Table 1 counts; atomics excluded);
 *   warp_splits       — every warp split the kernel itself executes, by the same event
 *                       definition: the model's ifs above plus the implementation's
 *                       lane-divergent loops (WLP: lane chunk tails of unequal length,
 *                       the warp's near-one log list; TLP mm1: its near-one list);
 *   total_cycles      — the kernel's makespan in SM cycles from clock64 (per SM, latest
 *                       warp end minus earliest warp start, max over SMs); uninstrumented
 *                       runs report kernel_ms x the SM clock instead.
 * Costs some speed; off by default. */
int wlp_set_hw_counters(int enable);

/* Tuning / test hook for later calls on this thread: which WLP kernel runs a model.
 * 0 = automatic (default); 1 = lane jumps (pi / walk: each lane jumps its stream to its
 * chunk; mm1: segment chaining by fixed-point rounds); 2 = warp pipeline (replications
 * move lane to lane, each lane runs its segment in order from the state its neighbour
 * hands over; rotating chunk lengths, fill and drain covered by wrap replications); 3 = walk: bitsliced warp pipeline (each pipeline
 * slot carries 32 replications as bit planes); 4 = walk: bitsliced lane chunks (a warp per
 * group of 32 replications, each lane jumps all 32 to its chunk). The walk picks 3 / 4 /
 * per-replication automatically by R; pi and mm1 treat 3 and 4 as 0. Outputs are
 * identical; only speed differs. */
int wlp_set_wlp_variant(int variant);

/* Tuning / test hook for later calls on this thread: lanes per replication S of the warp
 * pipelines (pi / walk per replication: 2, 4, 8, 16 or 32; walk bitsliced: lanes per
 * group of 32 replications, 4 to 32; mm1: 2 to 32). 32 = the whole warp is one pipeline;
 * 16 .. 2 = 32/S pipelines side by side in the warp, every replication still passing
 * through lanes of one warp only, split into S chunks (longer steps for the same
 * hand-over work). 0 = automatic: S = 2 when the run fills the grid with two-lane
 * pipelines (pi / walk with their wrap replications; mm1 >= 4 replications a pipeline);
 * else pi / walk the most lanes that give every lane >= 250 units per step, mm1 8 below
 * 2,048 clients and 32 above; the bitsliced walk the >= 250-steps rule with S >= 4.
 * Outputs are identical. */
int wlp_set_pipe_lanes(int lanes);

/* Test hook (this thread): near-one list entries per panel of the mm1 warp pipeline, a
 * power of two in [1, 128] (default 128). Small values force the rare overflow path (the
 * panel is redrawn and every lane fixes its own near-one draws); outputs are identical. */
int wlp_debug_set_near_cap(int cap);

/* The same for the TLP (thread-level) mapping: 0 = automatic (default: one thread per
 * replication, the paper's comparison mapping); 1 = one thread per replication; 2 = walk
 * bitsliced, one thread per 32 replications, each state bit of the 32 streams in one
 * word (pi / mm1 keep the per-replication kernel). Outputs are identical. */
int wlp_set_tlp_variant(int variant);

/* Summation order of the device statistics (confidence intervals, wlp_stats_device) for
 * later calls on this thread. 0 (default): accurate — a parallel double-double sum, within
 * a few ulps of the exact sums (the reference's naive loop, models.cpp:104-109, drifts by up
 * to ~n*2^-53 relative; 9e-12 at pi 10^7 x 10^3). 1: the reference's order — one
 * sequential fp64 sum in index order, bit-identical to confidence_interval's at any n, at
 * ~4 ns per sample (n <= 256 always sums this way). Multi-slice runs (wlp_run_devices,
 * sharded statistics) merge slice sums, so their sums are the accurate kind either way. */
int wlp_set_stats_order(int order);

/* Name of the model kernel the last run on this thread launched (e.g. "k_wlp_pipe<pi>",
 * "k_wlp_walk_bs_pipe", "k_tlp_mm1"); "" before any run. Static storage. */
const char* wlp_last_kernel(void);

/* validate_params (models.cpp:26-44): WLP_EDOMAIN on invalid values; a non-empty
 * warning (lambda >= mu) is copied into warn[cap]. */
int wlp_validate_params(int model, const wlp_params* p, char* warn, int warn_cap);

/* plan_launch (wlp.cpp:71-105): reference geometry per mode, PlanError above
 * grid_limit (the reference default is 65535), partial-warp warning. */
int wlp_plan_launch(int64_t replications, int mode, int tlp_block_size, int64_t grid_limit,
                    wlp_launch_cfg* cfg, char* warn, int warn_cap);

/* rng_state_from_seed (rng.cpp:36-40). */
int wlp_master_from_seed(uint64_t seed, uint32_t state_out[3]);

/* make_rng_state (rng.cpp:29-34). */
int wlp_make_state(uint32_t s1, uint32_t s2, uint32_t s3, uint32_t state_out[3]);

/* State after n taus_next calls (rng.cpp:42-51), by GF(2) jump-ahead on the host. */
int wlp_jump_host(const uint32_t state[3], uint64_t n, uint32_t state_out[3]);

/* inverse_normal_cdf (models.cpp:61-97). */
int wlp_inverse_normal_cdf(double p, double* z);

/* The reference's scalar rng utilities (rng.hpp:22-33), on the host: taus_next
 * (rng.cpp:42-51) advancing state[3] in place, uniform01 = taus_next * 2^-32
 * (rng.cpp:53-55), and exponential_from_u = -log(1-u)/rate (rng.cpp:58-61; WLP_EDOMAIN for
 * rate <= 0 or u outside [0,1), the reference's messages) through the same glibc-log port
 * the mm1 kernels run (bit-identical to libm's on the FMA path). Bulk forms on the
 * device: wlp_taus_stream, wlp_exponentials. */
int wlp_taus_next(uint32_t state[3], uint32_t* out);
int wlp_uniform01(uint32_t state[3], double* out);
int wlp_exponential_from_u(double u, double rate, double* out);

/* Exact rejection bookkeeping of random_spacing (rng.cpp:67-87) from the special
 * candidates of all shards: sorts them by index, marks every candidate whose key equals
 * an earlier accepted one, and merges with `prev`. Returns WLP_ESPACING if one stream
 * would need 1000 redraws. out may alias nothing; cap >= n_prev + n_special. */
int wlp_spacing_rejections(const wlp_special* specials, int64_t n_special, const int64_t* prev,
                           int64_t n_prev, int64_t* out, int64_t out_cap, int64_t* n_out);

/* Merge shard statistics (b into a), exactly in double-double. */
int wlp_stats_merge(wlp_stats* a, const wlp_stats* b);

/* confidence_interval (models.cpp:99-119) from merged second-pass statistics. */
int wlp_ci_from_stats(const wlp_stats* s, double level, wlp_ci* ci);

/* ---- device entry points --------------------------------------------------------- */

int wlp_device_count(int* n);

/* Raw taus88 stream: make_rng_state(s1,s2,s3) then n outputs of taus_next
 * (rng.cpp:29-51; the taus88.golden format). Generated in parallel by jump-ahead. */
int wlp_taus_stream(uint32_t s1, uint32_t s2, uint32_t s3, int64_t n, uint32_t* out,
                    int out_on_device, void* stream);

/* random_spacing(rng_state_from_seed(master_seed), R) (rng.cpp:67-87) for stream slots
 * [slot_begin, slot_begin + count) of a run, given the global rejection list
 * (sorted candidate indices, normally empty). Keys are written SoA: s[0..count) = s1,
 * s[count..2count) = s2, s[2count..3count) = s3. Special candidates met while filling
 * the slots are appended to specials (up to cap; *n_special gets the true count).
 * Synchronous. For a whole run use slot_begin = 0, count = R and iterate with
 * wlp_spacing_rejections until no new rejection appears (wlp_seed_streams_exact). */
int wlp_seed_streams(uint64_t master_seed, int64_t slot_begin, int64_t count,
                     const int64_t* rejected, int64_t n_rejected, uint32_t* s_out,
                     int out_on_device, void* stream, wlp_special* specials,
                     int64_t special_cap, int64_t* n_special);

/* Whole-run exact random_spacing (iterates the rejection fixpoint internally). */
int wlp_seed_streams_exact(uint64_t master_seed, int64_t count, uint32_t* s_out,
                           int out_on_device, void* stream);

/* random_spacing(master, count) (rng.cpp:67-87) from an explicit master state (not
 * re-mapped); master_out (may be NULL) receives the master after all consumed draws,
 * as the reference's by-reference master. Synchronous. */
int wlp_seed_streams_state(const uint32_t master[3], int64_t count, uint32_t* s_out,
                           int out_on_device, void* stream, uint32_t master_out[3]);

/* Replications over caller-given streams (SoA s[3*count], host or device):
 * pi_replication / mm1_replication / walk_replication (models.cpp:46-59) for each,
 * mapped per `mode` (TLP: thread per replication; WLP and SEQUENTIAL: warp per
 * replication). mm1 writes out0 = avgIdle, out1 = avgWaitQueue, out2 = avgSystem;
 * pi and walk write out0 only. */
int wlp_run_streams(int model, const wlp_params* p, int mode, const uint32_t* s, int64_t count,
                    int s_on_device, double* out0, double* out1, double* out2,
                    int out_on_device, void* stream, wlp_report* report);

/* run_model (models.cpp:329-397) for a shard [r_begin, r_begin + r_count) of a run of
 * p->replications: seeds the shard's streams on device (global rejection list as in
 * wlp_seed_streams), runs the model in `mode`, writes per-replication outputs.
 * Reports the shard's special candidates so the caller can check spacing collisions
 * across shards and re-run with a rejection list in the (astronomically rare) case of
 * one. Outputs on device without a report: the call returns once the seeding has
 * reported its special candidates, with the model kernel still running on `stream`
 * (stream-ordered like any CUDA call: read the outputs on `stream` or after syncing it). */
int wlp_run_shard(int model, const wlp_params* p, int mode, uint64_t master_seed,
                  int tlp_block_size, int64_t r_begin, int64_t r_count, const int64_t* rejected,
                  int64_t n_rejected, double* out0, double* out1, double* out2,
                  int out_on_device, void* stream, wlp_special* specials, int64_t special_cap,
                  int64_t* n_special, wlp_report* report);

/* run_model (models.cpp:329-397), single device, whole run: exact seeding, model,
 * outputs, optional report, and optional device-side confidence intervals of every
 * output (ci array of 1 or 3 entries, NULL to skip) at `level`. The outputs-on-host
 * form is the reference-facing call (e2e); warning text as in build_kernel
 * (models.cpp:294-299). Outputs on device without report or ci: returns once the seeding
 * has reported, the model kernel still running on `stream` (as wlp_run_shard). */
int wlp_run(int model, const wlp_params* p, int mode, uint64_t master_seed, int tlp_block_size,
            double* out0, double* out1, double* out2, int out_on_device, void* stream,
            wlp_report* report, wlp_ci* ci, double level, char* warn, int warn_cap);

/* run_model over several GPUs of this process (SURVEY §8b device_count): the run's
 * replications are split into contiguous slices, device k = devices[k] runs
 * [k*R/n, (k+1)*R/n) with one host thread per device, the random-spacing check is global
 * (every slice's special candidates, as wlp_run_shard), and the confidence intervals
 * come from the slices' statistics merged in device order (two passes about the merged
 * mean; within 1e-12 of the single-device sums). Outputs are HOST arrays of R entries
 * (each device writes its slice), bit-identical to wlp_run. Runs below 2^15
 * replications per device use fewer devices (R < 2^16: devices[0] alone, exactly
 * wlp_run). report: kernel_ms / cycles / waves the maximum over devices, counters summed.
 * The calling thread's wlp_set_* settings apply to every device. A device may be listed
 * more than once: its slices then take turns on it (phase by phase; this is how the
 * multi-device path is exercised on a one-GPU box). */
int wlp_run_devices(int model, const wlp_params* p, int mode, uint64_t master_seed, int tlp_block_size,
                    const int* devices, int n_devices, double* out0, double* out1, double* out2,
                    wlp_report* report, wlp_ci* ci, double level, char* warn, int warn_cap);

/* The reference's *_replication_u templates (models.hpp:49-108) on the device: replication
 * r runs the model body over the caller's uniforms u[r*2n .. r*2n + 2n), n = draws /
 * clients / steps of p (p->replications is ignored; `count` replications), consuming them
 * in the reference's order (pi: x then y; mm1: arrival then service; walk: direction then
 * the discarded draw). Any double values, as the templates accept. One thread per
 * replication; outputs as wlp_run_streams. Synchronous. */
int wlp_run_uniforms(int model, const wlp_params* p, const double* u, int64_t count, int u_on_device,
                     double* out0, double* out1, double* out2, int out_on_device, void* stream);

/* exponential_from_u (rng.cpp:58-61) over n uniforms on the device (glibc-log port):
 * out[i] = -log(1 - u[i]) / rate. WLP_EDOMAIN if rate <= 0 or any u outside [0,1).
 * Synchronous. */
int wlp_exponentials(const double* u, int64_t n, double rate, double* out, int on_device, void* stream);

/* Experimental plan (BASELINE config 5): n_sets factor-level sets of one model, set k
 * being run_model(model, sets[k], mode, master_seeds[k]) — its own parameters, replication
 * count and master seed — executed as ONE batched seeding launch and ONE model launch
 * (WLP: warps take replications from a global counter; TLP: thread per replication).
 * Outputs are concatenated in set order (set k starts at sum_{j<k} sets[j].replications)
 * and bit-identical to the n_sets separate runs. Units per replication < 2^32. Into device
 * buffers without a report it returns once the seeding has reported its specials count,
 * the model still running on `stream`; host outputs or a report synchronise. */
int wlp_run_plan(int model, const wlp_params* sets, const uint64_t* master_seeds, int n_sets, int mode,
                 int tlp_block_size, double* out0, double* out1, double* out2, int out_on_device,
                 void* stream, wlp_report* report);

/* Device statistics of a device array (pass 1: n and sum; pass 2: centred sum of
 * squares about stats->center). Synchronous; n <= 256 sums sequentially, bit-identical
 * to the reference's naive loop (models.cpp:104-109). */
int wlp_stats_device(const double* x, int64_t n, int pass, wlp_stats* stats, void* stream);

/* confidence_interval over a host array through the device reduction. */
int wlp_confidence_interval(const double* samples, int64_t n, double level, wlp_ci* ci);

/* Test hook: -log(1 - k[i]*2^-32) through the device glibc-log port (host arrays). */
int wlp_debug_neg_log1m(const uint32_t* k, int64_t n, double* out);

/* ---- kernel IR on the GPU ------------------------------------
 *
 * The reference's kernel IR (kernel_ir.hpp:67-141; text form kernel_text.hpp) executed
 * by a SIMT interpreter ON the B200 instead of the reference's host simulator
 * (simulate, device.cpp:140-226; WarpState::step, warp_exec.cpp:178-298). Each IR warp
 * runs on one hardware warp, IR lane l on lane l; the warp walks the statement tree
 * with the reference's mask-stack semantics (then before else, loop re-tests, permanent
 * halts, reconvergence, stores resolved in ascending lane order), so per-lane values,
 * memory contents and the issue / divergence / memory counters are the reference
 * simulator's exactly. IR warps of one launch run concurrently: kernels whose warps
 * communicate through global memory are outside that guarantee (the reference runs
 * them one after another); the bundled models never do.
 *
 * The host C++ layer (include/warpsim_ir_b200.hpp) builds / parses programs and
 * flattens them into this form: statements laid out so every statement list is a
 * contiguous index range, expressions as typed stack bytecode (opcodes WLP_IR_OP_*;
 * every expression ends with WLP_IR_OP_END). */

/* Statement kinds (StmtKind order, kernel_ir.hpp:101). */
#define WLP_IR_ASSIGN 0
#define WLP_IR_LOAD 1
#define WLP_IR_STORE 2
#define WLP_IR_IF 3
#define WLP_IR_WHILE 4
#define WLP_IR_HALT 5

/* Statement flags: faults the type rules decide statically, raised when executed. */
#define WLP_IR_F_REAL_INTO_INT 1 /* assign of a real value into an int local      */
#define WLP_IR_F_INT_TO_REAL 2   /* assign of an int value into a real local      */
#define WLP_IR_F_REAL_INDEX 4    /* load / store index is a real                   */

typedef struct wlp_ir_stmt {
    int32_t kind;
    int32_t slot;    /* assign / load: local slot; store: array param slot */
    int32_t arr;     /* load: array param slot */
    int32_t code_a;  /* expression offset: assign value, load / store index, if / while condition */
    int32_t code_b;  /* store value */
    int32_t b1_begin, b1_end; /* then / loop body */
    int32_t b2_begin, b2_end; /* else body */
    int32_t flags;
} wlp_ir_stmt;

/* Expression bytecode: per IR lane a stack of 64-bit slots whose types are static. */
enum {
    WLP_IR_OP_END = 0,
    WLP_IR_OP_CONST,    /* + 2 words (lo, hi of the 64-bit pattern) */
    WLP_IR_OP_LOCAL,    /* + slot */
    WLP_IR_OP_PARAM,    /* + slot */
    WLP_IR_OP_SREG,     /* + Sreg (kernel_ir.hpp:73-79 order) */
    WLP_IR_OP_DRAW,     /* uniform01 of the lane's taus88 stream */
    WLP_IR_OP_I2R_0,    /* int -> real, top of stack */
    WLP_IR_OP_I2R_1,    /* int -> real, second from the top */
    WLP_IR_OP_TRUTH_0,  /* real -> int truth (r != 0), top */
    WLP_IR_OP_TRUTH_1,  /* real -> int truth, second from the top */
    WLP_IR_OP_ADD_I, WLP_IR_OP_SUB_I, WLP_IR_OP_MUL_I, WLP_IR_OP_DIV_I, WLP_IR_OP_MOD_I,
    WLP_IR_OP_ADD_R, WLP_IR_OP_SUB_R, WLP_IR_OP_MUL_R, WLP_IR_OP_DIV_R, WLP_IR_OP_MOD_R,
    WLP_IR_OP_LT_I, WLP_IR_OP_LE_I, WLP_IR_OP_GT_I, WLP_IR_OP_GE_I, WLP_IR_OP_EQ_I, WLP_IR_OP_NE_I,
    WLP_IR_OP_LT_R, WLP_IR_OP_LE_R, WLP_IR_OP_GT_R, WLP_IR_OP_GE_R, WLP_IR_OP_EQ_R, WLP_IR_OP_NE_R,
    WLP_IR_OP_AND, WLP_IR_OP_OR, /* on int truths */
    WLP_IR_OP_NEG_I, WLP_IR_OP_NEG_R, WLP_IR_OP_LOG, WLP_IR_OP_FLOOR,
    WLP_IR_OP_COUNT
};

/* Interpreter limits (the host layer rejects larger programs with WLP_EDOMAIN). */
#define WLP_IR_MAX_LOCALS 64
#define WLP_IR_MAX_STACK 32

typedef struct wlp_ir_program {
    const wlp_ir_stmt* stmts;
    int32_t n_stmts;
    int32_t top_begin, top_end; /* the kernel body */
    const int32_t* code;
    int32_t n_code;
    int32_t n_locals;
    const int64_t* local_init; /* per local: initial bits (0 / +0.0 or an initial value) */
    int32_t n_params;
    const int64_t* param_bits; /* scalar params: value bits (reals already promoted) */
    const int32_t* param_is_array;
} wlp_ir_program;

/* simulate (device.cpp:140-226) on the GPU: runs every IR warp of `cfg` (warp_size in
 * [1, 32]; threads per block <= max_threads_per_block) over the arrays (indexed by
 * param slot; NULL for scalar params; host or device memory, sizes in array_len) with
 * lane streams streams[3*n_streams] (SoA; thread t draws from stream t, the default
 * state when t >= n_streams). mask_depth bounds the mask stack (SimOptions, 1..64);
 * max_issues (> 0) bounds the statements one IR warp may issue (a guard against
 * kernels that never terminate; WLP_EFAULT when hit). Fills the report's issue /
 * alu / memory / divergence counters exactly as the reference simulator counts them,
 * plus measured time. Lane faults (division by zero, log of a non-positive value, ...)
 * return WLP_EFAULT with the reference's message. Synchronous. */
int wlp_ir_simulate(const wlp_ir_program* prog, const wlp_launch_cfg* cfg, int64_t max_threads_per_block,
                    double* const* arrays, const int64_t* array_len, int arrays_on_device,
                    const uint32_t* streams, int64_t n_streams, int streams_on_device, int mask_depth,
                    int64_t max_issues, void* stream, wlp_report* report);

/* The same program compiled instead of interpreted: translated to CUDA C++, compiled for
 * sm_100a by NVRTC (loaded on first use; cached by source) and launched with the same
 * IR-warp mapping. Memory results equal the interpreter's for kernels without cross-lane
 * memory traffic between the two sides of a divergent branch; the report carries the
 * measured time only (the issue / divergence counters need the interpreter's lockstep
 * accounting). max_iterations (> 0) bounds the loop iterations of one IR thread
 * (WLP_EFAULT when hit). WLP_ECUDA when NVRTC is unavailable. */
int wlp_ir_jit_simulate(const wlp_ir_program* prog, const wlp_launch_cfg* cfg, int64_t max_threads_per_block,
                        double* const* arrays, const int64_t* array_len, int arrays_on_device,
                        const uint32_t* streams, int64_t n_streams, int streams_on_device, int64_t max_iterations,
                        void* stream, wlp_report* report);

/* The CUDA C++ source the JIT generates for a program (for inspection). */
int wlp_ir_jit_source(const wlp_ir_program* prog, char* out, int cap, int* need);

/* Release all device scratch of the current device. */
int wlp_shutdown(void);

#ifdef __cplusplus
}
#endif

#endif /* WLP_B200_H */
