#!/usr/bin/env python3
"""Benchmark of the MRIP replication runner (BASELINE.json metric: replications/sec per
model on 1/2/4/8 B200, with warp-exec efficiency / ALU-issue fraction from ncu).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (a "step"): BASELINE config 2 — Monte-Carlo pi, 10^6 replications x 10^4 draws
per GPU (weak scaling: rank g runs slots [g*10^6, (g+1)*10^6) of one run of N*10^6
replications), master seed 42, WLP mapping: exact random-spacing seeding on device +
the WLP replication kernel + the two-pass device statistics of the outputs, merged
across ranks (all_gather of sufficient statistics), -> mean / 95% CI.

  value  device-resident: outputs stay in HBM, CUDA events on the launching stream over
         exactly K steps after W warm-ups, barrier + synchronize on both sides, max over
         ranks. Inputs (the replications' 12-byte stream seeds) are generated in the step.
         The 8 MB output per GPU and the 120 MB of seeds are far below L2 capacity
         reuse distance: every step rewrites them (config "l2": "inputs regenerated").
  e2e    the same metric through the reference-facing call with HOST buffers: at N=1
         wlp_run (run_model) writing per-replication outputs to pinned host memory + device
         CI; at N>1 the sharded step plus the D2H of the shard's outputs. Wall clock
         (perf_counter with synchronize), max over ranks.

Extras (N=1): WLP and TLP rates for every model/config of BASELINE (2, 3, 4, 5), the
ALU-issue roofline of the dominant kernel, the IR path (interpreter and JIT), and the CPU
baseline (the reference's own replication functions, oracle/_ref, on all host cores,
bounded sample). Under torchrun (every N): "cfg4_sharded_1e7" — BASELINE config 4 as
stated, all three models with 10^7 replications in total sharded over the N GPUs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "replications/sec (pi, 1e6 reps x 1e4 draws per GPU, WLP)"
UNIT = "replications/s"
R_PER_GPU = 1_000_000
DRAWS = 10_000
SEED = 42

# Algorithmic instruction counts per unit (issue slots of one lane), see DESIGN.md §roofline:
# one taus88 draw = 16 SASS (6 IMAD.SHL, 3 shift-merge, 7 LOP3); pi point = 2 draws +
# 2 exact u32->f64 + 2 DMUL + DADD + DSETP + count = 39; walk step = 2 draws + shift +
# 2 compare/add = 35.
INSTR_PER_UNIT = {0: 39, 2: 35}
# Bitsliced walk (csrc/bitslice.cuh): LOP3 per walk step for 32 replications at once, as
# compiled (726 per 16-step carry-save block of k_tlp_walk_bs).
BS_LOP3_PER_STEP = 45.4
# mm1 is FP64-pipe work: per client two exponentials, each 1-u (1) + glibc log (15 fp ops
# on the table path as compiled in __log_fma, 26 on the near-one path taken 1 time in 16:
# 15.7 average) + negate/scale (1), plus the Lindley step (6 DADD + 1 compare) = 42.
FP64_PER_CLIENT = 42


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------------------------


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.flush()
        rows = [r.split(", ") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        loaded = [s for s in sm if mx and s >= 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def ncu_traffic() -> dict:
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    try:
        return json.loads((ROOT / "profiles" / "ncu_summary.json").read_text())
    except Exception:
        return {}


# ---------------------------------------------------------------------------------------------


def dist_setup():
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or "LOCAL_RANK" in os.environ:  # under torchrun: always the NCCL path
        import torch.distributed as dist

        torch.cuda.set_device(local)
        # NCCL's "NCCL version ..." banner goes to stdout at communicator creation; keep
        # stdout for the one JSON line by pointing fd 1 at stderr while the comm comes up
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
            torch.cuda.synchronize()
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def device_timed(step, steps: int, warmup: int, world: int):
    """CUDA-event time per step over exactly `steps` steps (after `warmup`), max over ranks."""
    import torch

    for _ in range(warmup):
        step()
    barrier(world)
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        step()
    e1.record(s)
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(e0.elapsed_time(e1) / steps, world)


def wall_timed(step, steps: int, warmup: int, world: int):
    import torch

    for _ in range(warmup):
        step()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    t = (time.perf_counter() - t0) * 1e3 / steps
    barrier(world)
    return max_over_ranks(t, world)


# ---------------------------------------------------------------------------------------------


def cpu_baseline(model: int, p, budget_s: float = 15.0, steps: int = 1):
    """The reference's own host path (oracle/_ref = proj/src compiled unmodified):
    random_spacing (sequential, as in the reference) + the replication functions on all
    host threads (they are pure), on a bounded sample of the workload."""
    import oracle

    ref = oracle.Oracle("reference") if oracle.available("reference") else oracle.Oracle("port")
    kind = "reference" if ref.kind == "reference" else "port"
    nth = os.cpu_count() or 1
    op = oracle.params_from(p)

    def run(S):
        t0 = time.perf_counter()
        keys = ref.random_spacing(SEED, S)
        t1 = time.perf_counter()
        if kind == "reference":
            ref.replications(model, op, keys, nthreads=nth)
        else:
            ref.replications(model, op, keys)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    S = 4 * nth
    a, b = run(S)
    per = (a + b) / S
    S = int(max(4 * nth, min(p.replications, budget_s / max(per, 1e-9))))
    S = max(nth, (S // nth) * nth)
    tot = [run(S) for _ in range(steps)]
    tsp = sum(x for x, _ in tot) / steps
    trep = sum(y for _, y in tot) / steps
    # single-core rate of the same functions on a small slice
    s1 = max(4, min(S, int(2.0 / max(per * nth, 1e-9))))
    keys = ref.random_spacing(SEED, s1)
    t0 = time.perf_counter()
    if kind == "reference":
        ref.replications(model, op, keys, nthreads=1)
    else:
        ref.replications(model, op, keys)
    t1 = time.perf_counter()
    return {"value": S / (tsp + trep), "unit": UNIT, "cores": nth if kind == "reference" else 1, "kind": kind,
            "sample": f"{S} of {p.replications} replications (seed {SEED}): random_spacing 1 thread "
                      f"{tsp:.3f}s + replications on {nth if kind == 'reference' else 1} threads {trep:.3f}s",
            "single_core_value": s1 / (t1 - t0 + tsp / S * s1), "single_core_sample": f"{s1} replications",
            "step_s": tsp + trep}


def ir_simulator_baseline() -> dict:
    """The reference's own simulator (simulate, device.cpp:140-226 via run_model Tlp) on the
    IR walk that extras.ir_walk_tlp_2e4x1e3 runs on the GPU interpreter, on a 10x smaller
    sample (R = 2000, 1 host thread: the simulator is single-threaded)."""
    try:
        import oracle

        t0 = time.perf_counter()
        rr = oracle.Oracle("reference").run_model_report(2, oracle.params(replications=2000, steps=1000, chunks=30),
                                                         SEED, 1)
        dt = time.perf_counter() - t0
        return {"sample": "walk TLP R=2000 x 1000 steps, 1 host thread", "seconds": dt, "issues": rr["issues"],
                "issues_per_s": rr["issues"] / dt, "cores": 1, "kind": "reference"}
    except Exception as e:  # pragma: no cover - oracle/_ref absent
        return {"unavailable": str(e)}


def run_reference_arm(args):
    """--impl reference: the reference CPU path on this box's host cores."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_1501_01405_b200 as w

    p = w.ModelParams(replications=R_PER_GPU * world, draws=DRAWS)
    # one calibration/warm-up step, then exactly K steps, each a bounded sample: ~6 s of CPU
    # work, less when K is large, so the whole arm stays within ~2.5 minutes
    budget = max(1.0, min(6.0, 150.0 / (args.steps + 1)))
    cal = cpu_baseline(0, p, budget_s=budget)
    rates = [cpu_baseline(0, p, budget_s=budget)["value"] for _ in range(args.steps)]
    v = statistics.mean(rates)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * p.replications / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
            "data": "synthetic (taus88 streams from master seed 42)",
            "config": {"workload": "BASELINE config 2: pi, 1e6 replications x 1e4 draws per GPU",
                       "replications": p.replications, "draws": DRAWS},
            "cpu_baseline": {k: cal[k] for k in ("kind", "cores", "sample")} | {"value": v, "unit": UNIT},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------


def model_rate(w, model, p, mode, steps=5, warmup=3):
    """Device-resident replications/s of one (model, mode) run on this GPU + kernel ms."""
    import torch

    from paper_1501_01405_b200 import OUTPUT_NAMES, SimReport

    outs = [torch.empty(p.replications, dtype=torch.float64, device="cuda") for _ in OUTPUT_NAMES[model]]
    kms = []

    def step():
        rep = SimReport()
        w.run_shard(model, p, mode, SEED, 0, p.replications, outs, on_device=True, report=rep)
        kms.append(rep.kernel_ms)

    ms = device_timed(step, steps, warmup, 1)
    k = kms[warmup:]
    return {"reps_per_s": p.replications / (ms * 1e-3), "ms_per_run": ms, "kernel_ms": sum(k) / len(k),
            "kernel": w.last_kernel()}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch

    import paper_1501_01405_b200 as w
    from paper_1501_01405_b200 import distributed as D

    world, rank, local = dist_setup()
    model, mode = w.ModelKind.Pi, w.ExecutionMode.Wlp
    R = R_PER_GPU * world
    p = w.ModelParams(replications=R, draws=DRAWS)
    stream = torch.cuda.current_stream().cuda_stream
    comm = D._Comm(device="cuda")
    kernel_ms: list = []
    runner = D.gpu_runner(model, p, mode, SEED, stream=stream, kernel_ms=kernel_ms)
    stats = D.gpu_stats(stream=stream)
    result = {}

    def step():
        result["r"] = D.run_sharded(model, R, runner, stats, comm=comm)

    clocks = Clocks(local)
    clocks.start()
    ms = device_timed(step, args.steps, args.warmup, world)
    clk = clocks.stop()
    k_ms = kernel_ms[args.warmup:]
    kernel_avg = sum(k_ms) / len(k_ms)
    kernel_avg = max_over_ranks(kernel_avg, world)
    value = R / (ms * 1e-3)
    # launches of our kernels per step: seed + model + 2 statistics passes (1 output)
    launches = args.steps * 4
    ci = result["r"].cis[0]

    # ---- e2e through the reference-facing call with host buffers
    count = result["r"].count
    host = [torch.empty(count, dtype=torch.float64, pin_memory=True)]
    if world == 1:
        def e2e_step():
            w.run_model_into(model, p, mode, SEED, [h.numpy() for h in host], on_device=False, ci_level=0.95)
    else:
        def e2e_step():
            r = D.run_sharded(model, R, runner, stats, comm=comm)
            host[0].copy_(r.outputs[0][:count], non_blocking=False)
    e2e_ms = wall_timed(e2e_step, args.steps, min(args.warmup, 3), world)

    # ---- roofline of the dominant kernel (ALU issue; no tensor cores on this path)
    peaks = measured_peaks()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    units = R_PER_GPU * DRAWS
    achieved = units * INSTR_PER_UNIT[0] / 32 / (kernel_avg * 1e-3) / 1e9  # G warp-instr/s
    peak = 4 * sms * fmax * 1e6 / 1e9
    # latest committed capture of this kernel at this workload (the capture names end in R)
    caps = {k: v for name in ("k_wlp_lanes<0>", "k_wlp_lanes<0, 0>")
            for k, v in ncu_traffic().get(name, {}).items() if k.endswith(f"_{R_PER_GPU}")}
    nc = caps[sorted(caps)[-1]] if caps else {}
    roofline = {"bound": "issue", "kernel": "k_wlp_lanes<0> (pi WLP)", "achieved": achieved, "peak": peak,
                "unit": "Gwarp-inst/s", "frac": achieved / peak, "traffic": nc.get("dram_bytes_per_launch"),
                "algorithmic": f"{INSTR_PER_UNIT[0]} lane-instr/point x {units:.0e} points per launch / 32",
                "peak_source": f"4 issue/clk x {sms} SMs x sm_max_mhz {fmax:.0f} (MEASURED_PEAKS.json); "
                               "no tensor/HBM roofline applies (integer/fp64 ALU work)",
                "kernel_ms": kernel_avg,
                "frac_at_measured_clock": (achieved / (4 * sms * clk["sm_mhz"] * 1e-3)) if clk.get("sm_mhz") else None,
                "hbm_gbs_output_writeout": (R_PER_GPU * 8 + 3 * 4 * R_PER_GPU) / (kernel_avg * 1e-3) / 1e9}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32+f64",
            "data": "synthetic (taus88 streams by random spacing from master seed 42)",
            "config": {"workload": "BASELINE config 2: pi, 1e6 replications x 1e4 draws per GPU, WLP",
                       "replications": R, "draws": DRAWS, "mode": "wlp", "parallelism": f"shard{world}",
                       "l2": "inputs regenerated every step (seeds 12 B/rep + outputs 8 B/rep)"},
            "e2e": {"value": R / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 64 * world,
                    "d2h_bytes_per_step": R * 8, "ms_per_step": e2e_ms,
                    "note": "inputs are (master seed, params) by value; outputs D2H to pinned host"},
            "gpu_launches": launches, "clocks": clk, "roofline": roofline,
            "result": {"mean": ci.mean, "half_width": ci.halfWidth, "n": ci.n}}

    if (world > 1 or "LOCAL_RANK" in os.environ) and not args.no_extras:
        # BASELINE config 4 as stated (every torchrun launch, N >= 1): all models, 10^7
        # replications in total sharded over the N GPUs (strong scaling), WLP, the two
        # statistics exchanges included; time is the max over ranks of the device time
        sharded = {}
        for name, m, kw in [("pi", w.ModelKind.Pi, dict(draws=1000)), ("mm1", w.ModelKind.Mm1, dict(clients=1000)),
                            ("walk", w.ModelKind.Walk, dict(steps=1000, chunks=30))]:
            p4 = w.ModelParams(replications=10_000_000, **kw)
            run4 = D.gpu_runner(m, p4, w.ExecutionMode.Wlp, SEED, stream=stream)

            def step4():
                D.run_sharded(m, p4.replications, run4, stats, comm=comm)

            ms4 = device_timed(step4, 3, 3, world)
            sharded[name] = {"reps_per_s": p4.replications / (ms4 * 1e-3), "ms_per_run": ms4}
        line["cfg4_sharded_1e7"] = sharded
    if world == 1 and not args.no_extras:
        extras = {}
        cfgs = [("cfg2_pi_1e6x1e4", w.ModelKind.Pi, dict(replications=1_000_000, draws=10_000)),
                ("cfg3_walk_1e5x1e3", w.ModelKind.Walk, dict(replications=100_000, steps=1000, chunks=30)),
                ("cfg4_pi_1e7x1e3", w.ModelKind.Pi, dict(replications=10_000_000, draws=1000)),
                ("cfg4_mm1_1e7x1e3", w.ModelKind.Mm1, dict(replications=10_000_000, clients=1000)),
                ("cfg4_walk_1e7x1e3", w.ModelKind.Walk, dict(replications=10_000_000, steps=1000, chunks=30))]
        for name, m, kw in cfgs:
            pp = w.ModelParams(**kw)
            extras[name] = {}
            for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
                r = model_rate(w, m, pp, md)
                units_ = pp.replications * pp.units(m)
                if "walk_bs" in r["kernel"]:  # bitsliced: ALU pipe against its own LOP3 count
                    r["alu_frac"] = units_ * BS_LOP3_PER_STEP / 32 / 32 / (r["kernel_ms"] * 1e-3) / (2 * sms * fmax * 1e6)
                elif m in INSTR_PER_UNIT:
                    r["issue_frac"] = units_ * INSTR_PER_UNIT[int(m)] / 32 / (r["kernel_ms"] * 1e-3) / (peak * 1e9)
                else:  # FP64 pipe: 64 lanes/clk/SM (measured, profiles/round1_microbench.txt)
                    r["fp64_frac"] = units_ * FP64_PER_CLIENT / (r["kernel_ms"] * 1e-3) / (64 * sms * fmax * 1e6)
                extras[name][w.mode_name(md)] = r
            if m == w.ModelKind.Walk:
                # the walk's other kernels (DESIGN.md §4 bitsliced walk): per-replication
                # WLP pipeline / lane jumps, and the bitsliced TLP (thread per 32 replications).
                # Bitsliced work is ~45 LOP3 per step per 32 replications, ALU pipe 2/clk/SM.
                units_ = pp.replications * pp.steps
                for label, wv, tv, md in (("wlp_per_replication", 2 if pp.replications >= 1_000_000 else 1, 0,
                                           w.ExecutionMode.Wlp),
                                          ("tlp_bitsliced", 0, 2, w.ExecutionMode.Tlp)):
                    with w.wlp_variant(wv), w.tlp_variant(tv):
                        r = model_rate(w, m, pp, md)
                    if "walk_bs" in r["kernel"]:
                        r["alu_frac"] = units_ * BS_LOP3_PER_STEP / 32 / 32 / (r["kernel_ms"] * 1e-3) / (2 * sms * fmax * 1e6)
                    else:
                        r["issue_frac"] = units_ * INSTR_PER_UNIT[2] / 32 / (r["kernel_ms"] * 1e-3) / (peak * 1e9)
                    extras[name][label] = r
        # config 3's warp-execution evidence (paper Table 1 / Fig. 7 analogue): divergence
        # events with the reference's definition and global memory warp-instructions, from
        # the instrumented kernels (outputs identical; counters cost a little speed)
        pw = w.ModelParams(replications=100_000, steps=1000, chunks=30)
        table1 = {}
        with w.hw_counters():
            for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
                rr = w.run_model(w.ModelKind.Walk, pw, md, master_seed=SEED).report
                table1[w.mode_name(md)] = {"divergence_events": rr.divergenceEvents, "mem_reads": rr.memReads,
                                           "mem_writes": rr.memWrites}
        extras["cfg3_walk_1e5x1e3"]["counters"] = table1
        # config 5: experimental plan, 64 factor-level sets x 30 replications, one launch
        sets = [w.ModelParams(replications=30, clients=10_000, lambda_=0.1 + 0.8 * k / 63, mu=1.0) for k in range(64)]
        seeds = [SEED + k for k in range(64)]
        extras["cfg5_plan_mm1_64x30x1e4"] = {}
        for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            outs = [torch.empty(64 * 30, dtype=torch.float64, device="cuda") for _ in range(3)]
            kms = []

            def pstep():
                rep = w.SimReport()
                w.run_plan(w.ModelKind.Mm1, sets, seeds, md, outs, on_device=True, report=rep)
                kms.append(rep.kernel_ms)

            pms = device_timed(pstep, 5, 3, 1)
            extras["cfg5_plan_mm1_64x30x1e4"][w.mode_name(md)] = {
                "reps_per_s": 1920 / (pms * 1e-3), "ms_per_run": pms, "kernel_ms": sum(kms[3:]) / len(kms[3:])}
        # config 5's trip-count-heterogeneous variant: walk sets with
        # steps_k = 100 + 30k, so a TLP warp spanning two sets idles lanes; one launch each
        hsets = [w.ModelParams(replications=30, steps=100 + 30 * k, chunks=30) for k in range(64)]
        extras["cfg5_plan_walk_hetero_64x30"] = {}
        for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            hout = [torch.empty(64 * 30, dtype=torch.float64, device="cuda")]
            hk = []

            def hstep():
                rep = w.SimReport()
                w.run_plan(w.ModelKind.Walk, hsets, seeds, md, hout, on_device=True, report=rep)
                hk.append(rep.kernel_ms)

            hms = device_timed(hstep, 5, 3, 1)
            extras["cfg5_plan_walk_hetero_64x30"][w.mode_name(md)] = {
                "reps_per_s": 1920 / (hms * 1e-3), "ms_per_run": hms, "kernel_ms": sum(hk[3:]) / len(hk[3:])}
        # the reference's own IR kernel (TLP walk) on the GPU IR interpreter:
        # statements issued per second, counters exact; the reference's host simulator on
        # a 10x smaller sample beside it when the CPU legs run
        from paper_1501_01405_b200 import ir

        pir = w.ModelParams(replications=20_000, steps=1000, chunks=30)
        runs = [ir.run_model(w.ModelKind.Walk, pir, w.ExecutionMode.Tlp, SEED) for _ in range(3)]
        kms = min(r.report.kernel_ms for r in runs)
        extras["ir_walk_tlp_2e4x1e3"] = {"kernel_ms": kms, "issues": runs[-1].report.issues,
                                         "divergence_events": runs[-1].report.divergenceEvents,
                                         "issues_per_s": runs[-1].report.issues / (kms * 1e-3)}
        # the same IR kernel compiled (IR -> CUDA C++ -> NVRTC), first call compiles
        jruns = [ir.run_model(w.ModelKind.Walk, pir, w.ExecutionMode.Tlp, SEED, jit=True) for _ in range(4)]
        jms = min(r.report.kernel_ms for r in jruns[1:])
        assert all((r.primary == runs[-1].primary).all() for r in jruns)
        extras["ir_walk_tlp_2e4x1e3"]["jit"] = {"kernel_ms": jms, "speedup_vs_interpreter": kms / jms}
        line["extras"] = extras
    if world == 1 and rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = {k: v for k, v in cpu_baseline(0, p).items() if k != "step_s"}
        if "extras" in line:  # the reference's host simulator beside the GPU IR interpreter
            line["cpu_baseline"]["ir_reference_simulator"] = ir_simulator_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
