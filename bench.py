#!/usr/bin/env python3
"""Benchmark of the MRIP replication runner (BASELINE.json metric: replications/sec per
model on 1/2/4/8 B200, with the warp-exec / ALU-issue evidence).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 outside torchrun, bench.py re-launches itself under
`torch.distributed.run` with N ranks (one per GPU, NCCL, 127.0.0.1); under torchrun it
checks WORLD_SIZE == N. `--dry-run` brings the ranks up over gloo on CPU and exercises
only that launch / barrier / max-over-ranks plumbing (tests/test_bench_launch.py).

Headline (a "step"): BASELINE config 2 — Monte-Carlo pi, 10^6 replications x 10^4 draws
per GPU (weak scaling: rank g runs slots [g*10^6, (g+1)*10^6) of one run of N*10^6
replications), master seed 42, WLP: exact random-spacing seeding on device + the WLP
replication kernel + the two-pass device statistics, merged across ranks (all_gather of
sufficient statistics) -> mean / 95% CI.

  value  device-resident: CUDA events on the launching stream over exactly K steps after
         W warm-ups, barrier + synchronize on both sides, max over ranks. The step's
         inputs (12-byte stream keys per replication) are generated in the step and its
         outputs (8 B per replication) rewritten, every step.
  e2e    the same metric through the reference-facing call with HOST buffers: at N=1
         wlp_run (run_model) writing per-replication outputs to pinned host memory plus the
         device CI; at N>1 each rank's wlp_run_shard writing its slice to pinned host memory
         plus the statistics exchange. Synchronised wall clock, max over ranks.

"models" (every N): BASELINE config 4 as stated — each model with 10^7 replications in
total sharded over the N GPUs (strong scaling), WLP, N = 1000 units: device value, e2e
(host buffers), the roofline of the model's kernel (name taken from the run), and at
N=1 the reference's own CPU path on all host cores (bounded sample).

Extras (N=1): WLP vs TLP for configs 2-5, the walk's alternative kernels, the measured
divergence counters, the IR path, and the CPU baselines.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "replications/sec (pi, 1e6 reps x 1e4 draws per GPU, WLP)"
UNIT = "replications/s"
R_PER_GPU = 1_000_000
DRAWS = 10_000
SEED = 42
R_CFG4 = 10_000_000

# Algorithmic instruction counts per unit (issue slots of one lane), see DESIGN.md §6:
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

CFG4 = [("pi", 0, dict(draws=1000)), ("mm1", 1, dict(clients=1000)), ("walk", 2, dict(steps=1000, chunks=30))]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dry-run", action="store_true", help="launch plumbing only (gloo, CPU)")
    return ap.parse_args()


# ---- launch ----------------------------------------------------------------------------------


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> None:
    """--gpus N > 1 outside torchrun: re-run this command as N torchrun ranks (returns
    only when already under torchrun or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    sys.stdout.flush()
    r = subprocess.run(cmd)
    sys.exit(r.returncode)


def world_of(args) -> tuple[int, int, int]:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but torchrun started {world} ranks")
    return world, rank, local


def dist_setup(args):
    import torch

    world, rank, local = world_of(args)
    if "LOCAL_RANK" in os.environ:  # under torchrun: always the NCCL path (even at N = 1)
        import torch.distributed as dist

        torch.cuda.set_device(local)
        # NCCL's banner goes to stdout at communicator creation; keep stdout for the one
        # JSON line by pointing fd 1 at stderr while the communicator comes up
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
        assert dist.get_world_size() == args.gpus
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def dry_run(args) -> None:
    """The launch plumbing without a GPU: gloo ranks, barrier, max over ranks."""
    import torch
    import torch.distributed as dist

    world, rank, _ = world_of(args)
    if "LOCAL_RANK" in os.environ:
        dist.init_process_group("gloo")
        assert dist.get_world_size() == args.gpus
    t = torch.tensor([float(rank + 1)])
    if dist.is_initialized():
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world, "world": world,
                          "backend": dist.get_backend() if dist.is_initialized() else None,
                          "max_over_ranks": float(t.item())}), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


# ---- timing ----------------------------------------------------------------------------------


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
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
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


def ncu_capture(kernel: str, config: str = "") -> dict:
    """The committed ncu summary of `kernel` (profiles/ncu_summary.json, keyed by the name
    wlp_last_kernel reports) for this configuration: the capture whose label ends with
    `config` (e.g. "cfg4_pi_wlp", tools/prof_round2.sh), else none."""
    try:
        caps = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get(kernel, {})
    except Exception:
        return {}
    keys = sorted(k for k in caps if config and k.endswith(config))
    return caps[keys[-1]] if keys else {}


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


# ---- CPU path of the reference ----------------------------------------------------------------


def cpu_sample(model: int, p, S: int):
    """The reference's own host path (oracle/_ref = proj/src compiled unmodified) over the
    first S replications of the run: random_spacing (sequential, as in the reference) +
    the replication functions on all host threads (pure functions).
    Returns (seconds spacing, seconds replications, kind, threads)."""
    import oracle

    ref = oracle.Oracle("reference") if oracle.available("reference") else oracle.Oracle("port")
    kind = "reference" if ref.kind == "reference" else "port"
    nth = (os.cpu_count() or 1) if kind == "reference" else 1
    op = oracle.params_from(p)
    t0 = time.perf_counter()
    keys = ref.random_spacing(SEED, S)
    t1 = time.perf_counter()
    if kind == "reference":
        ref.replications(model, op, keys, nthreads=nth)
    else:
        ref.replications(model, op, keys)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, kind, nth


def cpu_baseline(model: int, p, budget_s: float = 10.0) -> dict:
    """Replications/s of the reference's CPU path on a bounded sample (~budget_s seconds)
    of the run, plus the single-core rate of the replication functions."""
    nth = os.cpu_count() or 1
    a, b, kind, used = cpu_sample(model, p, 4 * nth)
    per = (a + b) / (4 * nth)
    S = int(max(4 * nth, min(p.replications, budget_s / max(per, 1e-9))))
    S = max(nth, (S // nth) * nth)
    tsp, trep, kind, used = cpu_sample(model, p, S)
    s1 = max(4, min(S, int(2.0 / max(trep / S * used, 1e-9))))
    _, t1rep, _, _ = cpu_sample_single(model, p, s1)
    return {"value": S / (tsp + trep), "unit": UNIT, "cores": used, "kind": kind,
            "sample": f"first {S} of {p.replications} replications (seed {SEED}): random_spacing 1 thread "
                      f"{tsp:.3f}s + replications on {used} threads {trep:.3f}s",
            "single_core_value": s1 / (t1rep + tsp / S * s1), "single_core_sample": f"{s1} replications"}


def cpu_sample_single(model: int, p, S: int):
    import oracle

    ref = oracle.Oracle("reference") if oracle.available("reference") else oracle.Oracle("port")
    op = oracle.params_from(p)
    keys = ref.random_spacing(SEED, S)
    t0 = time.perf_counter()
    if ref.kind == "reference":
        ref.replications(model, op, keys, nthreads=1)
    else:
        ref.replications(model, op, keys)
    return 0.0, time.perf_counter() - t0, ref.kind, 1


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


def headline_config(n: int) -> dict:
    return {"workload": "BASELINE config 2: pi, 1e6 replications x 1e4 draws per GPU, WLP",
            "replications": R_PER_GPU * n, "draws": DRAWS, "mode": "wlp", "parallelism": f"shard{n}",
            "l2": "inputs regenerated every step (seeds 12 B/rep + outputs 8 B/rep)"}


def run_reference_arm(args):
    """--impl reference: the reference's CPU path (oracle/_ref) on this box's host cores, on
    the headline workload (N*10^6 pi replications x 10^4 draws). Each timed step is one
    measured pass over a bounded sample of it — the whole run when it fits — sized so the
    arm ends within a few minutes; ms_per_step is that pass's measured time."""
    world, rank, _ = world_of(args)
    if rank != 0:
        return
    import paper_1501_01405_b200 as w

    n = args.gpus
    p = w.ModelParams(replications=R_PER_GPU * n, draws=DRAWS)
    nth = os.cpu_count() or 1
    a, b, kind, used = cpu_sample(0, p, 4 * nth)  # calibration (not a step)
    per = (a + b) / (4 * nth)
    budget = max(2.0, 150.0 / max(args.steps, 1))
    S = int(min(p.replications, max(nth, budget / max(per, 1e-9))))
    S = max(nth, (S // nth) * nth) if S < p.replications else S
    for _ in range(args.warmup):
        cpu_sample(0, p, max(nth, S // 50))  # short warm-up passes (page-in, threads)
    times = []
    for _ in range(args.steps):
        tsp, trep, kind, used = cpu_sample(0, p, S)
        times.append(tsp + trep)
    step_s = sum(times) / len(times)
    v = S / step_s
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": n,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * step_s,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32+f64",
            "data": "synthetic (taus88 streams by random spacing from master seed 42)",
            "config": headline_config(n),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": used, "kind": kind,
                             "sample": f"each step: the first {S} of {p.replications} replications "
                                       f"(random_spacing on 1 thread + pi_replication on {used} threads)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- GPU arm -----------------------------------------------------------------------------------


def roofline_of(model: int, kernel: str, units: int, kernel_ms: float, sms: int, fmax: float,
                capture: str = "") -> dict:
    """The roofline that bounds `kernel`: issue slots (pi, per-replication
    walk), the ALU pipe (bitsliced walk: LOP3) or the FP64 pipe (mm1). No tensor-core or
    HBM roofline applies (integer / FP64 ALU work, ~20 B of HBM per replication)."""
    t = kernel_ms * 1e-3
    if "walk_bs" in kernel:
        achieved = units * BS_LOP3_PER_STEP / 32 / 32 / t / 1e9
        peak, bound = 2 * sms * fmax * 1e-3, "alu_pipe"
        algo = f"{BS_LOP3_PER_STEP} LOP3 per step per 32 replications x {units:.0e} steps / 32 lanes"
    elif model == 1:
        achieved = units * FP64_PER_CLIENT / 32 / t / 1e9
        peak, bound = 2 * sms * fmax * 1e-3, "fp64_pipe"
        algo = f"{FP64_PER_CLIENT} FP64 lane-ops per client x {units:.0e} clients / 32"
    else:
        achieved = units * INSTR_PER_UNIT[model] / 32 / t / 1e9
        peak, bound = 4 * sms * fmax * 1e-3, "issue"
        algo = f"{INSTR_PER_UNIT[model]} lane-instr per unit x {units:.0e} units / 32"
    cap = ncu_capture(kernel, capture)
    return {"bound": bound, "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "Gwarp-inst/s",
            "frac": achieved / peak, "traffic": cap.get("dram_bytes_per_launch"), "algorithmic": algo,
            "kernel_ms": kernel_ms,
            "peak_source": f"{'4 issue' if bound == 'issue' else '2 warp-instr'}/clk/SM x {sms} SMs x "
                           f"sm_max_mhz {fmax:.0f} (MEASURED_PEAKS.json; pipe rates profiles/round1_microbench.txt)"}


def model_rate(w, model, p, mode, steps=5, warmup=3):
    """Device-resident replications/s of one (model, mode) run on this GPU + kernel ms.

    ms_per_run: whole run_shard calls back to back (seeding, model, the specials readback
    and the host's own work; CUDA events over `steps` calls). kernel_ms: the model kernel
    alone, from separate calls with a SimReport (its timing events keep the kernel from
    overlapping the seeding, so those calls are not the ones timed per run)."""
    import torch

    from paper_1501_01405_b200 import OUTPUT_NAMES, SimReport

    outs = [torch.empty(p.replications, dtype=torch.float64, device="cuda") for _ in OUTPUT_NAMES[model]]

    def step():
        w.run_shard(model, p, mode, SEED, 0, p.replications, outs, on_device=True)

    ms = device_timed(step, steps, warmup, 1)
    kms = []
    for _ in range(max(steps, 3)):
        rep = SimReport()
        w.run_shard(model, p, mode, SEED, 0, p.replications, outs, on_device=True, report=rep)
        kms.append(rep.kernel_ms)
    k = kms[1:]
    kernel_ms = sum(k) / len(k)
    return {"reps_per_s": p.replications / (ms * 1e-3), "ms_per_run": ms, "kernel_ms": kernel_ms,
            "run_over_kernel": ms / kernel_ms, "kernel": w.last_kernel()}


def model_kernel_ms(D, model, p, R, stats, comm, stream, calls: int = 4) -> float:
    """The model kernel's own time (CUDA events around its launch), from separate calls
    after the timed steps: the events keep the kernel from overlapping the seeding, so
    the timed steps run without them."""
    import paper_1501_01405_b200 as w

    kms: list = []
    runner = D.gpu_runner(model, p, w.ExecutionMode.Wlp, SEED, stream=stream, kernel_ms=kms)
    for _ in range(calls):
        D.run_sharded(model, R, runner, stats, comm=comm)
    return sum(kms[1:]) / len(kms[1:])


def sharded_record(w, D, model: int, p, world: int, comm, stats, stream, steps: int, warmup: int, sms, fmax,
                   e2e_single_call: bool) -> dict:
    """One run of p.replications sharded over the ranks: device value, e2e with host
    buffers, and the roofline of the model kernel that ran."""
    import torch

    R = p.replications
    runner = D.gpu_runner(model, p, w.ExecutionMode.Wlp, SEED, stream=stream)
    res = {}

    def step():
        res["r"] = D.run_sharded(model, R, runner, stats, comm=comm)

    ms = device_timed(step, steps, warmup, world)
    kernel = w.last_kernel()
    kernel_avg = max_over_ranks(model_kernel_ms(D, model, p, R, stats, comm, stream), world)
    r = res["r"]
    nout = len(w.OUTPUT_NAMES[w.ModelKind(model)])
    host = [torch.empty(max(r.count, 1), dtype=torch.float64, pin_memory=True) for _ in range(nout)]
    if e2e_single_call:  # N = 1: the reference-facing run_model (wlp_run) into host buffers
        def e2e_step():
            w.run_model_into(model, p, w.ExecutionMode.Wlp, SEED, [h.numpy() for h in host], on_device=False,
                             ci_level=0.95)
    else:  # each rank: its shard written to host memory + the statistics exchange
        def e2e_step():
            rr = D.run_sharded(model, R, runner, stats, comm=comm)
            for h, o in zip(host, rr.outputs):
                h[: rr.count].copy_(o[: rr.count])

    e2e_ms = wall_timed(e2e_step, steps, min(warmup, 3), world)
    units = r.count * p.units(w.ModelKind(model))  # this rank's units per launch
    ci = r.cis[w.OUTPUT_NAMES[w.ModelKind(model)].index(w.PRIMARY[w.ModelKind(model)])]
    return {"value": R / (ms * 1e-3), "unit": UNIT, "ms_per_run": ms, "kernel": kernel,
            "e2e": {"value": R / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_run": e2e_ms,
                    "h2d_bytes_per_step": 64 * world, "d2h_bytes_per_step": 8 * nout * R,
                    "call": "wlp_run (run_model) into pinned host arrays" if e2e_single_call
                    else "wlp_run_shard per rank into pinned host arrays + statistics exchange"},
            "roofline": roofline_of(model, kernel, units, kernel_avg, sms, fmax,
                                    capture=f"cfg4_{w.model_name(w.ModelKind(model))}_wlp"),
            "result": {"mean": ci.mean, "half_width": ci.halfWidth, "n": ci.n},
            "gpu_launches_per_step": 2 + (3 if world == 1 else 2) * nout}


def ncu_warp_efficiency() -> dict:
    """Warp-execution evidence per configuration and mapping from the committed ncu
    captures of the same kernels (profiles/round2_ncu.json, tools/prof_round2.sh): branch
    uniformity (smsp__sass_average_branch_targets_threads_uniform.pct) and active threads
    per warp-instruction. Captured on the B200 with ncu; not measured by this run (ncu
    replays each kernel ~40 times)."""
    try:
        caps = json.loads((ROOT / "profiles" / "round2_ncu.json").read_text())
    except Exception:
        return {}
    return {label: {"kernel": c.get("kernel"), "branch_uniform_pct": c.get("branch_uniform_pct"),
                    "threads_per_warp_instr": c.get("threads_per_warp_instr"), "issue_pct": c.get("issue_pct")}
            for label, c in caps.items() if label != "cfg3_seed"}


def extras_single_gpu(w, sms, fmax, peak_issue) -> dict:
    import torch

    extras = {"ncu_warp_efficiency": ncu_warp_efficiency()}
    cfgs = [("cfg2_pi_1e6x1e4", w.ModelKind.Pi, dict(replications=1_000_000, draws=10_000)),
            ("cfg3_walk_1e5x1e3", w.ModelKind.Walk, dict(replications=100_000, steps=1000, chunks=30)),
            ("cfg4_pi_1e7x1e3", w.ModelKind.Pi, dict(replications=R_CFG4, draws=1000)),
            ("cfg4_mm1_1e7x1e3", w.ModelKind.Mm1, dict(replications=R_CFG4, clients=1000)),
            ("cfg4_walk_1e7x1e3", w.ModelKind.Walk, dict(replications=R_CFG4, steps=1000, chunks=30))]
    for name, m, kw in cfgs:
        pp = w.ModelParams(**kw)
        extras[name] = {}
        variants = [("wlp", w.ExecutionMode.Wlp, 0, 0), ("tlp", w.ExecutionMode.Tlp, 0, 0)]
        if m == w.ModelKind.Pi and pp.replications >= 1_000_000:
            # the whole-warp pipeline (32 lanes per replication) beside the automatic choice
            variants += [("wlp_whole_warp_pipeline", w.ExecutionMode.Wlp, 2, 0)]
        if m == w.ModelKind.Walk:
            # the walk's other kernels: per-replication WLP (lane jumps /
            # pipeline) and the bitsliced TLP (thread per 32 replications)
            variants += [("wlp_per_replication", w.ExecutionMode.Wlp, 2 if pp.replications >= 1_000_000 else 1, 0),
                         ("tlp_bitsliced", w.ExecutionMode.Tlp, 0, 2)]
        for label, md, wv, tv in variants:
            lanes = 32 if label == "wlp_whole_warp_pipeline" else 0
            with w.wlp_variant(wv), w.tlp_variant(tv), w.pipe_lanes(lanes):
                r = model_rate(w, m, pp, md)
            units_ = pp.replications * pp.units(m)
            rl = roofline_of(int(m), r["kernel"], units_, r["kernel_ms"], sms, fmax,
                             capture=f"{name[:4]}_{w.model_name(m)}_{label}")
            r[{"issue": "issue_frac", "alu_pipe": "alu_frac", "fp64_pipe": "fp64_frac"}[rl["bound"]]] = rl["frac"]
            extras[name][label] = r
    # measured warp-execution evidence (paper Table 1 / Fig. 7 analogue): divergence events
    # with the reference's definition and global memory warp-instructions, from the
    # instrumented kernels (outputs identical; counters cost a little speed)
    for name, m, kw in [("cfg3_walk_1e5x1e3", w.ModelKind.Walk, dict(replications=100_000, steps=1000, chunks=30)),
                        ("cfg4_mm1_1e7x1e3", w.ModelKind.Mm1, dict(replications=1_000_000, clients=1000))]:
        table1 = {}
        with w.hw_counters():
            for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
                rr = w.run_model(m, w.ModelParams(**kw), md, master_seed=SEED)
                rep = rr.report
                table1[w.mode_name(md)] = {"kernel": w.last_kernel(), "divergence_events": rep.divergenceEvents,
                                           "mem_reads": rep.memReads, "mem_writes": rep.memWrites,
                                           "total_cycles": rep.totalCycles}
        table1["replications"] = kw["replications"]
        extras[name]["counters"] = table1
    # config 5: experimental plan, 64 factor-level sets x 30 replications, one launch
    sets = [w.ModelParams(replications=30, clients=10_000, lambda_=0.1 + 0.8 * k / 63, mu=1.0) for k in range(64)]
    seeds = [SEED + k for k in range(64)]
    hsets = [w.ModelParams(replications=30, steps=100 + 30 * k, chunks=30) for k in range(64)]
    for label, m, ss, nout in (("cfg5_plan_mm1_64x30x1e4", w.ModelKind.Mm1, sets, 3),
                               ("cfg5_plan_walk_hetero_64x30", w.ModelKind.Walk, hsets, 1)):
        extras[label] = {}
        plan = w.PlanSets(ss, seeds)  # marshalled once, as a caller re-running a plan would
        for md in (w.ExecutionMode.Wlp, w.ExecutionMode.Tlp):
            outs = [torch.empty(64 * 30, dtype=torch.float64, device="cuda") for _ in range(nout)]

            def pstep():  # (as a caller runs it: no report, so no timing events around the model)
                w.run_plan(m, plan, None, md, outs, on_device=True)

            pms = device_timed(pstep, 5, 3, 1)
            kms = []  # the model kernel's own time, from separate reported calls
            for _ in range(5):
                rep = w.SimReport()
                w.run_plan(m, plan, None, md, outs, on_device=True, report=rep)
                kms.append(rep.kernel_ms)
            extras[label][w.mode_name(md)] = {"reps_per_s": 1920 / (pms * 1e-3), "ms_per_run": pms,
                                              "kernel_ms": sum(kms[2:]) / len(kms[2:])}
    # the reference's own IR kernel (TLP walk) on the GPU IR interpreter:
    # statements issued per second, counters exact; then compiled (IR -> CUDA C++ -> NVRTC)
    from paper_1501_01405_b200 import ir

    pir = w.ModelParams(replications=20_000, steps=1000, chunks=30)
    runs = [ir.run_model(w.ModelKind.Walk, pir, w.ExecutionMode.Tlp, SEED) for _ in range(3)]
    kms = min(r.report.kernel_ms for r in runs)
    extras["ir_walk_tlp_2e4x1e3"] = {"kernel_ms": kms, "issues": runs[-1].report.issues,
                                     "divergence_events": runs[-1].report.divergenceEvents,
                                     "issues_per_s": runs[-1].report.issues / (kms * 1e-3)}
    jruns = [ir.run_model(w.ModelKind.Walk, pir, w.ExecutionMode.Tlp, SEED, jit=True) for _ in range(4)]
    jms = min(r.report.kernel_ms for r in jruns[1:])
    assert all((r.primary == runs[-1].primary).all() for r in jruns)
    extras["ir_walk_tlp_2e4x1e3"]["jit"] = {"kernel_ms": jms, "speedup_vs_interpreter": kms / jms}
    return extras


def main():
    args = parse()
    if args.dry_run:
        self_launch(args)
        dry_run(args)
        return
    if args.impl == "reference":
        # rank 0 alone times the CPU path; no GPU and no re-launch needed
        run_reference_arm(args)
        return
    self_launch(args)
    import torch

    import paper_1501_01405_b200 as w
    from paper_1501_01405_b200 import distributed as D

    world, rank, local = dist_setup(args)
    model, mode = w.ModelKind.Pi, w.ExecutionMode.Wlp
    R = R_PER_GPU * world
    p = w.ModelParams(replications=R, draws=DRAWS)
    stream = torch.cuda.current_stream().cuda_stream
    comm = D._Comm(device="cuda")
    runner = D.gpu_runner(model, p, mode, SEED, stream=stream)
    stats = D.gpu_stats(stream=stream)
    result = {}

    def step():
        result["r"] = D.run_sharded(model, R, runner, stats, comm=comm)

    clocks = Clocks(local)
    clocks.start()
    ms = device_timed(step, args.steps, args.warmup, world)
    clk = clocks.stop()
    kernel = w.last_kernel()
    kernel_avg = max_over_ranks(model_kernel_ms(D, model, p, R, stats, comm, stream), world)
    value = R / (ms * 1e-3)
    # per step: seeding + model + the statistics (one rank: pass 1, its device fold, pass 2;
    # several: pass 1 and pass 2 around the exchange)
    launches = args.steps * (5 if world == 1 else 4)
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

    # ---- roofline of the dominant kernel, named by the run itself
    peaks = measured_peaks()
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    fmax = float(peaks.get("sm_max_mhz", 1965.0))
    roofline = roofline_of(0, kernel, R_PER_GPU * DRAWS, kernel_avg, sms, fmax, capture="cfg2_pi_wlp")
    roofline["frac_at_measured_clock"] = (roofline["achieved"] / (4 * sms * clk["sm_mhz"] * 1e-3)
                                          if clk.get("sm_mhz") else None)
    roofline["hbm_gbs_output_writeout"] = (R_PER_GPU * 8 + 3 * 4 * R_PER_GPU) / (kernel_avg * 1e-3) / 1e9

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32+f64",
            "data": "synthetic (taus88 streams by random spacing from master seed 42)",
            "config": headline_config(world),
            "e2e": {"value": R / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 64 * world,
                    "d2h_bytes_per_step": R * 8, "ms_per_step": e2e_ms,
                    "note": "inputs are (master seed, params) by value; outputs D2H to pinned host"},
            "gpu_launches": launches, "clocks": clk, "roofline": roofline,
            "result": {"mean": ci.mean, "half_width": ci.halfWidth, "n": ci.n}}

    # ---- BASELINE config 4 per model: 10^7 replications sharded over the N GPUs
    models = {}
    for name, m, kw in CFG4:
        p4 = w.ModelParams(replications=R_CFG4, **kw)
        models[name] = sharded_record(w, D, m, p4, world, comm, stats, stream, args.steps, args.warmup, sms, fmax,
                                      e2e_single_call=(world == 1 and "LOCAL_RANK" not in os.environ))
        models[name]["config"] = {"workload": f"BASELINE config 4: {name}, 1e7 replications sharded over "
                                              f"{world} GPU(s), WLP", "replications": R_CFG4, **kw,
                                  "parallelism": f"shard{world}", "scaling": "strong"}
    line["models"] = models

    if world == 1 and not args.no_extras:
        line["extras"] = extras_single_gpu(w, sms, fmax, 4 * sms * fmax * 1e-3)
    if world == 1 and rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(0, p)
        for name, m, kw in CFG4:
            models[name]["cpu_baseline"] = cpu_baseline(m, w.ModelParams(replications=R_CFG4, **kw), budget_s=5.0)
        if "extras" in line:  # the reference's host simulator beside the GPU IR interpreter
            line["cpu_baseline"]["ir_reference_simulator"] = ir_simulator_baseline()
    if rank == 0:
        print(json.dumps(line), flush=True)
    import torch.distributed as dist

    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
