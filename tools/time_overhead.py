#!/usr/bin/env python3
"""Where a small run's time goes (run on the GPU box): whole run_shard vs its pieces.

    python tools/time_overhead.py walk 100000 1000
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

model = w.model_from_name(sys.argv[1])
R, N = int(sys.argv[2]), int(sys.argv[3])
p = w.ModelParams(replications=R, draws=N, clients=N, steps=N)
outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[model]]


def timed(label, fn, iters=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3 / iters
    print(f"{label:44s} device {e0.elapsed_time(e1) / iters:8.4f} ms   wall {wall:8.4f} ms", flush=True)


rep = w.SimReport()
timed("run_shard (report)", lambda: w.run_shard(model, p, w.ExecutionMode.Wlp, 42, 0, R, outs, on_device=True,
                                                report=rep))
print("   kernel_ms", rep.kernel_ms, w.last_kernel())
timed("run_shard (no report)", lambda: w.run_shard(model, p, w.ExecutionMode.Wlp, 42, 0, R, outs, on_device=True))
timed("run_model_into (device, CI)", lambda: w.run_model_into(model, p, w.ExecutionMode.Wlp, 42, outs, on_device=True)
      if hasattr(w, "run_model_into") else None)
seeds = torch.empty(3 * R, dtype=torch.int32, device="cuda")
timed("seed_streams_exact only", lambda: w._lib.wlp_seed_streams_exact(42, R, seeds.data_ptr(), 1, None))
timed("run_streams only (device seeds)", lambda: w._lib.wlp_run_streams(int(model), w.C.byref(w._params(p)), 2,
                                                                        seeds.data_ptr(), R, 1,
                                                                        *[o.data_ptr() for o in outs],
                                                                        *([None] * (3 - len(outs))), 1, None, None))

# the same call with every argument marshalled once (Python's share of the run)
pp = w._params(p)
o = [x.data_ptr() for x in outs] + [None] * (3 - len(outs))
sp = w._special_buffer(4096)
nsp = w.C.c_int64()
rr = w._Report()
timed("wlp_run_shard, args pre-marshalled (report)", lambda: w._lib.wlp_run_shard(
    int(model), w.C.byref(pp), 2, 42, 256, 0, R, None, 0, o[0], o[1], o[2], 1, None, sp, 4096, w.C.byref(nsp),
    w.C.byref(rr)))
timed("wlp_run_shard, args pre-marshalled (no report)", lambda: w._lib.wlp_run_shard(
    int(model), w.C.byref(pp), 2, 42, 256, 0, R, None, 0, o[0], o[1], o[2], 1, None, sp, 4096, w.C.byref(nsp),
    None))

# host-side issue cost per call (no synchronisation inside the loop: the launch queue
# absorbs the GPU work, so wall / call is the host's own overhead)
def host_cost(label, fn, iters=200):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{label:44s} host issue {(t1 - t0) * 1e3 / iters:8.4f} ms / call", flush=True)


host_cost("wlp_run_shard pre-marshalled (no report)", lambda: w._lib.wlp_run_shard(
    int(model), w.C.byref(pp), 2, 42, 256, 0, R, None, 0, o[0], o[1], o[2], 1, None, None, 0, None, None))
host_cost("wlp_run_streams pre-marshalled", lambda: w._lib.wlp_run_streams(
    int(model), w.C.byref(pp), 2, seeds.data_ptr(), R, 1, *o, 1, None, None))
host_cost("torch empty-kernel baseline (x.add_(1))", lambda: outs[0].add_(1.0))
