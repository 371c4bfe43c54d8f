import sys, time
sys.path.insert(0, '.')
import torch, numpy as np
import paper_1501_01405_b200 as w
for name, m, kw in [("pi", 0, dict(replications=10_000_000, draws=1000)), ("mm1", 1, dict(replications=10_000_000, clients=1000)),
                    ("walk", 2, dict(replications=10_000_000, steps=1000, chunks=30)), ("pi2", 0, dict(replications=1_000_000, draws=10_000))]:
    p = w.ModelParams(**kw)
    names = w.OUTPUT_NAMES[w.ModelKind(m)]
    host = [torch.empty(p.replications, dtype=torch.float64, pin_memory=True) for _ in names]
    pg = [np.empty(p.replications) for _ in names]
    for label, outs in (("pinned", [h.numpy() for h in host]), ("pageable", pg)):
        for _ in range(2):
            w.run_model_into(w.ModelKind(m), p, w.ExecutionMode.Wlp, 42, outs, on_device=False, ci_level=0.95)
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            w.run_model_into(w.ModelKind(m), p, w.ExecutionMode.Wlp, 42, outs, on_device=False, ci_level=0.95)
            ts.append(time.perf_counter() - t0)
        print(name, label, "e2e ms", round(min(ts) * 1e3, 3), flush=True)
