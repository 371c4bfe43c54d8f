timeout 300 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
import paper_1501_01405_b200 as w
from paper_1501_01405_b200 import ir
for R in (20000, 200000):
    p = w.ModelParams(replications=R, steps=1000, chunks=30)
    t0 = time.time(); a = ir.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, 42, jit=True); t1 = time.time()
    b = ir.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, 42, jit=True)
    c = ir.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, 42)
    hand = w.run_model(w.ModelKind.Walk, p, w.ExecutionMode.Tlp, master_seed=42)
    print(R, "jit first call %.2fs" % (t1 - t0), "jit ms", b.report.kernel_ms, "interp ms", c.report.kernel_ms,
          "hand TLP ms", hand.report.kernel_ms, (a.primary == c.primary).all() and (b.primary == hand.primary).all())
for m in (0, 1):
    p = w.ModelParams(replications=200000, draws=1000, clients=1000)
    b = ir.run_model(w.ModelKind(m), p, w.ExecutionMode.Tlp, 42, jit=True)
    b = ir.run_model(w.ModelKind(m), p, w.ExecutionMode.Tlp, 42, jit=True)
    hand = w.run_model(w.ModelKind(m), p, w.ExecutionMode.Tlp, master_seed=42)
    print("model", m, "jit ms", b.report.kernel_ms, "hand TLP ms", hand.report.kernel_ms,
          all((b.outputs[k] == hand.outputs[k]).all() for k in b.outputs))
PY
