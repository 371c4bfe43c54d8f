timeout 300 python - <<'PY'
import sys
sys.path.insert(0, ".")
import torch
import paper_1501_01405_b200 as w
for R in (16384, 32768, 65536, 131072, 262144):
    p = w.ModelParams(replications=R, clients=1000)
    outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in range(3)]
    res = {}
    for name, mode, var in (("chain", w.ExecutionMode.Wlp, 1), ("pipe", w.ExecutionMode.Wlp, 2), ("tlp", w.ExecutionMode.Tlp, 0)):
        ms = []
        with w.wlp_variant(var):
            for i in range(4):
                rep = w.SimReport()
                w.run_shard(w.ModelKind.Mm1, p, mode, 42, 0, R, outs, on_device=True, report=rep)
                if i: ms.append(rep.kernel_ms)
        res[name] = min(ms)
    print(R, {k: round(v, 4) for k, v in res.items()})
PY
