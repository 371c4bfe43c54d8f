import sys, torch
sys.path.insert(0, '.')
import paper_1501_01405_b200 as w
m = w.model_from_name(sys.argv[1]); R, N = int(sys.argv[2]), int(sys.argv[3])
p = w.ModelParams(replications=R, draws=N, clients=N, steps=N)
outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[m]]
for _ in range(3):
    w.run_shard(m, p, w.ExecutionMode.Wlp, 42, 0, R, outs, on_device=True, report=w.SimReport())
torch.cuda.synchronize()
