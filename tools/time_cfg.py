#!/usr/bin/env python3
"""Time replication kernels on the GPU box (device-resident outputs, SimReport kernel_ms).

    python tools/time_cfg.py mm1:wlp:10000000:1000 mm1:tlp:10000000:1000 walk:wlp:1000000:1000:wv=3 ...
(extra key=value fields: ModelParams fields, wv= / tv= the WLP / TLP kernel variant, pl= pipeline lanes)
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_1501_01405_b200 as w  # noqa: E402

for spec in sys.argv[1:]:
    model, mode, R, N = spec.split(":")[:4]
    extra = dict(kv.split("=") for kv in spec.split(":")[4:])
    m = w.model_from_name(model)
    R, N = int(R), int(N)
    kw = dict(replications=R, draws=N, clients=N, steps=N)
    wv, tv = int(extra.pop("wv", 0)), int(extra.pop("tv", 0))  # WLP / TLP kernel variants
    pl = int(extra.pop("pl", 0))  # pipeline lanes per replication
    for k, v in extra.items():
        kw[k] = float(v) if "." in v else int(v)
    p = w.ModelParams(**kw)
    outs = [torch.empty(R, dtype=torch.float64, device="cuda") for _ in w.OUTPUT_NAMES[m]]
    ms = []
    with w.wlp_variant(wv), w.tlp_variant(tv), w.pipe_lanes(pl):
        for i in range(4):
            rep = w.SimReport()
            w.run_shard(m, p, w.mode_from_name(mode), 42, 0, R, outs, on_device=True, report=rep)
            torch.cuda.synchronize()
            if i:
                ms.append(rep.kernel_ms)
    print(f"{spec:40s} kernel_ms min {min(ms):9.3f} med {sorted(ms)[len(ms) // 2]:9.3f}", flush=True)
