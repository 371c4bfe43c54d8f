#!/usr/bin/env python3
"""One-screen summary of a bench.py JSON line: python tools/bench_brief.py bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = d["roofline"]
print(f"headline {d['value']:.4g} {d['unit']}  {d['ms_per_step']:.3f} ms/step  kernel {r['kernel']} "
      f"{r['kernel_ms']:.3f} ms  frac {r['frac']:.3f}  e2e {d['e2e']['value']:.4g} ({d['e2e']['ms_per_step']:.3f} ms)  "
      f"launches {d['gpu_launches']}  clocks {d['clocks']}")
for m, v in d.get("models", {}).items():
    print(f"  cfg4 {m:5s} {v['kernel']:22s} run {v['ms_per_run']:8.3f}  kernel {v['roofline']['kernel_ms']:8.3f}  "
          f"{v['roofline']['bound']} {v['roofline']['frac']:.3f}  e2e {v['e2e']['ms_per_run']:8.3f}  "
          f"cpu {v.get('cpu_baseline', {}).get('value', 0):.3g}")
for k, v in d.get("extras", {}).items():
    if not k.startswith("cfg"):
        continue
    for lab, x in v.items():
        if isinstance(x, dict) and "kernel_ms" in x:
            fr = {kk: round(vv, 3) for kk, vv in x.items() if kk.endswith("frac") or kk == "run_over_kernel"}
            print(f"  {k:28s} {lab:24s} {str(x.get('kernel')):22s} run {x['ms_per_run']:8.4f}  "
                  f"kernel {x['kernel_ms']:8.4f}  {fr}")
cb = d.get("cpu_baseline", {})
print("cpu_baseline", cb.get("value"), cb.get("cores"), cb.get("kind"))
