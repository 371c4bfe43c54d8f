#!/usr/bin/env python3
"""Golden fixtures of the kernel-IR path, produced by the REFERENCE (oracle/_ref: the
reference sources compiled unmodified) in this container, for tests that must run where
/root/reference is absent (the GPU box).

    python tools/gen_ir_golden.py

Writes tests/golden/ir/:
  <model>_<body|tlp|wlp>.sexp  dump_kernel of build_model_body / wrap_tlp / wrap_wlp
  corpus.json                  per tests/ir_corpus.py case: the reference simulator's
                               final arrays (hex doubles) and SimReport counters; per
                               fault case: the reference's error message
  models.json                  run_model(Tlp / Wlp) SimReport counters of the bundled models
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from ir_corpus import CASES, FAULTS, fresh_arrays, streams_for  # noqa: E402

OUT = ROOT / "tests" / "golden" / "ir"
KEYS = ("issues", "aluIssues", "memReads", "memWrites", "divergenceEvents")
MODEL_RUNS = [(m, mode, kw, blk) for m in range(3) for mode in (1, 2) for kw, blk in [
    (dict(replications=1, draws=20, clients=20, steps=20, chunks=5), 256),
    (dict(replications=37, draws=50, clients=40, steps=60, chunks=7), 256),
    (dict(replications=70, draws=30, clients=30, steps=30, chunks=30, lambda_=0.9, mu=1.0), 48),
    (dict(replications=33, draws=64, clients=64, steps=64, chunks=3, lambda_=1.5, mu=1.0), 20),
]]


def main():
    ref = oracle.Oracle("reference")
    OUT.mkdir(parents=True, exist_ok=True)
    names = {0: "pi", 1: "mm1", 2: "walk"}
    for m in range(3):
        for mode, tag in ((0, "body"), (1, "tlp"), (2, "wlp")):
            (OUT / f"{names[m]}_{tag}.sexp").write_text(ref.ir_model_text(m, mode))
    corpus = {}
    for name, c in CASES.items():
        arrays = fresh_arrays(c)
        rep = ref.ir_simulate(c["text"], c["cfg"], c["scalars"], arrays, streams_for(c), c["mask_depth"])
        corpus[name] = {"arrays": {k: [float(x).hex() for x in v] for k, v in arrays.items()},
                        "report": {k: rep[k] for k in KEYS}}
    faults = {}
    for name, (text, _) in FAULTS.items():
        depth = 3 if name == "mask_stack" else 32
        try:
            ref.ir_simulate(text, (32, 1, 1, 1, 1, 32), {}, {"o": np.zeros(4)}, None, depth)
            faults[name] = None
        except oracle.OracleError as e:
            faults[name] = {"code": e.code, "message": str(e).split("] ", 1)[1]}
    (OUT / "corpus.json").write_text(json.dumps({"cases": corpus, "faults": faults}, indent=1) + "\n")
    runs = []
    for m, mode, kw, blk in MODEL_RUNS:
        rep = ref.run_model_report(m, oracle.params(**kw), 42, mode, blk)
        runs.append({"model": m, "mode": mode, "params": kw, "tlp_block": blk, "seed": 42,
                     "report": {k: rep[k] for k in KEYS}})
    (OUT / "models.json").write_text(json.dumps(runs, indent=1) + "\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
