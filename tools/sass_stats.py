#!/usr/bin/env python3
"""Opcode histogram of kernels in the built library (no GPU needed).

    python tools/sass_stats.py SUBSTRING [--loop]

--loop restricts to the innermost backward-branch loop with > 80 instructions (the hot
loop of the replication kernels).
"""
import re
import subprocess
import sys
from collections import Counter
from pathlib import Path

LIB = Path(__file__).resolve().parent.parent / "paper_1501_01405_b200" / "libwlp_b200.so"


def functions():
    txt = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True, check=True).stdout
    for f in re.split(r"\n\s+Function : ", txt)[1:]:
        name = f.split("\n", 1)[0]
        lines = [l for l in f.split("\n") if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
        yield name, lines


def addr(l):
    return int(re.match(r"\s+/\*([0-9a-f]+)\*/", l).group(1), 16)


def main():
    pat = sys.argv[1]
    loop = "--loop" in sys.argv
    for name, lines in functions():
        if pat not in name:
            continue
        body = lines
        if loop:
            loops = []
            for l in lines:
                m = re.search(r"BRA (0x[0-9a-f]+)", l)
                if m and int(m.group(1), 16) < addr(l):
                    loops.append((int(m.group(1), 16), addr(l)))
            inner = [x for x in loops if (x[1] - x[0]) // 16 > 80]
            if not inner:
                continue
            lo, hi = min(inner, key=lambda x: x[1] - x[0])
            body = [l for l in lines if lo <= addr(l) <= hi]
        ops = Counter()
        for l in body:
            m = re.search(r"\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", l)
            if m:
                ops[m.group(2)] += 1
        short = re.sub(r"_ZN3wlp43_GLOBAL__N__\w+?kernels_cu_[0-9a-f]+", "", name)
        print(f"{short}: {len(body)} instr  " + " ".join(f"{k}:{v}" for k, v in ops.most_common(14)))


if __name__ == "__main__":
    main()
