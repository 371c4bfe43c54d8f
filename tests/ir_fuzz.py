"""Random kernel-IR programs for differential tests of the GPU interpreter / JIT against
the reference simulator (tests/test_ir_fuzz_gpu.py).

Programs use every operator with int / real operands, draws, special registers, loads,
stores, nested ifs, bounded while loops and halts. Each thread owns SLOTS elements of
`out`; the lanes of one IR warp share one element of `w` (conflicting stores resolved in
lane order, read back by the same warp). They avoid what the two sides cannot agree on
by design: memory shared between IR warps (the reference runs warps one after another,
the GPU concurrently) and INT64_MIN / -1 (undefined behaviour; x86 traps). Faults
(division by zero, log of a non-positive value, floor overflow, a real index) are allowed:
both sides must then fault."""
import random

import numpy as np

BIN = ["add", "sub", "mul", "div", "mod", "lt", "le", "gt", "ge", "eq", "ne", "and", "or"]
UN = ["neg", "log", "floor"]
SREG = ["tid.x", "tid.y", "tid.z", "bid.x", "bid.y", "bdim.x", "bdim.y", "bdim.z", "gdim.x", "gdim.y", "warpsize"]
INTS = ["i0", "i1", "i2"]
REALS = ["r0", "r1", "r2"]
SLOTS = 5  # elements of `out` per thread
GEOMS = [(32, 1, 1), (16, 2, 1), (8, 2, 3), (50, 1, 1), (7, 3, 1), (64, 1, 1)]
GRIDS = [(1, 1), (2, 1), (2, 2), (3, 1)]


class Gen:
    def __init__(self, seed):
        self.r = random.Random(seed)

    def leaf(self):
        k = self.r.random()
        if k < 0.2:
            return str(self.r.randint(-9, 9))
        if k < 0.4:
            return repr(self.r.choice([0.5, -1.25, 3.0, 0.1, 2.0, -0.0, 1e10, 7.5, 1e300]))
        if k < 0.55:
            return self.r.choice(INTS + ["k1", "k2", "k3"])
        if k < 0.7:
            return self.r.choice(REALS)
        if k < 0.8:
            return self.r.choice(["n", "a", "g"])
        if k < 0.9:
            return self.r.choice(SREG)
        return "(draw)"

    def expr(self, depth=3):
        if depth == 0 or self.r.random() < 0.3:
            return self.leaf()
        if self.r.random() < 0.2:
            op = self.r.choice(UN)
            inner = self.expr(depth - 1)
            if op == "log" and self.r.random() < 0.9:  # mostly positive arguments
                inner = f"(add (mul {inner} {inner}) 0.5)"
            return f"({op} {inner})"
        op = self.r.choice(BIN)
        b = self.expr(depth - 1)
        if op in ("div", "mod") and self.r.random() < 0.85:  # mostly non-zero divisors
            b = f"(add (mul {b} {b}) 1)"
        return f"({op} {self.expr(depth - 1)} {b})"

    def int_expr(self, depth=2):
        k = self.r.random()
        if k < 0.6:
            return f"(floor {self.expr(depth)})"
        if k < 0.8:
            return f"(add {self.r.choice(INTS)} {self.r.randint(-2, 3)})"
        return self.r.choice(SREG + ["g", "n"])

    def index(self, m):
        """An int in [0, m) (a real operand makes the index real: a fault on both sides)."""
        x = self.int_expr() if self.r.random() < 0.97 else self.expr(1)
        return f"(mod (add (mod {x} {m}) {m}) {m})"

    def stmts(self, depth, n):
        return "\n".join(self.stmt(depth) for _ in range(n))

    def stmt(self, depth):
        k = self.r.random()
        if k < 0.22:
            return f"(assign {self.r.choice(REALS)} {self.expr()})"
        if k < 0.34:
            return f"(assign {self.r.choice(INTS)} {self.int_expr()})"
        if k < 0.48:
            return f"(store out (add (mul g {SLOTS}) {self.index(SLOTS)}) {self.expr()})"
        if k < 0.54:
            return f"(store w wid {self.expr()})"
        if k < 0.6:
            return f"(load {self.r.choice(REALS)} buf {self.index(16)})"
        if k < 0.64:
            return f"(load {self.r.choice(REALS)} out (add (mul g {SLOTS}) {self.index(SLOTS)}))"
        if k < 0.67:
            return f"(load {self.r.choice(REALS)} w wid)"
        if k < 0.82 and depth > 0:
            s = f"(if {self.expr(2)}\n(then {self.stmts(depth - 1, self.r.randint(0, 3))})"
            if self.r.random() < 0.6:
                s += f"\n(else {self.stmts(depth - 1, self.r.randint(0, 3))})"
            return s + ")"
        if k < 0.94 and depth > 0:  # k<depth> is assigned by nothing else: the loop ends
            c = f"k{depth}"
            bound = self.r.choice([str(self.r.randint(1, 6)), f"(add (mod tid.x 4) 1)",
                                   f"(floor (mul (draw) 5))"])
            return (f"(assign {c} 0)\n(while (lt {c} {bound})\n{self.stmts(depth - 1, self.r.randint(0, 3))}\n"
                    f"(assign {c} (add {c} 1)))")
        if self.r.random() < 0.3:
            return "(if (lt (draw) 0.05) (then (halt)))"
        return f"(assign {self.r.choice(REALS)} (draw))"

    def case(self):
        bx, by, bz = self.r.choice(GEOMS)
        gx, gy = self.r.choice(GRIDS)
        ws = self.r.choice([32, 32, 16, 8, 5])
        tpb = bx * by * bz
        wpb = (tpb + ws - 1) // ws
        threads = tpb * gx * gy
        body = self.stmts(3, self.r.randint(3, 10))
        text = f"""(kernel
  (param n int) (param a real) (param wpb int) (param out array) (param w array) (param buf array)
  (local g int) (local wid int) (local i0 int) (local i1 int) (local i2 int)
  (local k1 int) (local k2 int) (local k3 int) (local r0 real) (local r1 real) (local r2 real)
  (body
    (assign g (add tid.x (mul bdim.x (add tid.y (mul bdim.y (add tid.z (mul bdim.z (add bid.x (mul gdim.x bid.y)))))))))
    (assign wid (add (div (add tid.x (mul bdim.x (add tid.y (mul bdim.y tid.z)))) warpsize) (mul wpb (add bid.x (mul gdim.x bid.y)))))
    {body}))"""
        seed = self.r.getrandbits(32)
        rng = np.random.default_rng(seed)
        st = rng.integers(0, 2**32, size=(3, threads), dtype=np.uint64).astype(np.uint32)
        st[0] |= 2
        st[1] |= 8
        st[2] |= 16
        arrays = {"out": np.zeros(threads * SLOTS), "w": np.zeros(wpb * gx * gy),
                  "buf": rng.standard_normal(16) * 4}
        scalars = {"n": self.r.randint(-5, 50), "a": self.r.choice([0.25, -3.5, 1e-3, 17.0]), "wpb": wpb}
        return dict(text=text, cfg=(bx, by, bz, gx, gy, ws), scalars=scalars, arrays=arrays, streams=st)
