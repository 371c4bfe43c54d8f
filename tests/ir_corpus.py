"""Kernel-IR corpus for the GPU interpreter's parity tests (tests/test_ir_*.py).

Each case: kernel text (kernel_text.hpp form), launch (bx, by, bz, gx, gy, warpSize),
scalar params, array params (name -> initial float64 values) and a lane-stream seed (None:
every lane keeps the default RngState). The cases exercise the reference simulator's rules
(warp_exec.cpp:178-298) one by one: divergence and its event definition, then-before-else,
loop masks, halts, partial warps, odd warp sizes, 2-D/3-D geometry, conflicting stores,
every operator with int/real promotion, and the faults. IR warps of different blocks run
concurrently on the GPU, so no case lets two blocks write one element."""
import numpy as np

CASES = {}


def case(name, text, cfg, scalars=None, arrays=None, seed=None, mask_depth=32):
    CASES[name] = dict(text=text, cfg=cfg, scalars=scalars or {}, arrays=arrays or {}, seed=seed,
                       mask_depth=mask_depth)


def streams_for(c):
    """(3, n) uint32 lane streams, one per launch thread, from the case seed (None: none)."""
    if c["seed"] is None:
        return None
    bx, by, bz, gx, gy, _ = c["cfg"]
    n = bx * by * bz * gx * gy
    rng = np.random.default_rng(c["seed"])
    s = rng.integers(0, 2**32, size=(3, n), dtype=np.uint64).astype(np.uint32)
    s[0] |= 2  # keep components above their minimums (make_rng_state would re-map them)
    s[1] |= 8
    s[2] |= 16
    return s


def fresh_arrays(c):
    return {k: np.array(v, dtype=np.float64) for k, v in c["arrays"].items()}


# --- geometry and special registers ----------------------------------------------------
case("sregs_3d", """(kernel
  (param out array)
  (local g int)
  (body
    (assign g (add tid.x (mul bdim.x (add tid.y (mul bdim.y (add tid.z (mul bdim.z (add bid.x (mul gdim.x bid.y)))))))))
    (store out g (add (mul 1000.0 bid.y) (add (mul 100 bid.x) (add (mul 10 tid.z) (add (mul 3 tid.y) (add tid.x (mul warpsize 0.5)))))))))
""", (4, 3, 2, 3, 2, 8), arrays={"out": np.full(144, -1.0)})

case("partial_warps", """(kernel
  (param out array) (param n int)
  (local g int)
  (body
    (assign g (add tid.x (mul bdim.x bid.x)))
    (if (lt g n) (then (store out g (mul 2 g))))))
""", (50, 1, 1, 3, 1, 32), scalars={"n": 140}, arrays={"out": np.zeros(150)})

case("warpsize_8_and_1", """(kernel
  (param out array)
  (local g int) (local u real)
  (body
    (assign g (add tid.x (mul bdim.x bid.x)))
    (assign u (draw))
    (if (lt u 0.5) (then (store out g u)) (else (store out g (neg u))))))
""", (13, 1, 1, 2, 1, 8), arrays={"out": np.zeros(26)}, seed=3)

case("warpsize_1", """(kernel
  (param out array)
  (local g int) (local u real) (local k int)
  (body
    (assign g (add tid.x (mul bdim.x bid.x)))
    (while (lt k 5)
      (assign u (draw))
      (if (gt u 0.3) (then (assign k (add k 1))) (else (assign k (add k 2)))))
    (store out g (add u k))))
""", (3, 1, 1, 2, 1, 1), arrays={"out": np.zeros(6)}, seed=5)

# --- control flow -----------------------------------------------------------------------
case("divergent_if_then_before_else", """(kernel
  (param out array)
  (local x int)
  (body
    (assign x tid.x)
    (if (lt x 4)
      (then
        (assign x (add x 10))
        (if (lt x 12) (then (assign x (mul x 2))))
        (assign x (add x 1)))
      (else (halt)))
    (assign x (add x 100))
    (store out tid.x x)))
""", (8, 1, 1, 1, 1, 8), arrays={"out": np.full(8, -1.0)})

case("uniform_and_empty_sides", """(kernel
  (param out array)
  (local x int)
  (body
    (assign x tid.x)
    (if (lt x 0) (then (assign x -1)) (else (assign x (add x 5))))
    (if (ge x 0) (then (assign x (add x 1))))
    (if (lt x 7) (then) (else (assign x (mul x 3))))
    (store out (add tid.x (mul bdim.x bid.x)) x)))
""", (32, 1, 1, 2, 1, 32), arrays={"out": np.zeros(64)})

case("while_shrinking_masks", """(kernel
  (param out array)
  (local x int) (local n int)
  (body
    (assign x tid.x)
    (while (lt x 40)
      (assign x (add x (add 1 (mod tid.x 3))))
      (assign n (add n 1)))
    (store out tid.x (add (mul 1000 n) x))))
""", (32, 1, 1, 1, 1, 32), arrays={"out": np.zeros(32)})

case("halts_inside_loops", """(kernel
  (param out array)
  (local x int) (local u real) (local g int)
  (body
    (assign g (add tid.x (mul bdim.x bid.x)))
    (assign x 0)
    (while (lt x 20)
      (assign u (draw))
      (if (lt u 0.05) (then (store out g (neg x)) (halt)))
      (assign x (add x 1)))
    (store out g x)))
""", (64, 1, 1, 2, 1, 32), arrays={"out": np.zeros(128)}, seed=11)

case("nested_loops_and_branches", """(kernel
  (param acc array) (param rounds int)
  (local i int) (local j int) (local u real) (local s real)
  (body
    (while (lt i rounds)
      (assign j 0)
      (while (lt j (add 1 (mod (add tid.x i) 4)))
        (assign u (draw))
        (if (lt u 0.25)
          (then (assign s (add s u)))
          (else (if (lt u 0.5) (then (assign s (sub s u))) (else (assign s (mul s 1.5))))))
        (assign j (add j 1)))
      (assign i (add i 1)))
    (store acc (add tid.x (mul bdim.x bid.x)) s)))
""", (48, 1, 1, 3, 1, 32), scalars={"rounds": 6}, arrays={"acc": np.zeros(144)}, seed=17)

case("empty_loop_body_and_if_with_no_work", """(kernel
  (param out array)
  (local x int)
  (body
    (while (lt x 0))
    (if (eq tid.x 3) (then))
    (store out tid.x 1.0)))
""", (8, 1, 1, 1, 1, 8), arrays={"out": np.zeros(8)})

# --- memory -----------------------------------------------------------------------------
case("conflicting_stores_ascending_lane", """(kernel
  (param out array) (param cnt array)
  (local c real)
  (body
    (store out 0 tid.x)
    (store out (mod tid.x 3) (add 100 tid.x))
    (load c cnt 0)
    (store cnt 0 (add c 1.0))))
""", (32, 1, 1, 1, 1, 32), arrays={"out": np.zeros(4), "cnt": np.zeros(1)})

case("load_after_store_in_warp", """(kernel
  (param buf array) (param out array)
  (local v real)
  (body
    (store buf tid.x (mul tid.x tid.x))
    (load v buf (mod (add tid.x 1) bdim.x))
    (store out tid.x v)))
""", (16, 1, 1, 1, 1, 16), arrays={"buf": np.zeros(16), "out": np.zeros(16)})

# --- arithmetic -------------------------------------------------------------------------
case("int_arithmetic_truncation", """(kernel
  (param out array)
  (local a int) (local b int)
  (body
    (assign a (sub tid.x 7))
    (assign b (sub 3 (mod tid.x 5)))
    (if (ne b 0)
      (then
        (store out (mul 4 tid.x) (div a b))
        (store out (add 1 (mul 4 tid.x)) (mod a b))))
    (store out (add 2 (mul 4 tid.x)) (mul a (neg b)))
    (store out (add 3 (mul 4 tid.x)) (add (mul a 1000000000000) b))))
""", (16, 1, 1, 1, 1, 16), arrays={"out": np.zeros(64)})

case("real_ops_and_promotion", """(kernel
  (param out array) (param scale real)
  (local x real) (local k int) (local u real)
  (body
    (assign u (draw))
    (assign x (add (mul u scale) tid.x))
    (assign k (floor (mul x 3.0)))
    (store out (mul 8 tid.x) x)
    (store out (add 1 (mul 8 tid.x)) k)
    (store out (add 2 (mul 8 tid.x)) (mod (sub x 5) 2.5))
    (store out (add 3 (mul 8 tid.x)) (div x (add tid.x 3)))
    (store out (add 4 (mul 8 tid.x)) (log (add x 0.001)))
    (store out (add 5 (mul 8 tid.x)) (neg (floor (neg x))))
    (store out (add 6 (mul 8 tid.x)) (and (gt x 2) (le u 0.5)))
    (store out (add 7 (mul 8 tid.x)) (or (eq k 2) (ne x x)))))
""", (32, 1, 1, 1, 1, 32), scalars={"scale": 2.5}, arrays={"out": np.zeros(256)}, seed=23)

case("comparisons_with_nan_and_signed_zero", """(kernel
  (param out array)
  (local nan real) (local nz real) (local inf real)
  (body
    (assign inf (mul 1e308 10.0))
    (assign nan (sub inf inf))
    (assign nz (neg 0.0))
    (store out 0 (lt nan 1.0))
    (store out 1 (le nan 1.0))
    (store out 2 (gt nan 1.0))
    (store out 3 (ge nan 1.0))
    (store out 4 (eq nan nan))
    (store out 5 (ne nan nan))
    (store out 6 (and nan 1))
    (store out 7 (or 0.0 nz))
    (store out 8 nz)
    (store out 9 (eq nz 0))
    (store out 10 (mul nz 1))
    (store out 11 (floor -2.5))
    (store out 12 (floor 7))
    (store out 13 (mod -7.5 2.0))
    (store out 14 (div 1 3))
    (store out 15 (div 1.0 3))))
""", (1, 1, 1, 1, 1, 32), arrays={"out": np.zeros(16)})

case("int_local_from_real_via_floor_and_literals", """(kernel
  (param out array)
  (local k int) (local r real)
  (body
    (assign k (floor 1e3))
    (assign r k)
    (assign r (add r 1.5e-3))
    (assign k (add k -42))
    (store out 0 k)
    (store out 1 r)
    (store out 2 (mul 0.1 3))))
""", (1, 1, 1, 1, 1, 1), arrays={"out": np.zeros(3)})

# --- the paper's models, hand-written user-style (not the bundled bodies) -------------------
case("user_pi_tlp_counts_in_registers", """(kernel
  ; a user-defined pi kernel: thread per replication, hit count in a register
  (param replications int) (param draws int) (param out array)
  (local rid int) (local i int) (local x real) (local y real) (local c real)
  (body
    (assign rid (add tid.x (mul bdim.x bid.x)))
    (if (lt rid replications)
      (then
        (while (lt i draws)
          (assign x (draw))
          (assign y (draw))
          (assign c (add c (le (add (mul x x) (mul y y)) 1.0)))
          (assign i (add i 1)))
        (store out rid (div (mul 4.0 c) draws))))))
""", (64, 1, 1, 3, 1, 32), scalars={"replications": 150, "draws": 200}, arrays={"out": np.zeros(150)}, seed=42)

FAULTS = {
    "int_div_zero": ("(kernel (param o array) (local a int) (body (assign a (div 1 (sub tid.x 3)))))", "integer division by zero"),
    "real_div_zero": ("(kernel (param o array) (local a real) (body (assign a (div 1.0 (sub tid.x 3.0)))))", "division by zero"),
    "int_mod_zero": ("(kernel (param o array) (local a int) (body (assign a (mod 5 (sub tid.x 1)))))", "integer modulo by zero"),
    "real_mod_zero": ("(kernel (param o array) (local a real) (body (assign a (mod 5.5 (sub tid.x 1.0)))))", "modulo by zero"),
    "log_zero": ("(kernel (param o array) (local a real) (body (assign a (log tid.x))))", "log of a non-positive value"),
    "floor_range": ("(kernel (param o array) (local a int) (body (assign a (floor (mul 1e300 (add tid.x 1.0))))))",
                    "floor result outside the integer range"),
    "load_oob": ("(kernel (param o array) (local a real) (body (load a o (add tid.x 2))))", "out of bounds"),
    "store_oob": ("(kernel (param o array) (body (store o (sub tid.x 1) 1.0)))", "out of bounds"),
    "load_real_index": ("(kernel (param o array) (local a real) (body (load a o 0.0)))", "non-integer index"),
    "store_real_index": ("(kernel (param o array) (body (store o 1.5 1.0)))", "non-integer index"),
    "real_into_int": ("(kernel (param o array) (local a int) (body (if (eq tid.x 5) (then (assign a 0.5)))))",
                      "real value into int local 'a'"),
    "mask_stack": ("(kernel (param o array) (local a int) (body (if (lt tid.x 9) (then (if (lt tid.x 8) (then "
                   "(if (lt tid.x 7) (then (assign a 1)))))))))", "mask stack overflow"),
}
