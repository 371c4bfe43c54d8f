"""The GF(2) facts the device seeding relies on, checked
independently in Python. CPU only.

1. Each taus88 component word is a linear map of its 32 bits (so n steps = M^n).
2. The map from the 88 live master-state bits to the 96 bits of three consecutive
   outputs has rank 88: distinct live states give distinct raw candidate triples.
3. Component periods are maximal (2^k - 1), so master live states at candidate starts
   3i and 3j never coincide for i != j below ~2^88 / 3.
Hence two candidate keys can only collide through the re-mapping of a component below
its minimum, i.e. only between "special" candidates (some component < 2*min).
4. taus_c2x2 (two component-2 steps as one) is exact.
"""
import random

M32 = 0xFFFFFFFF
KQS = [(31, 13, 12), (29, 2, 4), (28, 3, 17)]


def step(c, s):
    k, q, sh = KQS[c]
    mask = (M32 << (32 - k)) & M32
    b = ((((s << q) & M32) ^ s) >> (k - sh))
    return (((s & mask) << sh) & M32) ^ b


def mat_of(f):
    return [f(1 << j) for j in range(32)]


def apply(m, x):
    y = 0
    j = 0
    while x:
        if x & 1:
            y ^= m[j]
        x >>= 1
        j += 1
    return y


def mul(a, b):
    return [apply(a, b[j]) for j in range(32)]


def mpow(m, n):
    r = [1 << j for j in range(32)]
    while n:
        if n & 1:
            r = mul(m, r)
        m = mul(m, m)
        n >>= 1
    return r


def test_components_are_linear():
    rnd = random.Random(1)
    for c in range(3):
        for _ in range(200):
            a, b = rnd.getrandbits(32), rnd.getrandbits(32)
            assert step(c, a ^ b) == step(c, a) ^ step(c, b)


def test_three_outputs_are_injective_on_live_state():
    live = [range(1, 32), range(3, 32), range(4, 32)]
    basis = {}
    rank = 0
    for c in range(3):
        for b in live[c]:
            st = [0, 0, 0]
            st[c] = 1 << b
            v = 0
            for k in range(3):
                st = [step(i, st[i]) for i in range(3)]
                v |= (st[0] ^ st[1] ^ st[2]) << (32 * k)
            while v:
                h = v.bit_length() - 1
                if h in basis:
                    v ^= basis[h]
                else:
                    basis[h] = v
                    rank += 1
                    break
    assert rank == 88


def test_component_periods_are_maximal():
    factors = {31: [2**31 - 1], 29: [233, 1103, 2089], 28: [3, 5, 29, 43, 113, 127]}
    for c, (k, _, _) in enumerate(KQS):
        m = mat_of(lambda x, c=c: step(c, x))
        period = 2**k - 1
        p = mpow(m, period)
        lo = 32 - k
        live = (M32 >> lo) << lo
        # M^period acts as identity on the live bits (the low 32-k bits of a word are a
        # by-product of the last step and never feed back)
        for j in range(lo, 32):
            assert p[j] & live == 1 << j
        for f in factors[k]:
            q = mpow(m, period // f)
            assert any(q[j] & live != 1 << j for j in range(lo, 32))


def test_component2_double_step():
    rnd = random.Random(7)
    for _ in range(20000):
        s = rnd.getrandbits(32)
        two = step(1, step(1, s))
        fast = (((s & 0xFFFFFFF8) << 8) & M32) ^ (((((s << 2) & M32) ^ s)) >> 21)
        assert two == fast
