"""Host-side pin of the offset-Fast2Sum accumulation used by the EXACT GPU products
(dot2.cuh: dot2_step_off; symv.cu, pcg_block.cu, the EXACT entry kernels).

The scheme, emulated here step by step in IEEE binary64 (numpy float64 scalars, round
to nearest): the accumulator's high part starts at a power of two C >= 2 sum|a_k b_k|,
so at every step |s| >= C/2 >= |a_k b_k| and Fast2Sum(s, p) is error-free; TwoProd
(p, e) = (RN(ab), RN(ab - p)) is error-free (emulated with exact rationals, which is what
the hardware fma delivers).  The result RN((s - C) + c) must be the correctly rounded
sum in practice -- checked here against the exact rational sum and against Dot2 (the
oracle's scheme, Ogita-Rump-Oishi Alg. 5.3) on cancelling sums of the lengths the GPU
uses (<= 512 products per accumulator).  Also pins the two facts the argument rests on:
Fast2Sum's error term is exact under |s| >= |p|, and s - C is exact (Sterbenz)."""
from fractions import Fraction

import numpy as np

f64 = np.float64


def two_prod(a, b):
    p = f64(a * b)
    e = f64(float(Fraction(float(a)) * Fraction(float(b)) - Fraction(float(p))))  # = fma(a, b, -p)
    return p, e


def two_sum(a, b):
    s = f64(a + b)
    z = f64(s - a)
    e = f64(f64(a - f64(s - z)) + f64(b - z))
    return s, e


def fast_two_sum(a, b):
    s = f64(a + b)
    e = f64(b - f64(s - a))
    return s, e


def pow2_above(v):
    if v == 0.0:
        return f64(0.0)
    m, ex = np.frexp(v)  # v = m 2^ex, 0.5 <= m < 1 -> 2^ex > v
    return f64(np.ldexp(1.0, int(ex)))


def dot2(a, b):
    s, c = f64(0.0), f64(0.0)
    for x, y in zip(a, b):
        p, pe = two_prod(x, y)
        s, se = two_sum(s, p)
        c = f64(c + f64(pe + se))
    return f64(s + c)


def offset_dot(a, b):
    C = pow2_above(2.0 * float(np.sum(np.abs(a) * np.abs(b))) * (1 + 2 ** -50))
    s, c = C, f64(0.0)
    for x, y in zip(a, b):
        p, pe = two_prod(x, y)
        assert abs(s) >= abs(p)  # the Fast2Sum precondition the offset guarantees
        s, se = fast_two_sum(s, p)
        c = f64(c + f64(pe + se))
    d = f64(s - C)
    assert Fraction(float(d)) == Fraction(float(s)) - Fraction(float(C))  # Sterbenz: exact
    return f64(d + c)


def exact_rn(a, b):
    ex = sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b))
    return float(ex)  # Fraction -> float rounds to nearest


def test_fast_two_sum_exact_under_precondition():
    r = np.random.default_rng(1)
    for _ in range(2000):
        a = f64(r.standard_normal() * 2.0 ** r.integers(-30, 30))
        b = f64(abs(a) * r.uniform(-1.0, 1.0))  # |b| <= |a|
        s, e = fast_two_sum(a, b)
        assert Fraction(float(s)) + Fraction(float(e)) == Fraction(float(a)) + Fraction(float(b))


def test_offset_dot_is_correctly_rounded_on_cancelling_sums():
    r = np.random.default_rng(7)
    for k in (8, 32, 64, 512):
        for trial in range(12):
            a = r.uniform(0.5, 2.0, k) * np.exp(r.uniform(-0.3, 0.7, k))  # K-like positive entries
            b = r.standard_normal(k) * np.exp2(r.integers(-12, 12, k))
            if trial % 3 == 0:  # force heavy cancellation: the last term cancels the rest
                b[-1] = -float(np.dot(a[:-1], b[:-1])) / a[-1] * (1 + r.uniform(-1e-9, 1e-9))
            got = offset_dot(a, b)
            assert got == exact_rn(a, b), (k, trial)
            assert got == dot2(a, b)


def test_offset_dot_degenerate_cases():
    assert offset_dot(np.zeros(5), np.ones(5)) == 0.0
    assert offset_dot(np.ones(3), np.array([1.0, -1.0, 0.0])) == 0.0
    a = np.array([2.0 ** 500, 1.0, -(2.0 ** 500)])
    b = np.array([1.0, 2.0 ** -600, 1.0])
    assert offset_dot(a, b) == exact_rn(a, b)
