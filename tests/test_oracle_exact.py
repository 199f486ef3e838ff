"""Pins of the oracle's exact-arithmetic pieces (oracle/laker_oracle.c) against
things other than itself: the paper's worked example (tests/golden), exact
rational arithmetic (fractions), a 200-bit decimal exp, closed forms and
special cases.  CPU only."""
import decimal
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_example.json")))


def exp_ref(x: float) -> float:
    """Correctly rounded exp via 60-digit decimal (independent of libquadmath)."""
    with decimal.localcontext() as ctx:
        ctx.prec = 60
        return float(decimal.Decimal(x).exp())


def dot_ref(x, y) -> float:
    """Exact rational dot product, rounded once to binary64."""
    return float(sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y)))


def entry_ref(ei, ej, scale) -> float:
    """Reading R18: K_ij = RN(exp(RN(scale * RN(<e_i, e_j>))))."""
    return exp_ref(float(scale) * dot_ref(ei, ej))


# ------------------------------------------------------------- exp and Dot2
def test_exp_cr_matches_decimal():
    r = np.random.default_rng(1)
    xs = np.concatenate([r.uniform(-1, 1, 3000), r.uniform(-700, 700, 500),
                         r.uniform(-1e-6, 1e-6, 200), [0.0, 1.0, -1.0, 0.5, 709.0, -708.0]])
    bad = [x for x in xs if O.exp_cr(x) != exp_ref(x)]
    assert not bad, bad[:5]


def test_dot2_is_correctly_rounded_on_ill_conditioned_dots():
    """Dot2 result = RN(exact) up to u*|s| + gamma_n^2 cond |s| (Ogita-Rump-Oishi
    Prop. 5.5); at cond ~1e8 and n = 200 that is RN in practice."""
    r = np.random.default_rng(2)
    ok = 0
    for t in range(200):
        n = 200
        x = r.standard_normal(n) * np.exp(r.uniform(-20, 20, n))
        y = r.standard_normal(n)
        # make it cancel: last term nearly cancels the rest
        s = float(np.dot(x[:-1], y[:-1]))
        y[-1] = 1.0
        x[-1] = -s * (1 + 1e-9 * r.standard_normal())
        got, ref = O.dot2(x, y), dot_ref(x, y)
        ok += got == ref
        assert abs(got - ref) <= 2 * np.spacing(abs(ref)) + 1e-300
    assert ok >= 198


# ----------------------------------------------------- worked example
def test_worked_example_kernel_T1():
    E = np.array(GOLD["E"])
    K, nov = O.assemble(E, 1.0)
    assert nov == 0
    assert np.abs(K - np.array(GOLD["G"])).max() <= GOLD["tol"]["G"]
    lamI = K + GOLD["lam"] * np.eye(3)
    assert np.abs(lamI - np.array(GOLD["lamI_plus_G"])).max() <= GOLD["tol"]["G"]
    for i in range(3):
        for j in range(3):
            assert K[i, j] == entry_ref(E[i], E[j], 1.0)


def _exact_solve3(A, y):
    """Gaussian elimination in rationals."""
    M = [[Fraction(float(A[i][j])) for j in range(3)] + [Fraction(float(y[i]))] for i in range(3)]
    for c in range(3):
        for r_ in range(c + 1, 3):
            f = M[r_][c] / M[c][c]
            M[r_] = [a - f * b for a, b in zip(M[r_], M[c])]
    x = [Fraction(0)] * 3
    for i in (2, 1, 0):
        x[i] = (M[i][3] - sum(M[i][j] * x[j] for j in range(i + 1, 3))) / M[i][i]
    return np.array([float(v) for v in x])


def test_worked_example_alpha_T3():
    E, y, lam = np.array(GOLD["E"]), np.array(GOLD["y"]), GOLD["lam"]
    K, _ = O.assemble(E, 1.0)
    alpha, rep = O.pcg(K, lam, y, O.P_NONE, tol=1e-13)
    assert rep.termination == O.TERM_RESIDUAL_TOL
    assert rep.iters <= 3 + 1          # CG finite termination at n = 3 (one extra in fp64 allowed)
    assert np.abs(alpha - np.array(GOLD["alpha"])).max() <= GOLD["tol"]["alpha"]
    exact = _exact_solve3(K + lam * np.eye(3), y)
    assert np.abs(alpha - exact).max() <= 1e-12 * np.abs(exact).max()
    assert np.allclose(O.reference_solve(K, lam, y), exact, rtol=1e-12, atol=0)


def test_worked_example_cross_kernel_and_prediction_T2_T4():
    E, y, lam = np.array(GOLD["E"]), np.array(GOLD["y"]), GOLD["lam"]
    es = np.array(GOLD["e_star"])[None, :]
    kx = O.cross_kernel(es, E, 1.0)[0]
    assert np.abs(kx - np.array(GOLD["cross"])).max() <= GOLD["tol"]["cross"]
    K, _ = O.assemble(E, 1.0)
    alpha = _exact_solve3(K + lam * np.eye(3), y)
    r_hat = O.predict(es, E, 1.0, alpha)[0]
    assert abs(r_hat - GOLD["r_hat"]) <= GOLD["tol"]["r_hat"]
    assert r_hat == dot_ref(kx, alpha)


# ------------------------------------------------------ special cases
def test_kernel_special_cases_T6():
    K, _ = O.assemble(np.zeros((5, 3)), 0.7)
    assert (K == 1.0).all()
    K, _ = O.assemble(np.array([[0.6, 0.8]]), 1.0)
    assert K[0, 0] == exp_ref(0.6 * 0.6 + 0.8 * 0.8) and abs(K[0, 0] - math.e) < 1e-15
    r = np.random.default_rng(3)
    E = r.standard_normal((7, 4)) * 0.3
    K, _ = O.assemble(E, 0.5)
    assert (O.cross_kernel(E[2:3], E, 0.5)[0] == K[2]).all()      # query = training point -> row i


def test_kernel_entries_bitwise_vs_rational_reference():
    r = np.random.default_rng(4)
    E = r.standard_normal((40, 16)) * 0.4
    scale = 1.0 / math.sqrt(32.0)   # not a power of two: exercises the RN(scale * dot) rounding
    K, _ = O.assemble(E, scale)
    for (i, j) in [(0, 0), (0, 39), (39, 0), (5, 17), (17, 5), (38, 39), (20, 20)]:
        assert K[i, j] == entry_ref(E[i], E[j], scale)
    assert (K == K.T).all()
    Kr = O.assemble_rows(E, scale, 8, 13)
    assert (Kr == K[8:13]).all()


def test_kernel_symmetric_psd_T5():
    from synth import make_problem
    P = make_problem(1)
    K, nov = O.assemble(P.E, P.scale)
    assert nov == 0 and (K == K.T).all() and (K > 0).all()
    np.linalg.cholesky(K + P.lam * np.eye(P.n))
    w = np.linalg.eigvalsh(K)
    assert w[0] > -1e-12 * w[-1]        # PSD up to rounding (Schur product theorem, R2)


def test_overflow_is_counted():
    E = np.array([[30.0, 0.0], [0.0, 1.0]])
    _, nov = O.assemble(E, 1.0)   # 900 > 709.78
    assert nov == 1


def test_apply_bitwise_vs_rational_reference():
    r = np.random.default_rng(5)
    n = 48
    K = np.exp(0.3 * r.standard_normal((n, n)))
    p = r.standard_normal(n) * np.exp(r.uniform(-5, 5, n))
    lam = 1e-4
    q = O.apply(K, lam, p)
    for i in range(n):
        ref = float(Fraction(lam) * Fraction(float(p[i])) +
                    sum(Fraction(float(K[i, j])) * Fraction(float(p[j])) for j in range(n)))
        assert q[i] == ref


def test_predict_matches_exact_on_small_case():
    r = np.random.default_rng(6)
    E = r.standard_normal((30, 8)) * 0.3
    Eq = r.standard_normal((5, 8)) * 0.3
    alpha = r.standard_normal(30) * 1e3
    out = O.predict(Eq, E, 0.25, alpha)
    for a in range(5):
        kx = [entry_ref(Eq[a], E[i], 0.25) for i in range(30)]
        assert out[a] == dot_ref(kx, alpha)


def test_jacobi_diag():
    r = np.random.default_rng(7)
    E = r.standard_normal((10, 4)) * 0.5
    lam = 0.01
    d = O.jacobi_diag(E, 0.5, lam)
    K, _ = O.assemble(E, 0.5)
    assert (d == 1.0 / (lam + np.diag(K))).all()
    # worked example diagonal: d = (1/1.391, 1/1.233, 1/1.289) at 3 decimals
    dex = O.jacobi_diag(np.array(GOLD["E"]), 1.0, GOLD["lam"])
    assert np.allclose(1.0 / dex, np.diag(GOLD["lamI_plus_G"]), atol=1e-3)
