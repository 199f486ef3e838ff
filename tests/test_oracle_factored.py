"""Oracle pins for the factored preconditioner P = a^{-1/2} I + Q M Q^T
(P = Sigma*^{-1/2}, Eq. preconditioner-Sigmma, in the structured
form of DESIGN.md O4': Sigma* = a I + Q (T - a I) Q^T with Q^T Q = I, hence
Sigma*^{-1/2} = a^{-1/2} I + Q (T^{-1/2} - a^{-1/2} I) Q^T).  Pinned against
exact rational arithmetic, numpy's dense product, the oracle's own dense P and
the defining property P Sigma* P = I."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from synth import make_problem, make_directions


def _exact_factored(Q, M, ainv, r):
    n, m = Q.shape
    F = lambda x: Fraction(float(x))  # noqa: E731
    z = [sum(F(Q[i, k]) * F(r[i]) for i in range(n)) for k in range(m)]
    w = [sum(F(M[k, j]) * z[j] for j in range(m)) for k in range(m)]
    return [F(ainv) * F(r[i]) + sum(F(Q[i, k]) * w[k] for k in range(m)) for i in range(n)]


def test_factored_apply_exact_dyadic():
    """Dyadic inputs: every intermediate is exactly representable, so each
    Dot2 is exact and theta must equal the rational result exactly -- a dropped
    term, a transposed Q or M, or a missing a^{-1/2} r term fails."""
    r = np.random.default_rng(1)
    n, m = 9, 4
    Q = r.integers(-4, 5, (n, m)) / 8.0
    M = r.integers(-3, 4, (m, m)).astype(float)
    M[0, 1] = 5.0  # non-symmetric on purpose: pins M vs M^T
    x = r.integers(-8, 9, n) / 4.0
    th = O.factored_apply(Q, M, 0.5, x)
    ex = _exact_factored(Q, M, 0.5, x)
    assert all(Fraction(float(t)) == e for t, e in zip(th, ex))


@pytest.mark.parametrize("n,m", [(1, 1), (7, 1), (50, 7), (300, 64)])
def test_factored_apply_vs_numpy_dense(n, m):
    r = np.random.default_rng(n + m)
    Q, _ = np.linalg.qr(r.standard_normal((n, m)))
    M = r.standard_normal((m, m))
    M = M + M.T
    x = r.standard_normal(n)
    P = 0.7 * np.eye(n) + Q @ M @ Q.T
    th = O.factored_apply(Q, M, 0.7, x)
    assert np.abs(th - P @ x).max() <= 1e-13 * np.abs(P).sum(axis=1).max() * np.abs(x).max()


def test_factors_reproduce_fitted_P_and_sigma_inverse_sqrt():
    P = make_problem(1)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(1, P.n, P.n_dirs)
    Pd, rep, st = O.cccp_fit_structured(K, P.lam, Z)
    Q, M, ainv = O.factors(st)
    Pf = ainv * np.eye(P.n) + Q @ M @ Q.T
    assert np.linalg.norm(Pf - Pd) / np.linalg.norm(Pd) <= 1e-12
    # P Sigma* P = I with Sigma* = a I + Q (T - a I) Q^T (T16)
    a = 1.0 / ainv ** 2
    S = a * np.eye(P.n) + Q @ (st.T - a * np.eye(st.T.shape[0])) @ Q.T
    assert np.abs(Pf @ S @ Pf - np.eye(P.n)).max() <= 1e-7 * np.sqrt(P.n)
    # applies agree with the dense one to rounding
    x = np.random.default_rng(4).standard_normal(P.n)
    assert np.abs(O.factored_apply(Q, M, ainv, x) - O.dense_apply(Pd, x)).max() <= 1e-10 * np.abs(Pd @ x).max()


def test_pcg_factored_matches_dense_and_cholesky():
    P = make_problem(1)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(1, P.n, P.n_dirs)
    Pd, _, st = O.cccp_fit_structured(K, P.lam, Z)
    Q, M, ainv = O.factors(st)
    af, rf = O.pcg_factored(K, P.lam, P.y, Q, M, ainv, tol=P.tol)
    ad, rd = O.pcg(K, P.lam, P.y, O.P_DENSE, Pd, tol=P.tol)
    assert rf.termination == O.TERM_RESIDUAL_TOL
    assert abs(rf.iters - rd.iters) <= 25  # R15(iii): rounding-level P changes move counts
    ref = O.reference_solve(K, P.lam, P.y)
    assert np.linalg.norm(af - ref) / np.linalg.norm(ref) <= 1e-6
    # with Q = 0 the factored P is a^{-1/2} I: the same recurrence as P = I scaled,
    # i.e. textbook CG iterates (the step lengths absorb the scale)
    n = P.n
    a0, r0 = O.pcg_factored(K, P.lam, P.y, np.zeros((n, 1)), np.zeros((1, 1)), 1.0, tol=P.tol)
    a1, r1 = O.pcg(K, P.lam, P.y, O.P_NONE, None, tol=P.tol)
    assert r0.iters == r1.iters and (a0 == a1).all()


def _exact_factored_qm(Q, QM, ainv, r):
    n, m = Q.shape
    F = lambda x: Fraction(float(x))  # noqa: E731
    z = [sum(F(Q[i, k]) * F(r[i]) for i in range(n)) for k in range(m)]
    return [F(ainv) * F(r[i]) + sum(F(QM[i, k]) * z[k] for k in range(m)) for i in range(n)]


def test_factored_qm_apply_exact_dyadic():
    """QM form (R21): theta = a^{-1/2} r + QM (Q^T r).  Dyadic inputs make
    every Dot2 exact: theta must equal the rational result; a QM used transposed, a
    Q^T r taken over the wrong index or a dropped a^{-1/2} r term fails."""
    r = np.random.default_rng(2)
    n, m = 9, 4
    Q = r.integers(-4, 5, (n, m)) / 8.0
    QM = r.integers(-3, 4, (n, m)).astype(float)
    x = r.integers(-8, 9, n) / 4.0
    th = O.factored_qm_apply(Q, QM, 0.5, x)
    assert all(Fraction(float(t)) == e for t, e in zip(th, _exact_factored_qm(Q, QM, 0.5, x)))


@pytest.mark.parametrize("n,m", [(1, 1), (50, 7), (300, 64)])
def test_factored_qm_apply_is_P_times_r(n, m):
    """With QM = Q M the QM form is the same operator a^{-1/2} I + Q M Q^T (dense
    numpy product as the independent reference), and M = 0 gives a^{-1/2} r exactly."""
    r = np.random.default_rng(3 * n + m)
    Q, _ = np.linalg.qr(r.standard_normal((n, m)))
    M = r.standard_normal((m, m))
    M = M + M.T
    x = r.standard_normal(n)
    P = 0.7 * np.eye(n) + Q @ M @ Q.T
    th = O.factored_qm_apply(Q, Q @ M, 0.7, x)
    assert np.abs(th - P @ x).max() <= 1e-13 * np.abs(P).sum(axis=1).max() * np.abs(x).max()
    assert (O.factored_qm_apply(Q, np.zeros((n, m)), 0.7, x) == 0.7 * x).all()


def test_pcg_factored_qm_solves():
    P = make_problem(1)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(1, P.n, P.n_dirs)
    _, _, st = O.cccp_fit_structured(K, P.lam, Z)
    Q, M, ainv = O.factors(st)
    aq, rq = O.pcg_factored_qm(K, P.lam, P.y, Q, Q @ M, ainv, tol=P.tol)
    af, rf = O.pcg_factored(K, P.lam, P.y, Q, M, ainv, tol=P.tol)
    assert rq.termination == O.TERM_RESIDUAL_TOL
    assert abs(rq.iters - rf.iters) <= 25  # R15(iii): a different rounding of the same P
    ref = O.reference_solve(K, P.lam, P.y)
    assert np.linalg.norm(aq - ref) / np.linalg.norm(ref) <= 1e-6
