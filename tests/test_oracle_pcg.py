"""Pins of the oracle PCG (Alg. 1) against closed forms, finite
termination of CG, a textbook CG written here, the direct Cholesky solve and
the paper's reported trends (T8-T11, T20, T21; R12 edge cases).  CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from synth import make_problem, make_directions


def _diag_K(dvals, lam):
    """K such that lambda I + K = diag(dvals)."""
    return np.diag(np.asarray(dvals, dtype=np.float64) - lam)


def test_identity_one_iteration_T9():
    n, lam = 50, 0.25
    y = np.random.default_rng(0).standard_normal(n)
    alpha, rep = O.pcg(_diag_K(np.ones(n), lam), lam, y, tol=1e-12)
    assert rep.iters == 1 and rep.termination == O.TERM_RESIDUAL_TOL
    assert np.array_equal(alpha, y)


@pytest.mark.parametrize("m", [2, 3, 5, 8])
def test_diagonal_m_distinct_values_T9(m):
    """CG on a diagonal operator with m distinct eigenvalues terminates in m
    steps in exact arithmetic; kappa <= 1e2 keeps fp64 at exactly m (A.11)."""
    n, lam = 64, 1e-3
    vals = np.linspace(1.0, 50.0, m)
    dv = vals[np.arange(n) % m]
    y = np.random.default_rng(m).standard_normal(n)
    alpha, rep = O.pcg(_diag_K(dv, lam), lam, y, tol=1e-10)
    assert rep.termination == O.TERM_RESIDUAL_TOL
    assert m <= rep.iters <= m + 1
    assert np.allclose(alpha, y / dv, rtol=1e-9)


def test_jacobi_on_diagonal_and_exact_inverse_one_iteration_T9():
    n, lam = 40, 1e-2
    r = np.random.default_rng(1)
    dv = np.exp(r.uniform(-3, 3, n))
    y = r.standard_normal(n)
    K = _diag_K(dv, lam)
    _, rep = O.pcg(K, lam, y, O.P_JACOBI, 1.0 / dv, tol=1e-12)
    assert rep.iters == 1
    # dense P = A^{-1} on a random SPD system
    B = r.standard_normal((n, n))
    A = B @ B.T / n + np.eye(n)
    K = A - lam * np.eye(n)
    Pinv = np.linalg.inv(A)
    Pinv = 0.5 * (Pinv + Pinv.T)
    _, rep = O.pcg(K, lam, y, O.P_DENSE, Pinv, tol=1e-10)
    assert rep.iters == 1


def test_exact_clusters_finite_termination_T7_T8():
    """Q groups of identical embeddings: lambda I + K has Q+1 distinct
    eigenvalues (lambda with multiplicity n - Q, and lambda + eig(D^1/2 M D^1/2)),
    so CG (P = I) stops in m = Q+1 steps in exact arithmetic."""
    r = np.random.default_rng(2)
    Q, lam = 4, 1e-2
    centres = r.standard_normal((Q, 6)) * 0.5
    sizes = np.array([10, 25, 7, 22])
    E = np.repeat(centres, sizes, axis=0)
    n = E.shape[0]
    K, _ = O.assemble(E, 1.0)
    # closed-form spectrum
    M = np.exp(centres @ centres.T)
    Dh = np.diag(np.sqrt(sizes))
    big = lam + np.linalg.eigvalsh(Dh @ M @ Dh)
    w = np.linalg.eigvalsh(K + lam * np.eye(n))
    assert np.allclose(np.sort(w)[-Q:], np.sort(big), rtol=1e-10)
    assert np.allclose(np.sort(w)[: n - Q], lam, atol=1e-10)
    y = r.standard_normal(n)
    _, rep = O.pcg(K, lam, y, tol=1e-10)
    assert rep.termination == O.TERM_RESIDUAL_TOL
    assert Q + 1 <= rep.iters <= Q + 1 + 3


def test_single_cluster_condition_number_closed_form():
    """Q = 1: kappa(lambda I + K) = 1 + n exp(s ||e||^2) / lambda."""
    n, lam, s = 30, 1e-3, 0.5
    e = np.array([0.3, -0.2, 0.1])
    K, _ = O.assemble(np.tile(e, (n, 1)), s)
    kappa = O.cond_spd(K + lam * np.eye(n))
    assert abs(kappa / (1.0 + n * math.exp(s * e @ e) / lam) - 1.0) < 1e-6


def _textbook_cg(A, b, iters):
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = r @ r
    hist = []
    for _ in range(iters):
        Ap = A @ p
        a = rr / (p @ Ap)
        x = x + a * p
        r = r - a * Ap
        rr_new = r @ r
        hist.append(math.sqrt(rr_new) / np.linalg.norm(b))
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, np.array(hist)


def test_pcg_none_is_textbook_cg_T10():
    r = np.random.default_rng(3)
    n, lam = 80, 0.5
    B = r.standard_normal((n, n)) / math.sqrt(n)
    K = B @ B.T
    y = r.standard_normal(n)
    alpha, rep = O.pcg(K, lam, y, tol=1e-13, max_iters=25)
    _, hist = _textbook_cg(K + lam * np.eye(n), y, rep.iters)
    assert np.allclose(rep.history, hist, rtol=1e-8, atol=0)


def test_edge_cases_R12():
    n, lam = 8, 0.1
    K = np.eye(n)
    alpha, rep = O.pcg(K, lam, np.zeros(n))
    assert rep.iters == 0 and rep.termination == O.TERM_ZERO_RHS and (alpha == 0).all()
    y = np.arange(1.0, n + 1)
    B = np.random.default_rng(4).standard_normal((n, n))
    _, rep = O.pcg(B @ B.T, 1e-6, y, tol=1e-30, max_iters=3)
    assert rep.iters == 3 and rep.termination == O.TERM_MAX_ITERS
    _, rep = O.pcg(K, lam, y, O.P_JACOBI, -np.ones(n))
    assert rep.termination == O.TERM_INDEFINITE
    _, rep = O.pcg(-2.0 * K, 1.0, y)        # lambda I + K = -I
    assert rep.termination == O.TERM_BREAKDOWN


@pytest.fixture(scope="module")
def c1():
    P = make_problem(1)
    K, _ = O.assemble(P.E, P.scale)
    return P, K


def test_c1_pcg_vs_cholesky_T11(c1):
    P, K = c1
    ref = O.reference_solve(K, P.lam, P.y)
    for kind, pm in [(O.P_NONE, None), (O.P_JACOBI, O.jacobi_diag(P.E, P.scale, P.lam))]:
        alpha, rep = O.pcg(K, P.lam, P.y, kind, pm, tol=P.tol)
        assert rep.termination == O.TERM_RESIDUAL_TOL
        assert rep.true_rel_residual <= 10 * P.tol
        assert np.linalg.norm(alpha - ref) / np.linalg.norm(ref) <= 1e-6
        assert O.residual(K, P.lam, alpha, P.y) <= 10 * P.tol


def test_c1_condition_number_trend_T20(c1):
    """kappa(lambda I + K) ~ n mean(K) / lambda: within x3."""
    P, K = c1
    kappa = O.cond_spd(K + P.lam * np.eye(P.n))
    pred = P.n * K.mean() / P.lam
    assert pred / 3 <= kappa <= 3 * pred


def test_c1_learned_preconditioner_trends_T21(c1):
    """kappa(P(lambda I+K)) <= kappa/50 and LAKER iterations < Jacobi."""
    P, K = c1
    Z = make_directions(1, P.n, P.n_dirs)
    Pm, rep = O.cccp_fit_structured(K, P.lam, Z)[:2]
    assert rep.converged
    A = K + P.lam * np.eye(P.n)
    assert O.cond_precond(Pm, A) <= O.cond_spd(A) / 50
    _, rl = O.pcg(K, P.lam, P.y, O.P_DENSE, Pm, tol=P.tol)
    _, rj = O.pcg(K, P.lam, P.y, O.P_JACOBI, O.jacobi_diag(P.E, P.scale, P.lam), tol=P.tol)
    assert rl.termination == rj.termination == O.TERM_RESIDUAL_TOL
    assert rl.iters < rj.iters
