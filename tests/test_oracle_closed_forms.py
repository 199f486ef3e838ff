"""Closed-form pins of the oracle's fit pieces that no other test fixes independently
(VERDICT r01 "What's weak" 1).  CPU only.

* The shrinkage CCCP step with gamma > 0, eps > 0, rho in (0, 1) (Eqs.
  kernel_shrinkage_cccp_F / _Sigma / _normalization), on directions
  ubar_k = V e_k (k < m < n, V orthogonal).  Then every iterate is
  Sigma_t = s1 Pi_1 + s2 Pi_2 with Pi_1 the projector on span{V e_k : k < m}, and
  one step maps (s1, s2) in closed form:
      qf = 1/s1,  w = 1/(qf + eps),
      f1 = ((n/m) w + gamma) / (1 + gamma/n),   f2 = gamma / (1 + gamma/n),
      t_i = (1 - rho) f_i + rho,  tr = m t1 + (n - m) t2,  s_i' = n t_i / tr.
  The ratio s1'/s2' = t1/t2 depends on the (1 + gamma/n)^{-1} factor, so a dropped or
  misplaced factor, a wrong sign, a transposed V or a missing eps fails here.  The
  closed form is evaluated in exact rational arithmetic (fractions.Fraction).
* The directions u_k = (lambda I + G) z_k, ubar_k = u_k / ||u_k|| (Eq.
  random_directions) on a diagonal and on a rank-one G, element by element.
* The objective R(alpha) = ||G alpha - y||^2 + lambda alpha^T G alpha (Eq.
  simu-R-definition) on a diagonal G, and its closed-form minimum value
  R(alpha*) = lambda y^T (lambda I + G)^{-1} y.
* T12: the structured fit (O4') equals the literal n x n iteration at C2.
"""
import math
from fractions import Fraction as Fr

import numpy as np
import pytest

import oracle as O
from synth import make_problem, make_directions


def _closed_step(s1, s2, n, m, gamma, eps, rho):
    """One shrinkage-CCCP step on Sigma = s1 Pi_1 + s2 Pi_2 (see module docstring), exact."""
    s1, s2, gamma, eps, rho = Fr(s1), Fr(s2), Fr(gamma), Fr(eps), Fr(rho)
    qf = 1 / s1
    w = 1 / (qf + eps)
    c = 1 / (1 + gamma / n)
    f1 = c * (Fr(n, m) * w + gamma)
    f2 = c * gamma
    t1 = (1 - rho) * f1 + rho
    t2 = (1 - rho) * f2 + rho
    tr = m * t1 + (n - m) * t2
    return n * t1 / tr, n * t2 / tr, t1, t2


def _frame(n, m, seed):
    V, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return V, V[:, :m].copy()


@pytest.mark.parametrize("n,m,gamma,eps,rho", [
    (12, 5, 0.1, 1e-3, 0.3),
    (30, 7, 0.1, 1e-12, 0.376),
    (9, 2, 2.5, 0.5, 0.05),
])
def test_cccp_step_literal_closed_form(n, m, gamma, eps, rho):
    V, Ub = _frame(n, m, n + m)
    Pi1 = Ub @ Ub.T
    Pi2 = np.eye(n) - Pi1
    s1, s2 = Fr(1), Fr(1)
    Sigma = np.eye(n)
    for step in range(4):
        s1n, s2n, t1, t2 = _closed_step(s1, s2, n, m, gamma, eps, rho)
        Snew, St = O.cccp_step_literal(Sigma, Ub, gamma, eps, rho, return_tilde=True)
        ref = float(s1n) * Pi1 + float(s2n) * Pi2
        ref_t = float(t1) * Pi1 + float(t2) * Pi2
        assert np.linalg.norm(Snew - ref) <= 1e-13 * np.linalg.norm(ref), step
        assert np.linalg.norm(St - ref_t) <= 1e-13 * np.linalg.norm(ref_t), step
        # the (1+gamma/n)^{-1} factor is visible: the complement eigenvalue before
        # normalisation is (1-rho) gamma/(1+gamma/n) + rho, not (1-rho) gamma + rho
        wrong = (1 - rho) * gamma + rho
        assert abs(float(t2) - wrong) > 1e3 * 2.0 ** -52 * wrong
        s1, s2, Sigma = s1n, s2n, Snew


@pytest.mark.parametrize("n,m,gamma,eps", [(16, 4, 0.1, 1e-12), (24, 5, 0.7, 1e-4)])
def test_cccp_fits_closed_form_fixed_point(n, m, gamma, eps):
    """Both oracle fits (literal and structured, with the R6 rho schedule) against the
    closed-form scalar iteration run to the same stopping rule (relative Frobenius
    change <= 1e-8, reading R8); P = Sigma*^{-1/2} then has eigenvalues s1^{-1/2}
    on span(Ubar) and s2^{-1/2} on its complement."""
    V, Ub = _frame(n, m, 3 * n + m)
    # structured/literal compute Ubar from (K, lambda, Z): choose G = 0, lambda = 1,
    # Z = Ub so that ubar_k = z_k / ||z_k|| = V e_k exactly as given
    K0, lam = np.zeros((n, n)), 1.0
    s1, s2 = Fr(1), Fr(1)
    steps, last_change = 0, None
    for t in range(200):
        lmin = min(float(s1), float(s2))
        rho = O.rho_schedule(m, n, gamma, lmin)
        s1n, s2n, _, _ = _closed_step(s1, s2, n, m, gamma, eps, rho)
        # ||Sigma' - Sigma||_F / ||Sigma||_F in closed form
        d2 = m * (s1n - s1) ** 2 + (n - m) * (s2n - s2) ** 2
        n2 = m * s1 ** 2 + (n - m) * s2 ** 2
        change = math.sqrt(float(d2 / n2))
        s1, s2 = s1n, s2n
        steps, last_change = t + 1, change
        if change <= 1e-8:
            break
    Pl, rl, Sl = O.cccp_fit_literal(K0, lam, Ub, gamma=gamma, eps=eps, return_sigma=True)
    Ps, rs, st = O.cccp_fit_structured(K0, lam, Ub, gamma=gamma, eps=eps)
    assert rl.iters == rs.iters == steps
    assert abs(rl.final_change - last_change) <= 1e-6 * last_change
    Pi1 = Ub @ Ub.T
    ref_S = float(s1) * Pi1 + float(s2) * (np.eye(n) - Pi1)
    ref_P = float(s1) ** -0.5 * Pi1 + float(s2) ** -0.5 * (np.eye(n) - Pi1)
    assert np.linalg.norm(Sl - ref_S) <= 1e-12 * np.linalg.norm(ref_S)
    for Pm in (Pl, Ps):
        assert np.linalg.norm(Pm - ref_P) <= 1e-12 * np.linalg.norm(ref_P)
    # structured state: Sigma = a I + Ubar diag(b) Ubar^T with a = s2, b_k = s1 - s2
    assert abs(st.a - float(s2)) <= 1e-14 * float(s2)
    assert np.allclose(st.b, float(s1 - s2), rtol=1e-12, atol=0)
    assert abs(rs.sigma_min_eig - float(min(s1, s2))) <= 1e-14


def test_directions_diagonal_and_rank_one():
    """u_k = lambda z_k + G z_k, ubar_k = u_k/||u_k||_2, element by element."""
    r = np.random.default_rng(11)
    n, Nr, lam = 9, 4, 0.37
    Z = r.standard_normal((n, Nr))
    g = np.exp(r.uniform(-2, 2, n))
    Ub, norms = O.directions(np.diag(g), lam, Z)
    for k in range(Nr):
        u = [(lam + g[i]) * Z[i, k] for i in range(n)]
        nu = math.sqrt(math.fsum(x * x for x in u))
        assert abs(norms[k] - nu) <= 4 * 2.0 ** -52 * nu
        for i in range(n):
            assert abs(Ub[i, k] - u[i] / nu) <= 8 * 2.0 ** -52
    # rank one G = v v^T: u_k = lambda z_k + v (v . z_k); non-square Z catches a transpose
    v = r.standard_normal(n)
    Ub, norms = O.directions(np.outer(v, v), lam, Z)
    for k in range(Nr):
        vz = math.fsum(v[j] * Z[j, k] for j in range(n))
        u = [lam * Z[i, k] + v[i] * vz for i in range(n)]
        nu = math.sqrt(math.fsum(x * x for x in u))
        for i in range(n):
            assert abs(Ub[i, k] - u[i] / nu) <= 1e-14


def test_objective_closed_forms():
    """R(alpha) = ||G alpha - y||^2 + lambda alpha^T G alpha on G = diag(g):
    exact rational value at a random alpha; R(0) = ||y||^2; the minimiser
    alpha* = (lambda I + G)^{-1} y gives R(alpha*) = lambda y^T (lambda I + G)^{-1} y."""
    r = np.random.default_rng(12)
    n, lam = 15, 0.01
    g = np.exp(r.uniform(-1, 2, n))
    y = r.standard_normal(n) * 10
    a = r.standard_normal(n)
    exact = sum((Fr(g[i]) * Fr(a[i]) - Fr(y[i])) ** 2 + Fr(lam) * Fr(g[i]) * Fr(a[i]) ** 2 for i in range(n))
    val = O.objective(np.diag(g), lam, a, y)
    assert abs(val - float(exact)) <= 1e-13 * float(exact)
    assert abs(O.objective(np.diag(g), lam, np.zeros(n), y) - float(sum(Fr(v) ** 2 for v in y))) <= 1e-13 * (y @ y)
    astar = y / (lam + g)
    rmin = sum(Fr(lam) * Fr(y[i]) ** 2 / (Fr(lam) + Fr(g[i])) for i in range(n))
    assert abs(O.objective(np.diag(g), lam, astar, y) - float(rmin)) <= 1e-11 * float(rmin)
    # the minimum is a minimum: any perturbation increases R
    for s in range(3):
        d = r.standard_normal(n) * 1e-3
        assert O.objective(np.diag(g), lam, astar + d, y) > O.objective(np.diag(g), lam, astar, y)


def test_literal_equals_structured_T12_C2():
    """T12 at C2 (n = 2048, N_r = 512): the pilot had both forms stop at the
    same step with the same convergence measure; qf/Sigma/P agree to the T12 bounds."""
    P = make_problem(2)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(2, P.n, P.n_dirs)
    Pl, rl, Sl = O.cccp_fit_literal(K, P.lam, Z, return_sigma=True)
    Ps, rs, st = O.cccp_fit_structured(K, P.lam, Z)
    assert rl.converged and rs.converged and rl.iters == rs.iters
    assert np.allclose(rl.changes, rs.changes, rtol=1e-5)
    Ss = st.a * np.eye(P.n) + (st.Ubar * st.b) @ st.Ubar.T
    assert np.linalg.norm(Ss - Sl) / np.linalg.norm(Sl) <= 1e-12
    assert np.linalg.norm(Ps - Pl) / np.linalg.norm(Pl) <= 1e-9
    assert abs(rs.sigma_min_eig - rl.sigma_min_eig) <= 1e-9 * rl.sigma_min_eig
