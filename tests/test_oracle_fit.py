"""Pins of the oracle CCCP fit (Alg. 1 l.5-14) against
an independent Tyler map, Theorem 1's invariants,
special cases and the literal <-> structured identity (T12-T16).
CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from synth import make_problem, make_directions


def _tyler_step(Sigma, S):
    """Eq. tyler-fixed-point followed by tr = n, written
    with an explicit inverse (independent of the oracle's Cholesky path)."""
    n, N = S.shape
    Si = np.linalg.inv(Sigma)
    acc = np.zeros((n, n))
    for k in range(N):
        s = S[:, k]
        acc += np.outer(s, s) / (s @ Si @ s)
    new = (n / N) * acc
    return new * n / np.trace(new)


def test_tyler_reduction_T13():
    r = np.random.default_rng(0)
    n, N = 12, 40
    S = r.standard_normal((n, N)) * np.exp(r.uniform(-1, 1, n))[:, None]
    S /= np.linalg.norm(S, axis=0)
    Sig = np.eye(n)
    ref = np.eye(n)
    for _ in range(3):
        Sig = O.cccp_step_literal(Sig, S, gamma=0.0, eps=0.0, rho=0.0)
        ref = _tyler_step(ref, S)
        assert np.linalg.norm(Sig - ref) / np.linalg.norm(ref) <= 1e-10


def test_full_shrinkage_gives_identity_T15():
    r = np.random.default_rng(1)
    n, N = 10, 4
    S = r.standard_normal((n, N))
    S /= np.linalg.norm(S, axis=0)
    Sig = O.cccp_step_literal(np.eye(n) * 2.0, S, gamma=0.1, eps=1e-12, rho=1.0)
    assert np.allclose(Sig, np.eye(n), atol=1e-15)


@pytest.fixture(scope="module")
def c1():
    P = make_problem(1)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(1, P.n, P.n_dirs)
    return P, K, Z


def test_literal_equals_structured_T12(c1):
    P, K, Z = c1
    Pl, rl, Sl = O.cccp_fit_literal(K, P.lam, Z, return_sigma=True)
    Ps, rs, st = O.cccp_fit_structured(K, P.lam, Z)
    assert rl.converged and rs.converged and rl.iters == rs.iters
    assert np.allclose(rl.changes, rs.changes, rtol=1e-6)
    Ss = st.a * np.eye(P.n) + (st.Ubar * st.b) @ st.Ubar.T
    assert np.linalg.norm(Ss - Sl) / np.linalg.norm(Sl) <= 1e-12
    assert np.linalg.norm(Ps - Pl) / np.linalg.norm(Pl) <= 1e-9
    assert abs(rs.sigma_min_eig - rl.sigma_min_eig) <= 1e-9 * rl.sigma_min_eig


def test_theorem1_invariants_T14_T16(c1):
    P, K, Z = c1
    Pl, rep, Sig = O.cccp_fit_literal(K, P.lam, Z, return_sigma=True)
    n = P.n
    assert abs(np.trace(Sig) - n) <= 1e-8 * n
    Ubar, _ = O.directions(K, P.lam, Z)
    TS, St = O.cccp_step_literal(Sig, Ubar, 0.1, 1e-12, rep.rho_used, return_tilde=True)
    assert np.linalg.norm(TS - Sig) / np.linalg.norm(Sig) <= 10 * 1e-8
    assert np.linalg.eigvalsh(St)[0] >= rep.rho_used * (1 - 1e-10)       # Sigma~ >= rho I
    # P = Sigma*^{-1/2}: P Sigma P = I, symmetric, SPD
    assert np.linalg.norm(Pl @ Sig @ Pl - np.eye(n)) <= 1e-7 * math.sqrt(n)
    assert (Pl == Pl.T).all() and np.linalg.eigvalsh(Pl)[0] > 0
    # kappa(c P A) = kappa(P A)
    A = K + P.lam * np.eye(n)
    assert abs(O.cond_precond(7.0 * Pl, A) / O.cond_precond(Pl, A) - 1) < 1e-6


def test_rho_schedule_R6():
    assert O.rho_schedule(100, 100, 0.1, 1.0) == 1e-3
    assert abs(O.rho_schedule(25, 100, 0.1, 1.0) - 0.376) < 1e-15
    assert O.rho_schedule(25, 100, 0.1, 1e-9) >= 0.2
    assert O.rho_schedule(100, 100, 0.1, 1e-9) == 0.2
    assert O.nr_schedule(50) == 50 and O.nr_schedule(200) == 114 and O.nr_schedule(2000) == 500


def test_isotropic_input_gives_near_identity_T15():
    """Identity operator (ubar_k = z_k/||z_k||), N_r = 50 n: Sigma* ~ I, P ~ I."""
    r = np.random.default_rng(2)
    n = 10
    Z = r.standard_normal((n, 50 * n))
    Pm, rep = O.cccp_fit_literal(np.zeros((n, n)), 1.0, Z)[:2]
    assert rep.converged
    assert O.cond_spd(Pm) < 2.0


def test_spectral_alignment():
    """on diag(100, 1, ..., 1) the top eigenvector of Sigma* is e_1."""
    r = np.random.default_rng(3)
    n = 8
    K = np.diag([100.0] + [1.0] * (n - 1)) - 1e-2 * np.eye(n)
    Z = r.standard_normal((n, 50 * n))
    Pm, rep, Sig = O.cccp_fit_literal(K, 1e-2, Z, return_sigma=True)
    w, V = np.linalg.eigh(Sig)
    assert abs(V[0, -1]) >= 0.99


def test_structured_handles_full_rank_directions():
    """N_r >= n: Q is square and lambda_min(Sigma) = lambda_min(T) (not a)."""
    r = np.random.default_rng(4)
    n = 20
    B = r.standard_normal((n, n))
    K = B @ B.T / n
    Z = r.standard_normal((n, 3 * n))
    Pl, rl, Sl = O.cccp_fit_literal(K, 0.1, Z, return_sigma=True)
    Ps, rs, _ = O.cccp_fit_structured(K, 0.1, Z)
    assert rl.iters == rs.iters
    assert np.linalg.norm(Ps - Pl) / np.linalg.norm(Pl) <= 1e-9
