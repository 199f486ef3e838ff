"""Pins of the oracle's block PCG (O'Leary 1980; oracle.block_pcg), the C4 block-CG variant
(SURVEY §8(f) NEXT-4): each against something other than itself."""
import numpy as np
import pytest

import oracle as O


def _spd(n, seed, cond=1e3):
    rng = np.random.default_rng(seed)
    Qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    w = np.geomspace(1.0, cond, n)
    return (Qm * w) @ Qm.T


def test_one_column_is_alg1_pcg():
    """m = 1: block CG is CG (O'Leary, Sec. 2) -- the same iterates as Alg. 1,
    here the oracle's Dot2 PCG with a dense preconditioner."""
    n = 80
    K = _spd(n, 1)
    lam = 1e-2
    rng = np.random.default_rng(2)
    y = rng.standard_normal(n)
    Pm = np.diag(1.0 / (np.diag(K) + lam))
    a1, r1 = O.pcg(K, lam, y, O.P_DENSE, Pm, tol=1e-10)
    ab, rb = O.block_pcg(K, lam, y, precond=lambda V: Pm @ V, tol=1e-10)
    assert rb.termination == O.TERM_RESIDUAL_TOL and r1.termination == O.TERM_RESIDUAL_TOL
    assert abs(rb.iters - r1.iters) <= 1
    assert np.linalg.norm(ab[:, 0] - a1) / np.linalg.norm(a1) <= 1e-8


def test_finite_termination_distinct_eigenvalues():
    """A of order k with k simple eigenvalues: the block Krylov space of m generic columns
    reaches dimension k after ceil(k / m) steps, so block CG terminates there (exact
    arithmetic; O'Leary Thm. 3), where single-vector CG needs k steps."""
    rng = np.random.default_rng(3)
    k, m = 24, 4
    Qm, _ = np.linalg.qr(rng.standard_normal((k, k)))
    K = (Qm * np.arange(1.0, k + 1.0)) @ Qm.T
    Y = rng.standard_normal((k, m))
    X, rep = O.block_pcg(K, 0.0, Y, tol=1e-10)
    assert rep.termination == O.TERM_RESIDUAL_TOL
    assert rep.iters <= int(np.ceil(k / m))
    assert np.all(rep.true_rel_residual <= 1e-9)
    _, rep1 = O.block_pcg(K, 0.0, Y[:, :1], tol=1e-10)
    assert rep1.iters >= k - 2


def test_exact_preconditioner_one_step():
    """P = A^{-1}: Z0 = A^{-1} Y = D0, alpha0 = I, X1 = A^{-1} Y (one step)."""
    n, m, lam = 50, 3, 0.5
    K = _spd(n, 4, cond=1e2)
    Ainv = np.linalg.inv(K + lam * np.eye(n))
    Y = np.random.default_rng(5).standard_normal((n, m))
    X, rep = O.block_pcg(K, lam, Y, precond=lambda V: Ainv @ V, tol=1e-10)
    assert rep.iters == 1 and rep.termination == O.TERM_RESIDUAL_TOL


@pytest.mark.parametrize("m", [2, 5])
def test_matches_dense_solve(m):
    """The block solution equals the dense Cholesky solve (reference_solve) column by column."""
    n, lam = 120, 1e-3
    K = _spd(n, 6, cond=1e4)
    Y = np.random.default_rng(7).standard_normal((n, m))
    X, rep = O.block_pcg(K, lam, Y, tol=1e-12)
    assert rep.termination == O.TERM_RESIDUAL_TOL
    for c in range(m):
        ref = O.reference_solve(K, lam, Y[:, c])
        assert np.linalg.norm(X[:, c] - ref) / np.linalg.norm(ref) <= 1e-8
