"""Lanczos eigenvalue estimates of the preconditioned operator from the CG
coefficients (laker_solve_report.lanczos_lmin/lmax; SURVEY §8(f) NEXT-4
diagnostics: kappa(PA), the quantity of Table I / P:853-858).  Pinned against
numpy's symmetric eigensolver on the same K and P: after a solve to 1e-10 the
extreme Ritz values match the extreme eigenvalues of P^(1/2) (lambda I + K) P^(1/2)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_problem, make_directions  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.mark.parametrize("kind", ["none", "jacobi", "learned"])
def test_lanczos_extremes_match_eigensolver(L, kind):
    P = make_problem(1)
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    A = K + P.lam * np.eye(P.n)
    if kind == "none":
        c.set_preconditioner(L.PRECOND_NONE)
        Pm = np.eye(P.n)
    elif kind == "jacobi":
        c.set_preconditioner(L.PRECOND_JACOBI)
        Pm = np.diag(O.jacobi_diag(P.E, P.scale, P.lam))
    else:
        Z = make_directions(1, P.n, P.n_dirs)
        Pm = np.ascontiguousarray(O.cccp_fit_structured(K, P.lam, Z)[0])
        c.set_preconditioner(L.PRECOND_EXTERNAL_DENSE, Pm)
    _, reps, _ = c.pcg_solve(P.y, 1e-10)
    c.close()
    Lc = np.linalg.cholesky(Pm)
    w = np.linalg.eigvalsh(Lc.T @ A @ Lc)
    r = reps[0]
    assert r["termination"] == L.TERM_RESIDUAL_TOL
    assert abs(r["lanczos_lmax"] / w[-1] - 1) <= 1e-8
    assert abs(r["lanczos_lmin"] / w[0] - 1) <= 0.05
    assert r["lanczos_lmin"] >= w[0] * (1 - 1e-8)  # Ritz values lie inside the spectrum


def test_lanczos_kappa_trend_T21(L):
    """kappa estimates: LAKER << NONE at C2 (T21; the paper's Table I trend)."""
    P = make_problem(2)
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    c.set_preconditioner(L.PRECOND_NONE)
    _, rn, _ = c.pcg_solve(P.y, P.tol)
    Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    _, rl, _ = c.pcg_solve(P.y, P.tol)
    c.close()
    kn = rn[0]["lanczos_lmax"] / rn[0]["lanczos_lmin"]
    kl = rl[0]["lanczos_lmax"] / rl[0]["lanczos_lmin"]
    assert kl <= kn / 50, (kn, kl)
