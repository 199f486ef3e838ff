"""LEARNED preconditioner with ON_THE_FLY storage ("LAKER
at C5"): the fit's directions GEMM U = (lambda I + K) Z consumes K's rows
assembled chunk by chunk into a transient buffer (K never stored),
and the solve applies K on the fly with the factored P.

* with one chunk the fit is the MATERIALIZED fit: identical factors, bitwise;
* with several chunks (LAKER_FIT_OTF_CHUNK) the factors agree to rounding;
* staged parity: the oracle's PCG with the GPU's factors on the oracle's K takes
  the same iterations to the same alpha, bitwise (EXACT on-the-fly entries are
  the correctly rounded K_ij, T19)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from staged import oracle_pcg_factored  # noqa: E402
from synth import make_problem, make_directions  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


def _fit(L, P, storage, Z):
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, storage, L.MODE_EXACT)
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_FACTORED)
    return c


@pytest.mark.parametrize("cid,n", [(2, None), (3, 1000)])
def test_otf_learned_matches_materialized(L, cid, n):
    P = make_problem(cid, n=n)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    cm = _fit(L, P, L.STORE_MATERIALIZED, Z)
    co = _fit(L, P, L.STORE_ON_THE_FLY, Z)
    Qm, Mm, am = cm.get_preconditioner_factors()
    Qo, Mo, ao = co.get_preconditioner_factors()
    assert am == ao and (Qm == Qo).all() and (Mm == Mo).all()
    a1, r1, _ = cm.pcg_solve(P.y, P.tol)
    a2, r2, _ = co.pcg_solve(P.y, P.tol)
    assert r1[0]["iters"] == r2[0]["iters"] and (a1 == a2).all()
    cm.close()
    co.close()


def test_otf_learned_chunked_staged_parity(L, monkeypatch):
    P = make_problem(3, n=1000)   # ragged: 1000 = 7 x 128 + 104
    Z = np.asfortranarray(make_directions(3, P.n, P.n_dirs))
    cm = _fit(L, P, L.STORE_MATERIALIZED, Z)
    Qm, Mm, am = cm.get_preconditioner_factors()
    cm.close()
    monkeypatch.setenv("LAKER_FIT_OTF_CHUNK", "300")   # 4 chunks, the last ragged
    co = _fit(L, P, L.STORE_ON_THE_FLY, Z)
    Q, M, a = co.get_preconditioner_factors()
    assert abs(a - am) <= 1e-12 * am
    # Q is unique up to rounding (positive-diagonal R); M is a smooth function of R
    assert np.abs(Q - Qm).max() <= 1e-9
    assert np.abs(M - Mm).max() <= 1e-8 * np.abs(Mm).max()
    K, _ = O.assemble(P.E, P.scale)
    ao, ro = oracle_pcg_factored(co, K, P.lam, P.y, Q, M, a, tol=P.tol)
    al, reps, _ = co.pcg_solve(P.y, P.tol)
    assert reps[0]["iters"] == ro.iters
    assert (al == ao).all()
    co.close()


def test_otf_learned_dense_layout(L):
    """DENSE p_layout with on-the-fly K: the dense rows are Q M Q^T + a^{-1/2} I
    formed from the same factors; the solve reaches the tolerance."""
    P = make_problem(2)
    Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_DENSE)
    Pd = c.get_preconditioner_rows()
    assert (Pd == Pd.T).all()
    a, reps, _ = c.pcg_solve(P.y, P.tol)
    K, _ = O.assemble(P.E, P.scale)
    ao, ro = O.pcg(K, P.lam, P.y, O.P_DENSE, Pd, tol=P.tol)
    assert reps[0]["iters"] == ro.iters and (a == ao).all()
    c.close()
