"""FAST on-the-fly operator / predict (otf_fast.cu, DMMA dots + CUDA exp,
fp64 row sums) against the oracle's correctly rounded Dot2 values: error
bounded by a few ulps of sum_j |K_ij p_j| (R15 iii envelope parity for the
solve)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_problem  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (5, 3000), (1, 77)])
def test_fast_on_the_fly_apply_and_predict(L, cid, n):
    P = make_problem(cid, n=n, grid=16)
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
    r = np.random.default_rng(1)
    p = r.standard_normal(P.n)
    q = c.apply_operator(p)
    K, _ = O.assemble(P.E, P.scale)
    qo = O.apply(K, P.lam, p)
    bound = (np.abs(K) @ np.abs(p) + P.lam * np.abs(p)) * 1e-13 + 1e-300
    assert (np.abs(q - qo) <= bound).all()
    alpha = r.standard_normal(P.n) * 1e3
    m = c.predict(P.Eq, alpha, mode=L.MODE_FAST)
    mo = O.predict(P.Eq, P.E, P.scale, alpha)
    Kx = O.cross_kernel(P.Eq, P.E, P.scale)
    assert (np.abs(m - mo) <= (np.abs(Kx) @ np.abs(alpha)) * 1e-13).all()
    # the FAST on-the-fly Jacobi solve reaches the tolerance; alpha within R14 of Cholesky
    if P.n <= 2048:
        c.set_preconditioner(L.PRECOND_JACOBI)
        a, reps, _ = c.pcg_solve(P.y, P.tol)
        ref = O.reference_solve(K, P.lam, P.y)
        assert reps[0]["termination"] == L.TERM_RESIDUAL_TOL
        assert np.linalg.norm(a - ref) / np.linalg.norm(ref) <= 1e-6
    c.close()
