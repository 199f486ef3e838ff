"""Symmetric on-the-fly operator (otf_sym.cu): with K never
stored, each off-diagonal tile of the block upper triangle is computed once and
used for its rows and its columns (K_ij = K_ji, reading R2).  EXACT entries are
the correctly rounded exp of the sequential-Dot2 argument, the same bits for
(i, j) and (j, i), and every row sum is a Dot2 over the same products, so the
apply equals the materialized one and the oracle's (O2) bitwise --
including ragged n (tiles of 64), n below one tile, and p with a wide dynamic
range; PCG solves on the fly take the oracle's iterations to its alpha."""
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


@pytest.fixture(scope="module")
def ctx(L):
    c = L.Context(0)
    yield c
    c.close()


def _bitwise(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    bad = np.flatnonzero(a.ravel() != b.ravel())
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}"


@pytest.mark.parametrize("cid,n", [(1, 50), (1, 64), (1, 65), (1, None), (2, 1000), (3, 2048)])
def test_otf_sym_apply_bitwise(ctx, L, cid, n):
    P = make_problem(cid, n=n)
    r = np.random.default_rng(11)
    ps = (r.standard_normal(P.n),
          np.where(np.arange(P.n) % 3 == 0, 1.0, -1.0) * np.exp(r.uniform(-8, 8, P.n)))
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    qm = [ctx.apply_operator(p) for p in ps]
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
    for p, q in zip(ps, qm):
        _bitwise(ctx.apply_operator(p), q, "on-the-fly (symmetric) vs materialized")
    if P.n <= 1000:
        K, _ = O.assemble(P.E, P.scale)
        for p in ps:
            _bitwise(ctx.apply_operator(p), O.apply(K, P.lam, p), "on-the-fly vs oracle O2")


@pytest.mark.parametrize("cid,n,kind", [(1, None, "jacobi"), (2, None, "learned"), (3, 777, "none")])
def test_otf_sym_pcg_staged_parity(ctx, L, cid, n, kind):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    if kind == "learned":
        Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
        ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_FACTORED)
        Q, M, ai = ctx.get_preconditioner_factors()
        ao, ro = oracle_pcg_factored(ctx, K, P.lam, P.y, Q, M, ai, tol=P.tol)
    elif kind == "jacobi":
        ctx.set_preconditioner(L.PRECOND_JACOBI)
        ao, ro = O.pcg(K, P.lam, P.y, O.P_JACOBI, O.jacobi_diag(P.E, P.scale, P.lam), tol=P.tol)
    else:
        ctx.set_preconditioner(L.PRECOND_NONE)
        ao, ro = O.pcg(K, P.lam, P.y, O.P_NONE, None, tol=P.tol)
    a, reps, _ = ctx.pcg_solve(P.y, P.tol)
    assert reps[0]["iters"] == ro.iters
    _bitwise(a, ao, "alpha")
