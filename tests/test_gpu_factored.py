"""GPU parity of the factored LEARNED preconditioner:
P = a^{-1/2} I + Q M Q^T kept as Q^T, Q and M (O4') and applied either
as three Dot2 GEMV passes, theta = a^{-1/2} r + Q (M (Q^T r)) (p_layout FACTORED),
or in the QM form a^{-1/2} r + (Q M)(Q^T r) (R21; AUTO / FACTORED_QM).

Staged parity (DESIGN.md §6 step 4): the oracle's PCG run with the GPU's own
factors (exported through laker_get_preconditioner_factors) on the same K takes
the same iterations with the same residual history and alpha, bitwise."""
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


LAYOUTS = {"3pass": (2, 1), "qm": (3, 2), "auto": (0, 2)}   # p_layout -> stats p_factored


@pytest.mark.parametrize("layout", ["3pass", "auto"])
@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (3, 2048), (3, 1000)])
def test_factored_staged_pcg_bitwise(ctx, L, cid, n, layout):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    pl, pf = LAYOUTS[layout]
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=pl)
    st = ctx.stats()
    assert rep["converged"] == 1 and st["p_factored"] == pf and st["n_dirs"] == P.n_dirs
    Q, M, ainv = ctx.get_preconditioner_factors()
    # Q has orthonormal columns (thin QR of Ubar) and M is symmetric
    assert np.abs(Q.T @ Q - np.eye(P.n_dirs)).max() <= 1e-10
    assert np.abs(M - M.T).max() <= 1e-9 * np.abs(M).max()
    K, _ = O.assemble(P.E, P.scale)
    ag, reps, hist = ctx.pcg_solve(P.y, P.tol, want_history=True)
    ao, ro = oracle_pcg_factored(ctx, K, P.lam, P.y, Q, M, ainv, tol=P.tol)
    assert reps[0]["termination"] == ro.termination == O.TERM_RESIDUAL_TOL
    assert reps[0]["iters"] == ro.iters
    _bitwise(hist, ro.history, "history")
    _bitwise(ag, ao, "alpha")
    if P.n <= 2048:
        ref = O.reference_solve(K, P.lam, P.y)
        assert np.linalg.norm(ag - ref) / np.linalg.norm(ref) <= 1e-6


@pytest.mark.parametrize("cid", [1, 2])
def test_qm_product_matches_factors(ctx, L, cid):
    """The QM form's n x N_r product (formed once at fit time by the int8-emulated GEMM,
    B8) is Q @ M of the exported factors to fp64-GEMM accuracy: a transposed, mis-padded
    or mis-sliced QM would fail here even though staged parity (which feeds the oracle
    the GPU's own QM) could not see it."""
    P = make_problem(cid)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    assert ctx.stats()["p_factored"] == 2
    Q, M, ainv = ctx.get_preconditioner_factors()
    QM = ctx.get_preconditioner_qm()
    ref = Q @ M
    assert np.abs(QM - ref).max() <= 1e-13 * np.abs(QM).max()
    # the three-pass fit of the same K and Z exports the same factors and no QM
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_FACTORED)
    assert ctx.stats()["p_factored"] == 1 and ctx.get_preconditioner_qm() is None
    Q3, M3, a3 = ctx.get_preconditioner_factors()
    assert (Q3 == Q).all() and (M3 == M).all() and a3 == ainv


def test_factored_equals_dense_layout_P(ctx, L):
    """The dense rows formed from the factors equal the rows of a DENSE-layout
    fit bitwise (same factors, same formation), and both solves converge to
    alpha within R14 of each other."""
    P = make_problem(2)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_DENSE)
    assert ctx.stats()["p_factored"] == 0 and ctx.stats()["symmetric_p"] == 1
    Pd = ctx.get_preconditioner_rows()
    ad, rd, _ = ctx.pcg_solve(P.y, P.tol)
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_FACTORED)
    assert ctx.stats()["p_factored"] in (1, 2)
    af, rf, _ = ctx.pcg_solve(P.y, P.tol)
    _bitwise(ctx.get_preconditioner_rows(), Pd, "P rows from factors vs dense layout")
    assert np.linalg.norm(af - ad) / np.linalg.norm(ad) <= 1e-6
    assert abs(rf[0]["iters"] - rd[0]["iters"]) <= 0.05 * rd[0]["iters"] + 2


@pytest.mark.parametrize("layout", ["3pass", "auto"])
def test_factored_block_solve_T18(ctx, L, layout):
    """nrhs > 1 (block solve, C4 path) applies the factored P in the single-RHS solve's
    form as Dot2 GEMMs (three passes: Z = Q^T R, W = M Z, Theta = Q W + a^{-1/2} R; QM
    form: Z = Q^T R, Theta = QM Z + a^{-1/2} R): every column equals the single-RHS
    factored solve bitwise (T18) and solves the system (R14)."""
    P = make_problem(1)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(1, P.n, P.n_dirs))
    pl, pf = LAYOUTS[layout]
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=pl)
    assert ctx.stats()["p_factored"] == pf
    Y = np.stack([P.y, -0.5 * P.y, np.roll(P.y, 7)], axis=1)
    A, reps, _ = ctx.pcg_solve(Y, P.tol)
    K, _ = O.assemble(P.E, P.scale)
    for j in range(Y.shape[1]):
        a1, r1, _ = ctx.pcg_solve(np.ascontiguousarray(Y[:, j]), P.tol)
        assert reps[j]["iters"] == r1[0]["iters"] and reps[j]["termination"] == L.TERM_RESIDUAL_TOL
        _bitwise(A[:, j], a1, f"block column {j}")
        ref = O.reference_solve(K, P.lam, Y[:, j])
        assert np.linalg.norm(A[:, j] - ref) / np.linalg.norm(ref) <= 1e-6


def test_factored_c3_full_size_certificate(ctx, L):
    """C3 (n = 16384, N_r = 4096), the bench workload: the factored solve
    converges with an oracle-computed residual certificate (T24), in fewer
    iterations than Jacobi; the first 3 iterations are bitwise the oracle's
    factored PCG on the GPU's factors."""
    P = make_problem(3)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.fit_preconditioner(L.PRECOND_LEARNED, seed=7)
    assert ctx.stats()["p_factored"] in (1, 2)
    Q, M, ainv = ctx.get_preconditioner_factors()
    K, _ = O.assemble(P.E, P.scale)
    a3, _, _ = ctx.pcg_solve(P.y, P.tol, max_iters=3)
    o3 = oracle_pcg_factored(ctx, K, P.lam, P.y, Q, M, ainv, tol=P.tol, max_iters=3)[0]
    _bitwise(a3, o3, "C3 alpha after 3 iterations")
    a, reps, _ = ctx.pcg_solve(P.y, P.tol)
    assert reps[0]["termination"] == L.TERM_RESIDUAL_TOL
    q = O.apply(K, P.lam, a)
    assert np.linalg.norm(q - P.y) / np.linalg.norm(P.y) <= 10 * P.tol
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    _, rj, _ = ctx.pcg_solve(P.y, P.tol)
    assert reps[0]["iters"] < rj[0]["iters"]
