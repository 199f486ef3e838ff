"""GPU parity of the factored LEARNED preconditioner:
P = a^{-1/2} I + Q M Q^T kept as Q^T, Q and M (O4') and applied as
three Dot2 GEMV passes, theta = a^{-1/2} r + Q (M (Q^T r)).

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


@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (3, 2048), (3, 1000)])
def test_factored_staged_pcg_bitwise(ctx, L, cid, n):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    st = ctx.stats()
    assert rep["converged"] == 1 and st["p_factored"] in (1, 2) and st["n_dirs"] == P.n_dirs
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


@pytest.mark.parametrize("cid,n", [(2, None), (3, 1000)])
def test_factored_symmetric_M_staged_bitwise(ctx, L, monkeypatch, cid, n):
    """LAKER_MSYM=1: w = M z through the symmetric GEMV (M is formed bitwise
    symmetric) -- the same Dot2-exact row sums, so the staged parity stays bitwise."""
    monkeypatch.setenv("LAKER_MSYM", "1")
    monkeypatch.setenv("LAKER_P_3PASS", "1")  # the M pass exists only in the three-pass form
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    Q, M, ainv = ctx.get_preconditioner_factors()
    assert (M == M.T).all()
    K, _ = O.assemble(P.E, P.scale)
    ag, reps, hist = ctx.pcg_solve(P.y, P.tol, want_history=True)
    ao, ro = oracle_pcg_factored(ctx, K, P.lam, P.y, Q, M, ainv, tol=P.tol)
    assert reps[0]["iters"] == ro.iters
    _bitwise(hist, ro.history, "history")
    _bitwise(ag, ao, "alpha")


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


def test_factored_block_solve_T18(ctx, L, monkeypatch):
    """nrhs > 1 (block solve, C4 path) applies the factored P as three Dot2 GEMMs
    (Z = Q^T R, W = M Z, Theta = Q W + a^{-1/2} R): every column equals the
    single-RHS factored solve bitwise (T18) and solves the system (R14).  T18 is a
    property of the three-pass form (the QM opt-in, R21, is single-RHS only)."""
    monkeypatch.setenv("LAKER_P_3PASS", "1")
    P = make_problem(1)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(1, P.n, P.n_dirs))
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    assert ctx.stats()["p_factored"] in (1, 2)
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
