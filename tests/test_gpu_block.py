"""Multi-RHS block PCG (row a10, config C4, reading R13): every column of the
block solve equals the single-RHS solve of that column (EXACT: bitwise, T18);
FAST (DMMA GEMM applies) within the R14 solution tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
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


@pytest.mark.parametrize("kind", ["none", "jacobi", "learned"])
def test_block_equals_single_columns_T18(ctx, L, kind):
    P = make_problem(4, n=1024, nrhs=6, tol=1e-8)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    if kind == "jacobi":
        ctx.set_preconditioner(L.PRECOND_JACOBI)
    elif kind == "learned":
        Z = np.asfortranarray(make_directions(4, P.n, P.n_dirs))
        ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    Y = np.asfortranarray(P.Y)
    Y[:, 3] = 0.0                      # a zero column terminates at once (ZERO_RHS)
    A, reps, _ = ctx.pcg_solve(Y, P.tol)
    for c in range(Y.shape[1]):
        a1, r1, _ = ctx.pcg_solve(np.ascontiguousarray(Y[:, c]), P.tol)
        assert reps[c]["iters"] == r1[0]["iters"] and reps[c]["termination"] == r1[0]["termination"]
        assert (A[:, c] == a1).all(), c
        assert reps[c]["true_rel_residual"] == r1[0]["true_rel_residual"]
    assert reps[3]["termination"] == L.TERM_ZERO_RHS and (A[:, 3] == 0).all()


def test_block_oracle_columns(ctx, L):
    P = make_problem(4, n=512, nrhs=4, tol=1e-8)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    A, reps, _ = ctx.pcg_solve(np.asfortranarray(P.Y), P.tol)
    K, _ = O.assemble(P.E, P.scale)
    d = O.jacobi_diag(P.E, P.scale, P.lam)
    for c in range(4):
        ao, ro = O.pcg(K, P.lam, P.Y[:, c], O.P_JACOBI, d, tol=P.tol)
        assert ro.iters == reps[c]["iters"] and (ao == A[:, c]).all()


def test_block_fast_mode(ctx, L):
    P = make_problem(4, n=2048, nrhs=8, tol=1e-8)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_FAST)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    A, reps, _ = ctx.pcg_solve(np.asfortranarray(P.Y), P.tol)
    K, _ = O.assemble(P.E, P.scale)
    for c in range(8):
        ref = O.reference_solve(K, P.lam, P.Y[:, c])
        assert reps[c]["termination"] == L.TERM_RESIDUAL_TOL
        assert np.linalg.norm(A[:, c] - ref) / np.linalg.norm(ref) <= 1e-6


@pytest.mark.parametrize("kind", ["jacobi", "learned"])
def test_block_fast_tensor_core_products(ctx, L, kind):
    """FAST block solve with its products on the tcgen05 int8 tensor cores
    (ozaki_skinny.cu: K and the P factors sliced once per solve, S = 7 digit
    slices): every column converges and solves the system to R14 and agrees
    with the DMMA products (LAKER_BLOCK_TC=0) to R14.  Iteration counts are
    FAST-mode envelope quantities (R15 iii): the S = 7 products carry ~2^-48
    of each column's max |x| (vs the DMMA GEMM's ~K u sum |k||x|), which at
    kappa ~ 1e7 (Jacobi) costs up to ~25% more iterations; bounded here at 35%."""
    import os
    P = make_problem(4, n=2048, nrhs=16, tol=1e-8)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_FAST)
    if kind == "learned":
        Z = np.asfortranarray(make_directions(4, P.n, P.n_dirs))
        ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    else:
        ctx.set_preconditioner(L.PRECOND_JACOBI)
    A, reps, _ = ctx.pcg_solve(np.asfortranarray(P.Y), P.tol)
    os.environ["LAKER_BLOCK_TC"] = "0"
    try:
        A0, reps0, _ = ctx.pcg_solve(np.asfortranarray(P.Y), P.tol)
    finally:
        del os.environ["LAKER_BLOCK_TC"]
    K, _ = O.assemble(P.E, P.scale)
    for c in range(P.Y.shape[1]):
        ref = O.reference_solve(K, P.lam, P.Y[:, c])
        assert reps[c]["termination"] == L.TERM_RESIDUAL_TOL
        assert np.linalg.norm(A[:, c] - ref) / np.linalg.norm(ref) <= 1e-6
        assert np.linalg.norm(A[:, c] - A0[:, c]) / np.linalg.norm(A0[:, c]) <= 1e-6
        assert abs(reps[c]["iters"] - reps0[c]["iters"]) <= 0.35 * reps0[c]["iters"] + 3
