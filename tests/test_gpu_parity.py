"""GPU parity: the CUDA path (through the C ABI, liblaker.so) against the fp64
oracle on the same seeded inputs.  Bars:
  * kernel entries (EXACT) and every Dot2 product/reduction: bitwise;
  * PCG on shared K and P (staged): identical iteration count and residual
    history, alpha bitwise;
  * FAST-mode entries: <= 1e-13 relative;
  * full BASELINE sizes: sampled rows / properties.
"""
import math

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


def _assert_bitwise(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    bad = np.flatnonzero(a.ravel() != b.ravel())
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]} {a.ravel()[bad[:3]]} vs {b.ravel()[bad[:3]]}"


# --------------------------------------------------------------- assembly
def test_exp_cr_through_assembly(ctx, L):
    """K_ij = exp(e_i e_j) with d = 1 spans ~260k distinct arguments in [-1, 1]."""
    r = np.random.default_rng(11)
    E = np.ascontiguousarray(r.uniform(-1, 1, (720, 1)))
    ctx.assemble_kernel(E, 1.0, 1e-3, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Kg = ctx.get_kernel_rows()
    Ko, _ = O.assemble(E, 1.0)
    _assert_bitwise(Kg, Ko, "exp_cr")
    assert ctx.stats()["exp_inconclusive"] == 0


@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (3, 1000), (3, 257)])
def test_assemble_exact_bitwise(ctx, L, cid, n):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Kg = ctx.get_kernel_rows()
    Ko, _ = O.assemble(P.E, P.scale)
    _assert_bitwise(Kg, Ko, f"K C{cid} n={P.n}")
    assert (Kg == Kg.T).all()


def test_assemble_fast_close(ctx, L):
    P = make_problem(2)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_FAST)
    Kf = ctx.get_kernel_rows()
    Ko, _ = O.assemble(P.E, P.scale)
    assert np.abs(Kf / Ko - 1).max() <= 1e-13
    assert (Kf == Kf.T).all()


def test_assemble_c3_full_size_sampled_rows(ctx, L):
    P = make_problem(3)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Kg = ctx.get_kernel_rows()
    assert (Kg == Kg.T).all()
    for r0 in (0, 8191, P.n - 3):
        _assert_bitwise(Kg[r0:r0 + 3], O.assemble_rows(P.E, P.scale, r0, r0 + 3), f"C3 rows {r0}")
    # operator apply on sampled rows vs the oracle's Dot2 row sums
    p = np.random.default_rng(3).standard_normal(P.n) * 1e3
    q = ctx.apply_operator(p)
    for i in (0, 4097, P.n - 1):
        Krow = O.assemble_rows(P.E, P.scale, i, i + 1)[0]
        ref = O.dot2(np.concatenate([[P.lam], Krow]), np.concatenate([[p[i]], p]))
        assert q[i] == ref


# ---------------------------------------------------------------- operator
@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (3, 1000), (1, 1), (1, 2)])
def test_apply_operator_bitwise(ctx, L, cid, n):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Ko, _ = O.assemble(P.E, P.scale)
    r = np.random.default_rng(7)
    for p in (r.standard_normal(P.n), np.where(np.arange(P.n) % 2 == 0, 1.0, -1.0) * np.exp(r.uniform(-8, 8, P.n))):
        _assert_bitwise(ctx.apply_operator(p), O.apply(Ko, P.lam, p), "apply")


def test_on_the_fly_equals_materialized_T19(ctx, L):
    P = make_problem(1)
    p = np.random.default_rng(5).standard_normal(P.n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    qm = ctx.apply_operator(p)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
    qf = ctx.apply_operator(p)
    _assert_bitwise(qf, qm, "on-the-fly vs materialized")


# --------------------------------------------------------------------- PCG
def _solve_both(ctx, L, P, K, kind, Pm=None, max_iters=0):
    if kind == O.P_NONE:
        ctx.set_preconditioner(L.PRECOND_NONE)
    elif kind == O.P_JACOBI:
        ctx.set_preconditioner(L.PRECOND_JACOBI)  # derived on the GPU from E
    else:
        ctx.set_preconditioner(L.PRECOND_EXTERNAL_DENSE, Pm)
    ag, reps, hist = ctx.pcg_solve(P.y, P.tol, max_iters=max_iters, want_history=True)
    ao, ro = O.pcg(K, P.lam, P.y, kind, Pm, tol=P.tol, max_iters=max_iters or None)
    return ag, reps[0], hist, ao, ro


@pytest.mark.parametrize("cid,n,kind", [(1, None, O.P_NONE), (1, None, O.P_JACOBI), (2, None, O.P_NONE),
                                        (2, None, O.P_JACOBI), (3, 4096, O.P_JACOBI), (3, 777, O.P_NONE)])
def test_pcg_staged_parity(ctx, L, cid, n, kind):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    Pm = O.jacobi_diag(P.E, P.scale, P.lam) if kind == O.P_JACOBI else None
    ag, rg, hist, ao, ro = _solve_both(ctx, L, P, K, kind, Pm)
    assert rg["termination"] == ro.termination == O.TERM_RESIDUAL_TOL
    assert rg["iters"] == ro.iters
    _assert_bitwise(hist, ro.history, "residual history")
    _assert_bitwise(ag, ao, "alpha")
    assert rg["true_rel_residual"] == ro.true_rel_residual


@pytest.mark.parametrize("cid,n", [(1, None), (3, 1024)])
def test_pcg_learned_dense_staged_parity(ctx, L, cid, n):
    """P from the oracle's CCCP fit, loaded through laker_set_preconditioner."""
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    Z = make_directions(cid, P.n, P.n_dirs)
    Pm = O.cccp_fit_structured(K, P.lam, Z)[0]
    ag, rg, hist, ao, ro = _solve_both(ctx, L, P, K, O.P_DENSE, np.ascontiguousarray(Pm))
    assert rg["iters"] == ro.iters and rg["termination"] == ro.termination
    _assert_bitwise(hist, ro.history, "history")
    _assert_bitwise(ag, ao, "alpha")
    ref = O.reference_solve(K, P.lam, P.y)
    assert np.linalg.norm(ag - ref) / np.linalg.norm(ref) <= 1e-6


def test_pcg_edge_cases(ctx, L):
    P = make_problem(1)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.set_preconditioner(L.PRECOND_NONE)
    a, reps, _ = ctx.pcg_solve(np.zeros(P.n), 1e-10)
    assert reps[0]["termination"] == L.TERM_ZERO_RHS and reps[0]["iters"] == 0 and (a == 0).all()
    a, reps, _ = ctx.pcg_solve(P.y, 1e-10, max_iters=5)
    assert reps[0]["termination"] == L.TERM_MAX_ITERS and reps[0]["iters"] == 5
    K, _ = O.assemble(P.E, P.scale)
    ao, ro = O.pcg(K, P.lam, P.y, O.P_NONE, None, tol=1e-10, max_iters=5)
    _assert_bitwise(a, ao, "alpha after 5")
    ctx.set_preconditioner(L.PRECOND_JACOBI, -np.ones(P.n))
    with pytest.raises(L.LakerError) as e:
        ctx.pcg_solve(P.y, 1e-10)
    assert e.value.status == 8
    with pytest.raises(L.LakerError):
        ctx.pcg_solve(P.y, 1.5)


def test_n_equals_one(ctx, L):
    E = np.array([[0.6, 0.8]])
    ctx.assemble_kernel(E, 1.0, 0.5, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K = ctx.get_kernel_rows()
    assert K[0, 0] == O.exp_cr(1.0)
    ctx.set_preconditioner(L.PRECOND_NONE)
    a, reps, _ = ctx.pcg_solve(np.array([3.0]), 1e-12)
    assert reps[0]["iters"] == 1
    assert a[0] == O.pcg(K, 0.5, np.array([3.0]), tol=1e-12)[0][0]


def test_device_buffers_match_host(ctx, L):
    import torch
    P = make_problem(1)
    Ed = torch.from_numpy(P.E).cuda()
    ctx.assemble_kernel(Ed, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    ad, _, _ = ctx.pcg_solve(torch.from_numpy(P.y).cuda(), P.tol)
    ah, _, _ = ctx.pcg_solve(P.y, P.tol)
    _assert_bitwise(ad.cpu().numpy(), ah, "device vs host")


# ----------------------------------------------------------------- predict
def test_predict_same_alpha_bitwise_R16(ctx, L):
    P = make_problem(1)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    alpha = O.pcg(K, P.lam, P.y, O.P_NONE, None, tol=P.tol)[0]
    rg = ctx.predict(P.Eq, alpha)
    ro = O.predict(P.Eq, P.E, P.scale, alpha)
    _assert_bitwise(rg, ro, "map")
    # at training points the map reproduces K alpha = y - lambda alpha - r (T17)
    rt = ctx.predict(P.E, alpha)
    assert np.abs(rt - (P.y - P.lam * alpha)).max() <= 1e-6 * np.abs(P.y).max()


def test_predict_c2_subgrid(ctx, L):
    P = make_problem(2)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    alpha = np.random.default_rng(9).standard_normal(P.n) * 1e5
    idx = np.arange(0, P.Eq.shape[0], 37)
    Eq = np.ascontiguousarray(P.Eq[idx])
    _assert_bitwise(ctx.predict(Eq, alpha), O.predict(Eq, P.E, P.scale, alpha), "map C2")


# ------------------------------------------------------ full-size certificate
def test_c3_full_size_solve_certificate(ctx, L):
    """C3 (n = 16384, Jacobi): the first 3 iterations are bitwise the oracle's;
    the converged alpha has an oracle-computed residual <= 10 tol (T24)."""
    P = make_problem(3)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    d = O.jacobi_diag(P.E, P.scale, P.lam)
    a3, _, _ = ctx.pcg_solve(P.y, P.tol, max_iters=3)
    o3 = O.pcg(K, P.lam, P.y, O.P_JACOBI, d, tol=P.tol, max_iters=3)[0]
    _assert_bitwise(a3, o3, "C3 alpha after 3 iterations")
    a, reps, _ = ctx.pcg_solve(P.y, P.tol)
    assert reps[0]["termination"] == L.TERM_RESIDUAL_TOL
    q = O.apply(K, P.lam, a)
    assert np.linalg.norm(q - P.y) / np.linalg.norm(P.y) <= 10 * P.tol
