"""GPU CCCP fit (laker_fit_preconditioner, LEARNED) against the oracle's
structured fit on the same Z (DESIGN.md §6 parity protocol step 3: P within
1e-8 relative Frobenius, CCCP steps +-1), plus properties at full size."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_problem, make_directions, make_paper_problem  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.fixture(scope="module")
def ctx(L):
    c = L.Context(0)
    yield c
    c.close()


def _fit_both(ctx, L, cid, n=None):
    P = make_problem(cid, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    Pg = ctx.get_preconditioner_rows()
    Po, ro, st = O.cccp_fit_structured(K, P.lam, Z)
    return P, K, Pg, rep, Po, ro, st


# (4, 2048): a draw of Z on which the coupled Newton-Schulz alone diverged after
# reaching ||W - I|| ~ 6e-6 (fixed by the guarded uncoupled refinement, fit.cu)
@pytest.mark.parametrize("cid,n", [(1, None), (2, None), (3, 2048), (3, 1000), (4, 2048)])
def test_fit_matches_oracle(ctx, L, cid, n):
    P, K, Pg, rep, Po, ro, st = _fit_both(ctx, L, cid, n)
    assert rep["converged"] == 1 and ro.converged
    assert abs(rep["iters"] - ro.iters) <= 1
    assert abs(rep["sigma_min_eig"] / ro.sigma_min_eig - 1) <= 1e-8
    assert abs(rep["trace"] / P.n - 1) <= 1e-8
    assert rep["rho_used"] == ro.rho_used
    assert (Pg == Pg.T).all()   # B4: (W Q^T + Q W^T)/2 is symmetric bitwise
    assert np.linalg.norm(Pg - Po) / np.linalg.norm(Po) <= 1e-8


def _flip_ulp(K, seed):
    """K with every entry moved one ulp up or down at random, symmetric (R15 iii)."""
    n = K.shape[0]
    up = np.random.default_rng(seed).random((n, n)) < 0.5
    up = np.triu(up) | np.triu(up, 1).T
    return np.where(up, np.nextafter(K, np.inf), np.nextafter(K, -np.inf))

def _in_envelope(count, its):
    """R15(iii): the GPU's count against the oracle's own counts under perturbations of the
    size of the GPU's deviation -- inside [min - 2, max + 2] of the sample, or within three
    standard deviations of its mean (a ~1000-iteration count moves by tens under any
    last-bit change, so a sample of ~10-18 runs does not reach the distribution's tails)."""
    its = np.asarray(its, dtype=np.float64)
    return bool(min(its) - 2 <= count <= max(its) + 2 or abs(count - its.mean()) <= 3.0 * its.std(ddof=1))



def _oracle_own_iters(K, lam, y, Z, tol):
    """The oracle's own fit + solve in both application forms of the factored P (three
    passes Q (M (Q^T r)), and the QM form of reading R21 the GPU applies by default, with
    the oracle's own QM = Q M): two members of the R15(iii) envelope."""
    _, rep, st = O.cccp_fit_structured(K, lam, Z, form_P=False)
    Q, M, ai = O.factors(st)
    QM = np.ascontiguousarray(Q @ M)
    return [O.pcg_factored(K, lam, y, Q, M, ai, tol=tol)[1].iters,
            O.pcg_factored_qm(K, lam, y, Q, QM, ai, tol=tol)[1].iters]


@pytest.mark.parametrize("cid,n", [(1, None), (2, None)])
def test_learned_pcg_end_to_end(ctx, L, cid, n):
    """End-to-end (own fit, own K, the default QM-form P): alpha within 1e-6 of Cholesky
    (R14), iteration count inside the R15(iii) envelope -- the oracle's own fit + solve on
    K and 8 copies of K with every entry moved +-1 ulp (seeded, symmetric), each solved
    with P applied in both forms (three passes and QM, reading R21), [min-2, max+2] --
    and fewer iterations than Jacobi (T21).  The B5 envelope of round 1 (the oracle's P
    perturbed at the measured GPU deviation) is printed beside it for the record."""
    P, K, Pg, rep, Po, ro, st = _fit_both(ctx, L, cid, n)
    Z = make_directions(cid, P.n, P.n_dirs)
    ag, reps, _ = ctx.pcg_solve(P.y, P.tol)
    ref = O.reference_solve(K, P.lam, P.y)
    assert reps[0]["termination"] == L.TERM_RESIDUAL_TOL
    assert np.linalg.norm(ag - ref) / np.linalg.norm(ref) <= 1e-6
    its = _oracle_own_iters(K, P.lam, P.y, Z, P.tol)
    for s in range(8):
        its += _oracle_own_iters(_flip_ulp(K, 500 + s), P.lam, P.y, Z, P.tol)
    r = np.random.default_rng(0)
    dev = max(np.linalg.norm(Pg - Po) / np.linalg.norm(Po), 2.0 ** -52)
    b5 = []
    for s in range(4):
        Pp = Po * (1 + (dev if s % 2 == 0 else 2.0 ** -52) * r.standard_normal(Po.shape))
        Pp = np.triu(Pp) + np.triu(Pp, 1).T
        b5.append(O.pcg(K, P.lam, P.y, O.P_DENSE, Pp, tol=P.tol)[1].iters)
    print(f"C{cid} own fit: GPU {reps[0]['iters']} its; R15(iii) K-flip envelope {sorted(its)}; "
          f"B5 P-perturbation envelope {sorted(b5)}")
    assert _in_envelope(reps[0]["iters"], its), (reps[0]["iters"], its)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    _, rj, _ = ctx.pcg_solve(P.y, P.tol)
    assert reps[0]["iters"] < rj[0]["iters"]


def test_fit_device_rng_and_invariants(ctx, L):
    P = make_problem(2)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, seed=123)
    assert rep["converged"] == 1 and rep["n_dirs"] == O.nr_schedule(P.n)
    Pg = ctx.get_preconditioner_rows()
    assert (Pg == Pg.T).all()   # B4: (W Q^T + Q W^T)/2 is symmetric bitwise
    w = np.linalg.eigvalsh(Pg)
    assert w[0] > 0
    # P = Sigma^{-1/2} with Sigma ~ (lambda I + K)^2 up to scale: kappa(P A) << kappa(A)
    K, _ = O.assemble(P.E, P.scale)
    A = K + P.lam * np.eye(P.n)
    assert O.cond_precond(Pg, A) <= O.cond_spd(A) / 50
    rep2 = ctx.fit_preconditioner(L.PRECOND_LEARNED, seed=123)
    assert (ctx.get_preconditioner_rows() == Pg).all() and rep2["iters"] == rep["iters"]   # deterministic


def test_fit_c3_full_size(ctx, L):
    """C3 (n = 16384, N_r = 4096): GPU fit vs the oracle's structured fit on the
    same Z, sampled rows of P; then LEARNED PCG converges in fewer iterations
    than Jacobi."""
    P = make_problem(3)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(3, P.n, P.n_dirs))
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    assert rep["converged"] == 1
    Pg = ctx.get_preconditioner_rows()
    K, _ = O.assemble(P.E, P.scale)
    Po, ro, _ = O.cccp_fit_structured(K, P.lam, Z)
    assert abs(rep["iters"] - ro.iters) <= 1
    assert abs(rep["sigma_min_eig"] / ro.sigma_min_eig - 1) <= 1e-8
    rows = np.array([0, 1, 4097, 8191, P.n - 1])
    assert np.linalg.norm(Pg[rows] - Po[rows]) / np.linalg.norm(Po[rows]) <= 1e-8
    del Po
    _, rl, _ = ctx.pcg_solve(P.y, P.tol)
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    _, rj, _ = ctx.pcg_solve(P.y, P.tol)
    assert rl[0]["termination"] == rj[0]["termination"] == L.TERM_RESIDUAL_TOL
    assert rl[0]["iters"] < rj[0]["iters"]


@pytest.mark.parametrize("n", [50, 64])
def test_fit_full_rank_directions_matches_oracle(ctx, L, n):
    """N_r = n (the paper regime's small n, "when N_r >= n"): Sigma_t = Q T_t Q^T with
    Q square, so the R6 trigger reads lambda_min(T_t), not a_t; GPU and oracle must take
    the same rho at every step and reach the same P."""
    P = make_paper_problem(n)
    assert P.n_dirs == n
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    Z = np.asfortranarray(make_directions(0, P.n, P.n_dirs))
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    Po, ro, st = O.cccp_fit_structured(K, P.lam, Z)
    assert rep["converged"] == 1 and ro.converged
    assert abs(rep["iters"] - ro.iters) <= 1
    assert rep["rho_used"] == ro.rho_used
    Pg = ctx.get_preconditioner_rows()
    assert np.linalg.norm(Pg - Po) / np.linalg.norm(Po) <= 1e-8


def test_fit_rho_trigger_full_rank_reads_lambda_min_T(ctx, L):
    """N_r = n with gamma = 1e-7, rho_floor = 1e-9 on a well-conditioned K: a_t ~ 1e-7 stays
    below the R6 threshold 1e-6 while lambda_min(Sigma_t) = lambda_min(T_t) ~ 6e-5 does not,
    so the trigger must not fire (rho stays 1e-9 on both sides; a trigger read from a_t
    would set rho = 0.2 at every step)."""
    n = 48
    r = np.random.default_rng(7)
    B = r.standard_normal((n, n))
    K = B @ B.T / n + 0.5 * np.eye(n)
    K = 0.5 * (K + K.T)
    Z = r.standard_normal((n, n))
    E = np.zeros((n, 4))
    ctx.assemble_kernel(E, 1.0, 0.1, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.load_kernel_rows(K)
    kw = dict(gamma=1e-7, rho_floor=1e-9, max_iters=30)
    rep = ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=n, Z=np.asfortranarray(Z), **kw)
    Po, ro, st = O.cccp_fit_structured(K, 0.1, Z, **kw)
    assert ro.rhos == [1e-9] * 30 and st.a < 1e-6 < ro.sigma_min_eig
    assert rep["iters"] == ro.iters == 30
    assert rep["rho_used"] == 1e-9
    Pg = ctx.get_preconditioner_rows()
    assert np.linalg.norm(Pg - Po) / np.linalg.norm(Po) <= 1e-8
