"""Parity at BASELINE.json's configuration sizes (VERDICT r01 "Next round" 1): the CUDA
path against the oracle on the full C3/C4 problems and on the C5 instruments that
SURVEY §8(c)/§8(d) M5 plan (the n = 8192, lambda = 1e-5 downscale through the
on-the-fly operator, and the T24 residual certificate at n = 65536).

* C3 staged (the bench workload: EXACT K, device-drawn Z with seed 7, factored P):
  the oracle's Alg. 1 with the GPU's P factors runs the whole solve;
  iteration count, residual history and alpha must be identical (protocol step 4).
* C3 own fit (harness Z): the oracle fits its own P (O4') and solves;
  alpha within 1e-6 (R14) and the GPU count inside the R15(iii) envelope: the
  oracle's own fit + solve on K and 8 copies of K with every entry moved +-1 ulp
  (seeded, symmetric), each with P applied in three passes and in the QM form (R21),
  [min - 2, max + 2].
* C4: 4 seeded columns of the 64-RHS LEARNED block solve, each identical to the
  single-RHS oracle solve with the same P (T18 + M5).
* C5 downscale (n = 8192, lambda = 1e-5, C5's generator): the on-the-fly EXACT
  operator (K never stored) against the oracle's materialized K --
  staged LAKER and Jacobi solves identical (T19); FAST on the fly within R14 of the
  oracle and inside its R15(iii) envelope taken at the FAST entries' error (1e-13
  relative perturbations of K instead of 1-ulp flips).
* T24 at n = 65536: the oracle's O2 residual of the GPU's alpha (FAST on-the-fly
  LAKER solve), ||(lambda I + K) alpha - y|| / ||y|| <= 10 tol, each row
  sum a correctly rounded oracle Dot2 of exact kernel entries.

The oracle runs minutes here (16 host cores); these tests carry the `slow` mark and
run in the driver's `-m gpu` suite."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

import oracle as O  # noqa: E402
from synth import make_problem, make_directions  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.fixture(scope="module")
def c3():
    P = make_problem(3)
    K, nov = O.assemble(P.E, P.scale)
    assert nov == 0
    return P, K


def _bitwise(a, b, what):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    bad = np.flatnonzero(a != b)
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}"


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



def _staged(K, lam, y, Q, M, ai, QM, **kw):
    """The oracle's PCG with the GPU's factored P, in the form the GPU applies it (QM form
    when the context exported a QM, else three passes; tests/staged.py)."""
    if QM is not None:
        return O.pcg_factored_qm(K, lam, y, Q, QM, ai, **kw)
    return O.pcg_factored(K, lam, y, Q, M, ai, **kw)


def _oracle_own(K, lam, y, Z, tol):
    """The oracle end to end with its own fit: O4' structured CCCP on Z, factored P,
    Alg. 1 PCG, with P applied in three passes and in the QM form of reading R21 (the
    oracle's own QM = Q M).  Returns (alpha of the three-pass solve, [iterations of both])."""
    _, rep, st = O.cccp_fit_structured(K, lam, Z, form_P=False)
    assert rep.converged
    Q, M, ai = O.factors(st)
    a, r = O.pcg_factored(K, lam, y, Q, M, ai, tol=tol)
    aq, rq = O.pcg_factored_qm(K, lam, y, Q, np.ascontiguousarray(Q @ M), ai, tol=tol)
    assert r.termination == O.TERM_RESIDUAL_TOL and rq.termination == O.TERM_RESIDUAL_TOL
    return a, [r.iters, rq.iters]


def test_c3_staged_full_solve(L, c3):
    """The bench workload (bench.py: EXACT, fit seed 7, factored P), whole solve."""
    P, K = c3
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        _bitwise(c.get_kernel_rows(), K, "C3 kernel matrix")
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        assert c.stats()["p_factored"] in (1, 2)
        Q, M, ai = c.get_preconditioner_factors()
        QM = c.get_preconditioner_qm()
        ag, rg, hg = c.pcg_solve(P.y, P.tol, want_history=True)
    finally:
        c.close()
    ao, ro = _staged(K, P.lam, P.y, Q, M, ai, QM, tol=P.tol)
    print(f"C3 staged: GPU {rg[0]['iters']} its, oracle {ro.iters} its")
    assert rg[0]["termination"] == ro.termination == O.TERM_RESIDUAL_TOL
    assert rg[0]["iters"] == ro.iters
    _bitwise(hg, ro.history, "C3 residual history")
    _bitwise(ag, ao, "C3 alpha")
    assert rg[0]["true_rel_residual"] == ro.true_rel_residual


def test_c3_own_fit_r14_r15(L, c3):
    P, K = c3
    Z = make_directions(3, P.n, P.n_dirs)
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=np.asfortranarray(Z))
        ag, rg, _ = c.pcg_solve(P.y, P.tol)
    finally:
        c.close()
    assert rg[0]["termination"] == L.TERM_RESIDUAL_TOL
    ao, it0 = _oracle_own(K, P.lam, P.y, Z, P.tol)
    err = np.linalg.norm(ag - ao) / np.linalg.norm(ao)
    its = list(it0)
    for s in range(8):
        its += _oracle_own(_flip_ulp(K, 1000 + s), P.lam, P.y, Z, P.tol)[1]
    print(f"C3 own fit: GPU {rg[0]['iters']} its, oracle {it0}, envelope {sorted(its)}, R14 {err:.2e}")
    assert err <= 1e-6
    assert _in_envelope(rg[0]["iters"], its), (rg[0]["iters"], its)


def test_c4_oracle_columns(L, c3):
    P3, K = c3
    P = make_problem(4)
    assert (P.E == P3.E).all()        # reading R5: C4 reuses C3's sensors and embeddings
    cols = np.sort(np.random.default_rng(25138).choice(P.Y.shape[1], 4, replace=False))
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        Q, M, ai = c.get_preconditioner_factors()
        QM = c.get_preconditioner_qm()
        A, reps, _ = c.pcg_solve(np.asfortranarray(P.Y), P.tol)
    finally:
        c.close()
    assert all(r["termination"] == L.TERM_RESIDUAL_TOL for r in reps)
    for j in cols:
        ao, ro = _staged(K, P.lam, np.ascontiguousarray(P.Y[:, j]), Q, M, ai, QM, tol=P.tol)
        print(f"C4 column {j}: GPU {reps[j]['iters']} its, oracle {ro.iters}")
        assert reps[j]["iters"] == ro.iters, j
        _bitwise(A[:, j], ao, f"C4 column {j}")
        assert reps[j]["true_rel_residual"] == ro.true_rel_residual


@pytest.fixture(scope="module")
def c5d():
    P = make_problem(5, n=8192)
    assert P.lam == 1e-5 and P.d == 64
    K, nov = O.assemble(P.E, P.scale)
    assert nov == 0
    return P, K


def test_c5_downscale_exact_on_the_fly(L, c5d):
    """T19 at the C5 regime: EXACT on the fly equals the oracle on the materialized K."""
    P, K = c5d
    nr = O.nr_schedule(P.n)
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
        rng = np.random.default_rng(8192)
        x = rng.standard_normal(P.n)
        _bitwise(c.apply_operator(x), O.apply(K, P.lam, x), "on-the-fly operator vs O2")
        c.set_preconditioner(L.PRECOND_JACOBI)
        aj, rj, hj = c.pcg_solve(P.y, P.tol, want_history=True)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=nr, seed=7)
        Q, M, ai = c.get_preconditioner_factors()
        QM = c.get_preconditioner_qm()
        al, rl, hl = c.pcg_solve(P.y, P.tol, want_history=True)
    finally:
        c.close()
    ao, ro = O.pcg(K, P.lam, P.y, O.P_JACOBI, O.jacobi_diag(P.E, P.scale, P.lam), tol=P.tol)
    print(f"C5 downscale Jacobi: GPU {rj[0]['iters']} its, oracle {ro.iters}")
    assert rj[0]["iters"] == ro.iters and ro.termination == O.TERM_RESIDUAL_TOL
    _bitwise(hj, ro.history, "Jacobi residual history")
    _bitwise(aj, ao, "Jacobi alpha")
    ao, ro = _staged(K, P.lam, P.y, Q, M, ai, QM, tol=P.tol)
    print(f"C5 downscale LAKER: GPU {rl[0]['iters']} its, oracle {ro.iters}")
    assert rl[0]["iters"] == ro.iters and ro.termination == O.TERM_RESIDUAL_TOL
    _bitwise(hl, ro.history, "LAKER residual history")
    _bitwise(al, ao, "LAKER alpha")


def _perturb_rel(K, seed, rel):
    """K with every entry scaled by (1 + rel xi), xi uniform in [-1, 1], symmetric: the
    R15(iii) perturbation at the size of the FAST entries' error (R15 FAST)."""
    n = K.shape[0]
    xi = np.random.default_rng(seed).uniform(-1.0, 1.0, (n, n))
    xi = np.triu(xi) + np.triu(xi, 1).T
    return K * (1.0 + rel * xi)


def test_c5_downscale_fast_on_the_fly(L, c5d):
    """FAST on the fly (tcgen05 QK^T + CUDA exp): operator within (1e-13 + n u) sum_j |K_ij x_j|
    of the exact O2 rows; the LAKER solve with its own fit within R14 of the oracle's own
    fit + solve and inside the R15(iii) envelope taken at FAST's own entry error: the
    oracle's own fit + solve on K and on 4 copies of K with every entry moved by up to
    1e-13 relative (seeded, symmetric), P in both application forms."""
    P, K = c5d
    nr = O.nr_schedule(P.n)
    Z = make_directions(5, P.n, nr)
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
        x = np.random.default_rng(8193).standard_normal(P.n)
        qf = c.apply_operator(x)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=nr, Z=np.asfortranarray(Z))
        af, rf, _ = c.pcg_solve(P.y, P.tol)
    finally:
        c.close()
    qo = O.apply(K, P.lam, x)
    # per-entry FAST error <= 1e-13 relative (test_gpu_otf) plus a recursive fp64 sum of n terms
    bound = (1e-13 + P.n * 2.0 ** -53) * (np.abs(K) @ np.abs(x) + P.lam * np.abs(x))
    assert (np.abs(qf - qo) <= bound).all()
    assert rf[0]["termination"] == L.TERM_RESIDUAL_TOL
    ao, it0 = _oracle_own(K, P.lam, P.y, Z, P.tol)
    err = np.linalg.norm(af - ao) / np.linalg.norm(ao)
    its = list(it0)
    for s in range(4):
        its += _oracle_own(_perturb_rel(K, 2000 + s, 1e-13), P.lam, P.y, Z, P.tol)[1]
    print(f"C5 downscale FAST: GPU {rf[0]['iters']} its, oracle envelope {sorted(its)}, R14 {err:.2e}")
    assert err <= 1e-6
    assert _in_envelope(rf[0]["iters"], its), (rf[0]["iters"], its)


def test_c5_certificate_T24(L):
    """n = 65536, lambda = 1e-5 (BASELINE configs[4]) on one GPU: FAST on-the-fly LAKER
    solve to 1e-8; the oracle recomputes the residual from exact kernel entries (its
    `predict` = one Dot2 per row of K alpha) -- a certificate the GPU cannot
    influence."""
    P = make_problem(5)
    assert P.n == 65536
    c = L.Context(0)
    try:
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=O.nr_schedule(P.n), seed=7)
        a, r, _ = c.pcg_solve(P.y, P.tol)
    finally:
        c.close()
    assert r[0]["termination"] == L.TERM_RESIDUAL_TOL
    Ka = O.predict(P.E, P.E, P.scale, a)          # K alpha, exact entries, Dot2 rows
    res = np.linalg.norm(P.lam * a + Ka - P.y) / np.linalg.norm(P.y)
    print(f"T24 at n=65536: GPU {r[0]['iters']} its, GPU true residual {r[0]['true_rel_residual']:.3e}, "
          f"oracle certificate {res:.3e}")
    assert res <= 10 * P.tol
