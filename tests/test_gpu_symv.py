"""GPU parity of the symmetric (block upper-triangle) Dot2 GEMV, csrc/symv.cu
(rows a4/a7/a9).  K is symmetric (P:141-147 with q = k,
reading R2) and the learned P = Sigma*^{-1/2} is formed bitwise symmetric
(B4), so each operator / preconditioner apply reads only half the
matrix.  Bars: every row of y = (lambda I + A) x is bitwise the oracle's Dot2 row
(O2) and bitwise the full-row GEMV's (gemv.cu, selected with LAKER_SYMV=0); the
path is selected only when the matrix is bitwise symmetric.
"""
import os

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


def _bitwise(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    bad = np.flatnonzero(a.ravel() != b.ravel())
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}"


def _vectors(n, seed):
    r = np.random.default_rng(seed)
    return [r.standard_normal(n),
            np.where(np.arange(n) % 3 == 0, 1.0, -1.0) * np.exp(r.uniform(-10, 10, n))]


def _with_symv_off(fn):
    old = os.environ.get("LAKER_SYMV")
    os.environ["LAKER_SYMV"] = "0"
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["LAKER_SYMV"]
        else:
            os.environ["LAKER_SYMV"] = old


# sizes: one tile, one block-row, ragged tails of both, several block-rows whose
# segments span many CTAs (n = 2048: ~3.7 tiles per CTA), and a non-multiple of 32
@pytest.mark.parametrize("n", [1, 2, 31, 33, 127, 128, 129, 257, 1000, 2048, 4133])
def test_symv_apply_bitwise_vs_oracle_and_full_gemv(ctx, L, n):
    P = make_problem(3, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert ctx.stats()["symmetric_k"] == 1
    Ko, _ = O.assemble(P.E, P.scale)
    xs = _vectors(n, 100 + n)
    ys = [ctx.apply_operator(x) for x in xs]
    for x, y in zip(xs, ys):
        _bitwise(y, O.apply(Ko, P.lam, x), f"symv vs oracle n={n}")

    def full():
        ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        assert ctx.stats()["symmetric_k"] == 0
        return [ctx.apply_operator(x) for x in xs]
    for y, yf in zip(ys, _with_symv_off(full)):
        _bitwise(y, yf, f"symv vs gemv n={n}")


def test_symv_loaded_symmetric_cancellation(ctx, L):
    """A loaded symmetric matrix with both signs and 1e+-6 magnitudes (heavy
    cancellation in every row): bitwise = oracle Dot2."""
    n = 1500
    r = np.random.default_rng(21)
    A = r.standard_normal((n, n)) * np.exp(r.uniform(-6, 6, (n, n)))
    A = np.triu(A) + np.triu(A, 1).T
    P = make_problem(1, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    ctx.load_kernel_rows(A)
    assert ctx.stats()["symmetric_k"] == 1
    for x in _vectors(n, 5):
        _bitwise(ctx.apply_operator(x), O.apply(A, P.lam, x), "loaded symmetric")


def test_symv_not_used_for_nonsymmetric(ctx, L):
    n = 700
    P = make_problem(1, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    A = K.copy()
    A[3, 600] = np.nextafter(A[3, 600], 2.0)  # one ulp breaks bitwise symmetry
    ctx.load_kernel_rows(A)
    assert ctx.stats()["symmetric_k"] == 0
    x = _vectors(n, 6)[0]
    _bitwise(ctx.apply_operator(x), O.apply(A, P.lam, x), "non-symmetric falls back to gemv")


def test_symv_pcg_learned_gpu_fit(ctx, L):
    """GPU-fitted dense P is bitwise symmetric -> both applies use symv; the staged
    PCG (same K, the GPU's own P) equals the oracle's PCG bitwise."""
    P = make_problem(2)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))
    ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_DENSE)
    st = ctx.stats()
    assert st["symmetric_k"] == 1 and st["symmetric_p"] == 1 and st["p_factored"] == 0
    Pm = ctx.get_preconditioner_rows()
    K, _ = O.assemble(P.E, P.scale)
    ag, reps, hist = ctx.pcg_solve(P.y, P.tol, want_history=True)
    ao, ro = O.pcg(K, P.lam, P.y, O.P_DENSE, Pm, tol=P.tol)
    assert reps[0]["iters"] == ro.iters and reps[0]["termination"] == ro.termination
    _bitwise(hist, ro.history, "history")
    _bitwise(ag, ao, "alpha")


def test_symv_c3_full_size_pcg_matches_full_gemv(ctx, L):
    """C3 (n = 16384, the bench workload), Jacobi: the symv solve and the
    full-row GEMV solve take the same iterations and give the same alpha bitwise
    (every row of every apply is the correctly rounded row sum in both)."""
    P = make_problem(3)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert ctx.stats()["symmetric_k"] == 1
    ctx.set_preconditioner(L.PRECOND_JACOBI)
    a1, r1, h1 = ctx.pcg_solve(P.y, P.tol, want_history=True)

    def full():
        ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        ctx.set_preconditioner(L.PRECOND_JACOBI)
        return ctx.pcg_solve(P.y, P.tol, want_history=True)
    a2, r2, h2 = _with_symv_off(full)
    assert r1[0]["iters"] == r2[0]["iters"]
    _bitwise(h1, h2, "C3 history")
    _bitwise(a1, a2, "C3 alpha")


def _with_env(name, value, fn):
    old = os.environ.get(name)
    os.environ[name] = value
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old


# The exact int8 tensor-core form of the same apply (csrc/symv_tc.cu): K's entries are
# exact in 8 seven-bit digit slices with one exponent, so every tile product is an exact
# integer sum and each row is again the unrounded pair the finalize rounds once.  Bars:
# it is selected for the configs' K, and every row is bitwise the oracle's and the fp64
# symmetric kernel's (LAKER_SYMV_TC=0).
@pytest.mark.parametrize("cfg,n", [(1, None), (2, None), (3, 1), (3, 65), (3, 129), (3, 1000), (3, 2048),
                                   (3, 4133), (4, 3000), (5, 2500)])
def test_symv_tensor_core_bitwise(ctx, L, cfg, n):
    P = make_problem(cfg, n=n) if n else make_problem(cfg)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    st = ctx.stats()
    assert st["symmetric_k"] == 1 and st["k_tensor_core"] == 1
    Ko, _ = O.assemble(P.E, P.scale)
    xs = _vectors(P.n, 300 + P.n) + [np.zeros(P.n)]
    ys = [ctx.apply_operator(x) for x in xs]
    for x, y in zip(xs, ys):
        _bitwise(y, O.apply(Ko, P.lam, x), f"tensor-core symv vs oracle cfg={cfg} n={P.n}")

    def fp64():
        ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        assert ctx.stats()["k_tensor_core"] == 0
        return [ctx.apply_operator(x) for x in xs]
    for y, yf in zip(ys, _with_env("LAKER_SYMV_TC", "0", fp64)):
        _bitwise(y, yf, f"tensor-core vs fp64 symv n={P.n}")


def test_symv_tensor_core_not_used_when_inexact(ctx, L):
    """A K entry off the 8-slice grid (an odd multiple of 2^-55 while max |K| in [2, 4)
    puts the grid at 2^(eK-55) = 2^-53) keeps the fp64 kernel."""
    n = 600
    P = make_problem(1, n=n)
    ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    K, _ = O.assemble(P.E, P.scale)
    A = K.copy()
    assert 2.0 <= K.max() < 4.0
    A[5, 400] = A[400, 5] = np.ldexp(float(2 ** 52 + 1), -55)
    ctx.load_kernel_rows(A)
    st = ctx.stats()
    assert st["symmetric_k"] == 1 and st["k_tensor_core"] == 0
    x = _vectors(n, 8)[0]
    _bitwise(ctx.apply_operator(x), O.apply(A, P.lam, x), "inexact K -> fp64 symv")


def test_symv_tensor_core_c3_pcg_matches_fp64(ctx, L):
    """C3 (n = 16384), the default learned solve: the tensor-core apply and the fp64
    symmetric apply give the same history and alpha bitwise."""
    P = make_problem(3)
    Z = np.asfortranarray(make_directions(3, P.n, P.n_dirs))

    def run():
        ctx.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        tc = ctx.stats()["k_tensor_core"]
        ctx.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
        a, r, h = ctx.pcg_solve(P.y, P.tol, want_history=True)
        return tc, a, r, h
    tc1, a1, r1, h1 = run()
    tc0, a0, r0, h0 = _with_env("LAKER_SYMV_TC", "0", run)
    assert tc1 == 1 and tc0 == 0
    assert r1[0]["iters"] == r0[0]["iters"]
    _bitwise(h1, h0, "C3 history")
    _bitwise(a1, a0, "C3 alpha")
