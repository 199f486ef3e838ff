"""EXACT parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (C3: n = 16384, K materialized, symmetric apply; C4: 64 right-hand sides).

The hot K apply accumulates with the offset-Fast2Sum scheme (symv.cu, pcg_block.cu),
whose error bound grows with the products per accumulator; these checks pin it where
the small parity cases cannot: at n = 16384 the symmetric apply equals the full-row
Dot2 GEMV bitwise and the oracle's O2 row sums on sampled rows, and the
block EXACT products equal the Dot2 block products bitwise over several iterations."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_problem  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


def _bitwise(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    bad = np.flatnonzero(a.ravel() != b.ravel())
    assert bad.size == 0, f"{what}: {bad.size} mismatches, first {bad[:5]}"


def test_c3_symmetric_apply_fullsize(L, monkeypatch):
    P = make_problem(3)
    n = P.n
    rng = np.random.default_rng(31)
    xs = [rng.standard_normal(n),
          np.where(rng.random(n) < 0.5, -1.0, 1.0) * np.exp(rng.uniform(-10, 10, n)),
          P.y / np.abs(P.y).max() + 1e-3 * rng.standard_normal(n),  # smooth, cancelling K.x
          np.cos(np.arange(n) * 0.37)]
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert c.stats()["symmetric_k"] == 1
    q_sym = [c.apply_operator(x) for x in xs]
    monkeypatch.setenv("LAKER_SYMV", "0")
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert c.stats()["symmetric_k"] == 0
    q_full = [c.apply_operator(x) for x in xs]
    c.close()
    for k, (a, b) in enumerate(zip(q_sym, q_full)):
        _bitwise(a, b, f"symmetric vs full-row apply, x #{k}")
    # sampled rows against the oracle's one-Dot2-per-row definition (O2)
    idx = np.unique(np.concatenate([[0, 1, 127, 128, n - 1], rng.integers(0, n, 27)]))
    Kr = O.cross_kernel(P.E[idx], P.E, P.scale)
    for k, x in enumerate(xs):
        for t, i in enumerate(idx):
            ref = O.dot2(np.concatenate([[P.lam], Kr[t]]), np.concatenate([[x[i]], x]))
            assert q_sym[k][i] == ref, (k, i, q_sym[k][i], ref)


def test_c4_block_exact_products_fullsize(L, monkeypatch):
    P = make_problem(4)
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    c.set_preconditioner(L.PRECOND_JACOBI)
    Y = np.asfortranarray(P.Y)
    a_off, r_off, _ = c.pcg_solve(Y, P.tol, max_iters=6)
    monkeypatch.setenv("LAKER_BLOCK_OFFSET", "0")
    a_d2, r_d2, _ = c.pcg_solve(Y, P.tol, max_iters=6)
    c.close()
    _bitwise(a_off, a_d2, "block alpha after 6 iterations: offset-Fast2Sum vs Dot2 products")
    assert [r["rel_residual"] for r in r_off] == [r["rel_residual"] for r in r_d2]


def test_symmetric_apply_beyond_offset_range(L, monkeypatch):
    """n = 20000 (> 512 column tiles per block-row): the row accumulators fall back to
    plain Dot2 (the column chains keep their offsets); still bitwise the full-row GEMV."""
    P = make_problem(3, n=20000)
    rng = np.random.default_rng(5)
    xs = [rng.standard_normal(P.n), np.where(rng.random(P.n) < 0.5, -1.0, 1.0) * np.exp(rng.uniform(-8, 8, P.n))]
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert c.stats()["symmetric_k"] == 1
    q_sym = [c.apply_operator(x) for x in xs]
    monkeypatch.setenv("LAKER_SYMV", "0")
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    q_full = [c.apply_operator(x) for x in xs]
    c.close()
    for k, (a, b) in enumerate(zip(q_sym, q_full)):
        _bitwise(a, b, f"n=20000 symmetric vs full-row apply, x #{k}")
