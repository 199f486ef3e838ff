"""The row-sharded NCCL code path (pcg_dist.cu) on one GPU: a 1-rank
communicator (laker_create with world = 1 and an NCCL id) runs the collective
path -- per-rank Dot2 pairs, all-gathers, rank-order combine -- which must give
bitwise the single-GPU path's results (rank invariance, at W = 1).
Multi-rank runs need several GPUs (bench.py under torchrun); the host logic of
W = 2 is covered on CPU by tests/test_dist_cpu.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from synth import make_problem, make_directions  # noqa: E402


@pytest.fixture(scope="module")
def L():
    from paper_2604_25138_b200 import laker
    return laker


@pytest.mark.parametrize("cid,n,kind", [(1, None, "none"), (1, None, "jacobi"), (2, None, "learned"),
                                        (2, None, "factored"), (3, 2048, "factored"),
                                        (3, 1024, "jacobi"), (1, None, "onthefly")])
def test_collective_path_equals_single(L, cid, n, kind):
    P = make_problem(cid, n=n)
    res = []
    for use_nccl in (False, True):
        c = L.Context(0, 0, 1, L.laker_get_unique_id() if use_nccl else None)
        storage = L.STORE_ON_THE_FLY if kind == "onthefly" else L.STORE_MATERIALIZED
        c.assemble_kernel(P.E, P.scale, P.lam, storage, L.MODE_EXACT)
        if kind == "jacobi":
            c.set_preconditioner(L.PRECOND_JACOBI)
        elif kind == "learned":
            Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
            # dense rows on both sides (AUTO picks the factored P on the single-GPU path)
            c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_DENSE)
        elif kind == "factored":
            # the sharded factored apply: z and w entries per rank + two gathers (pcg_dist.cu)
            Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
            c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z, p_layout=L.P_AUTO)
        a, reps, hist = c.pcg_solve(P.y, P.tol, want_history=True)
        q = c.apply_operator(a)
        res.append((a, reps[0], hist, q))
        c.close()
    (a0, r0, h0, q0), (a1, r1, h1, q1) = res
    assert r0["iters"] == r1["iters"] and r0["termination"] == r1["termination"]
    assert (h0 == h1).all() and (a0 == a1).all() and (q0 == q1).all()
    assert r0["true_rel_residual"] == r1["true_rel_residual"]
    if kind in ("none", "jacobi"):
        K, _ = O.assemble(P.E, P.scale)
        pk = O.P_NONE if kind == "none" else O.P_JACOBI
        dv = O.jacobi_diag(P.E, P.scale, P.lam) if kind == "jacobi" else None
        ao, ro = O.pcg(K, P.lam, P.y, pk, dv, tol=P.tol)
        assert ro.iters == r1["iters"] and (ao == a1).all()


@pytest.mark.parametrize("W", [2, 4])
def test_row_sharded_assembly_and_predict_layouts(L, W):
    """Detached shards (world = W, no communicator) on one GPU: each rank's K rows
    are the rows [r n/W, (r+1) n/W) of the full kernel, bitwise (EXACT and FAST);
    each rank's predict rows match the full map; the dense P loaded per rank
    round-trips.  (The collectives themselves need W GPUs.)"""
    P = make_problem(3, n=2048)
    full = L.Context(0)
    for mode in (L.MODE_EXACT, L.MODE_FAST):
        full.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
        Kf = full.get_kernel_rows()
        alpha = np.random.default_rng(1).standard_normal(P.n)
        Eq = np.ascontiguousarray(P.Eq[:1000])
        mf = full.predict(Eq, alpha, mode=mode)
        for r in range(W):
            c = L.Context(0, r, W, None)
            c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
            Kr = c.get_kernel_rows()
            rows = slice(r * P.n // W, (r + 1) * P.n // W)
            if mode == L.MODE_EXACT:
                assert (Kr == Kf[rows]).all()
            else:
                assert np.abs(Kr / Kf[rows] - 1).max() <= 1e-13
            out = np.full(Eq.shape[0], np.nan)
            c.predict(Eq, alpha, mode=mode, out=out)
            per = -(-Eq.shape[0] // W)
            sl = slice(r * per, min(Eq.shape[0], (r + 1) * per))
            assert (out[sl] == mf[sl]).all() and np.isnan(np.delete(out, np.r_[sl])).all()
            c.set_preconditioner(L.PRECOND_EXTERNAL_DENSE, np.ascontiguousarray(Kf[rows]))
            assert (c.get_preconditioner_rows() == Kf[rows]).all()
            with pytest.raises(L.LakerError):
                c.pcg_solve(P.y, 1e-8)
            c.close()
    full.close()
