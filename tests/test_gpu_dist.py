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
            c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
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


def test_fused_iteration_equals_unfused(L):
    """gemv.cu's fused two-kernel iteration (LAKER_FUSED=1) is the same recurrence."""
    import os
    P = make_problem(2)
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    a0, r0, h0 = c.pcg_solve(P.y, P.tol, want_history=True)
    os.environ["LAKER_FUSED"] = "1"
    try:
        a1, r1, h1 = c.pcg_solve(P.y, P.tol, want_history=True)
    finally:
        del os.environ["LAKER_FUSED"]
    c.close()
    assert r0[0]["iters"] == r1[0]["iters"] and (h0 == h1).all() and (a0 == a1).all()
