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


# n = 1000: n/W is not a multiple of 256, so the sharded path streams full K rows (gemv)
@pytest.mark.parametrize("cid,n,kind", [(1, None, "none"), (1, None, "jacobi"), (2, None, "learned"),
                                        (2, None, "factored"), (3, 2048, "factored"),
                                        (3, 1024, "jacobi"), (3, 1000, "jacobi"), (3, 1000, "factored"),
                                        (1, None, "onthefly")])
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
        res.append((a, reps[0], hist, q, c.stats()["k_tensor_core"]))
        c.close()
    (a0, r0, h0, q0, t0), (a1, r1, h1, q1, t1) = res
    # the stored symmetric K of the configs takes the exact tensor-core apply on both paths
    # (the sharded one reduce-scatters its int64 level groups); the sharded path with
    # n = 1000 (n/W not a multiple of 256) streams full rows
    stored = kind != "onthefly"
    assert t0 == int(stored) and t1 == int(stored and P.n % 256 == 0), (t0, t1)
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


@pytest.mark.parametrize("W", [2, 3, 4, 5, 8])
def test_sharded_symmetric_apply_detached_ranks(L, W):
    """The row-sharded symmetric K apply (symv.cu tri_plan_dist + pcg_dist.cu combine) run
    rank by rank on one GPU (detached shards, no communicator): each rank's tile partials
    (laker_debug_dist_symv_partials) are exchanged here exactly as pcg_dist.cu's
    send/recv does (rank w's rows receive the pairs of ranks w-1 .. w-W/2) and combined
    by the library's own combine kernel; the concatenated rows must equal the single-GPU
    symmetric apply -- and so the oracle's O2 rows -- bitwise, and every pair a rank
    would not send must be zero."""
    n = {3: 3072, 5: 2560}.get(W, 4096)
    P = make_problem(3, n=n)
    full = L.Context(0)
    full.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert full.stats()["symmetric_k"] == 1
    Kf = full.get_kernel_rows()
    rowmax = np.ascontiguousarray(np.abs(Kf).max(axis=1))
    rng = np.random.default_rng(W)
    xs = [rng.standard_normal(n), np.where(rng.random(n) < 0.5, -1.0, 1.0) * np.exp(rng.uniform(-6, 6, n))]
    refs = [full.apply_operator(x) for x in xs]
    full.close()
    nloc, D = n // W, W // 2
    ctxs = []
    for w in range(W):
        c = L.Context(0, w, W, None)
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        assert c.stats()["symmetric_k"] == 1
        ctxs.append(c)
    for x, ref in zip(xs, refs):
        parts = []
        for w, c in enumerate(ctxs):
            pr = np.zeros(2 * n)
            L.laker_debug_dist_symv_partials(c.h, x, rowmax, pr)
            pr = pr.reshape(n, 2)
            sent = {w} | {(w + d) % W for d in range(1, D + 1)}
            for o in range(W):
                if o not in sent:
                    assert (pr[o * nloc:(o + 1) * nloc] == 0).all(), (w, o)
            parts.append(pr)
        q = np.empty(n)
        for w, c in enumerate(ctxs):
            rows = slice(w * nloc, (w + 1) * nloc)
            own = np.ascontiguousarray(parts[w][rows])
            recv = np.ascontiguousarray(np.stack([parts[(w - d) % W][rows] for d in range(1, D + 1)]))
            ql = np.zeros(nloc)
            L.laker_debug_dist_symv_combine(c.h, x, own, recv, ql)
            q[rows] = ql
        bad = np.flatnonzero(q != ref)
        assert bad.size == 0, (W, bad.size, bad[:5])
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("kind", ["jacobi", "learned"])
def test_collective_block_solve_equals_single(L, kind):
    """The row-sharded multi-RHS solve (pcg_block.cu pcg_solve_block_dist: per-rank column
    pairs all-gathered and combined in rank order, the factored P's Q^T R from gathered
    partial products) on a 1-rank communicator equals the single-GPU block solve bitwise,
    and every column equals the single-RHS oracle solve (T18)."""
    P = make_problem(4, n=1024, nrhs=6, tol=1e-8)
    Y = np.asfortranarray(P.Y)
    res = []
    for use_nccl in (False, True):
        c = L.Context(0, 0, 1, L.laker_get_unique_id() if use_nccl else None)
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        if kind == "jacobi":
            c.set_preconditioner(L.PRECOND_JACOBI)
        else:
            Z = np.asfortranarray(make_directions(4, P.n, P.n_dirs))
            c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
        A, reps, _ = c.pcg_solve(Y, P.tol)
        res.append((A, [r["iters"] for r in reps], [r["true_rel_residual"] for r in reps]))
        c.close()
    (A0, i0, t0), (A1, i1, t1) = res
    assert i0 == i1 and t0 == t1 and (A0 == A1).all()
    if kind == "jacobi":
        K, _ = O.assemble(P.E, P.scale)
        d = O.jacobi_diag(P.E, P.scale, P.lam)
        for j in range(Y.shape[1]):
            ao, ro = O.pcg(K, P.lam, Y[:, j], O.P_JACOBI, d, tol=P.tol)
            assert ro.iters == i1[j] and (ao == A1[:, j]).all()


@pytest.mark.parametrize("W", [2, 3, 4, 8])
def test_tensor_core_groups_of_shards_sum_to_one_rank(L, W):
    """The exact tensor-core apply on the sharded plan (symv_tc.cu with dist_tiles at
    128 x 128; B13, §8): every shard's int64 level groups of all rows
    (laker_debug_tc_groups, detached shards on one GPU) add up, as integers, to the one-rank
    groups -- each symmetric pair of entries is streamed once over the shards -- so the
    int64 reduce-scatter of pcg_dist.cu gives every rank exactly the one-rank row sums, and
    its combine (the finalize's arithmetic) the one-rank apply bitwise."""
    n = {3: 3072}.get(W, 4096)
    P = make_problem(3, n=n)
    full = L.Context(0)
    full.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    assert full.stats()["k_tensor_core"] == 1
    rowmax = np.ascontiguousarray(np.abs(full.get_kernel_rows()).max(axis=1))
    rng = np.random.default_rng(40 + W)
    xs = [rng.standard_normal(n), np.where(rng.random(n) < 0.5, -1.0, 1.0) * np.exp(rng.uniform(-8, 8, n))]
    ones = []
    for x in xs:
        g = np.zeros(8 * n, dtype=np.int64)
        L.laker_debug_tc_groups(full.h, x, None, g)
        ones.append(g)
    full.close()
    sums = [np.zeros(8 * n, dtype=np.int64) for _ in xs]
    for w in range(W):
        c = L.Context(0, w, W, None)
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        for x, acc in zip(xs, sums):
            g = np.zeros(8 * n, dtype=np.int64)
            L.laker_debug_tc_groups(c.h, x, rowmax, g)
            acc += g
        assert c.stats()["k_tensor_core"] == 1
        c.close()
    for acc, one in zip(sums, ones):
        bad = np.flatnonzero(acc != one)
        assert bad.size == 0, (W, bad.size, bad[:5])
        assert np.abs(one).max() > 0

