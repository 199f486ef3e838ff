"""World-size-2 CPU (gloo) model of the row-sharded PCG that pcg_dist.cu implements
(SURVEY §3.3, §8(e)), in the exchange layout it uses: rank w owns rows
[w n/W, (w+1) n/W) of alpha, r, q, theta and keeps p whole.  Per iteration:

* K apply, symmetric and sharded: rank w streams the tiles the library's own host
  planner assigns it (laker_debug_dist_tiles, called here through liblaker.so: each
  symmetric entry pair once over all ranks); every tile gives row partials K_IJ p_J and,
  off the diagonal block, column partials K_IJ^T p_I; the partials of the rows of ranks
  w+1 .. w+W/2 are sent to them, those of w's rows received from w-1 .. w-W/2, and each
  own row is rounded once (symv_combine_kernel);
* the p.q partials are gathered and summed in rank order;
* factored P, rank-local factors: the N_r partials Q_loc^T r_loc travel with the
  ||r||^2 partial, are summed in rank order and rounded (z), then
  theta_loc = a^{-1/2} r_loc + QM_loc z (QM form) or + Q_loc (M z) (three passes, w by
  row blocks of M and a gather); dense P and P = I / Jacobi use the r / theta gathers;
* theta slices are gathered and p = theta + beta p is formed on every rank.

Partials travel unrounded -- here exact rationals standing in for the kernels' (s, c)
Dot2 pairs -- and are rounded once after the combine, so every rank takes identical
decisions and the sharded iteration equals the single-rank oracle PCG bitwise (T23)."""
import os
from fractions import Fraction

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

P_FACTORED, P_FACTORED_QM = 3, 4  # test-local tags: P = a^{-1/2} I + Q M Q^T in factored form
BR, TC = 8, 4                     # tiles of the model (the library plans 128 x 64)


def _F(x):
    return Fraction(float(x))


def _exact_dot(x, y):
    return sum((_F(a) * _F(b) for a, b in zip(x, y)), Fraction(0))


def _fma(a, b, c):
    """RN(a*b + c) elementwise (numpy has no fma): a two-term Dot2."""
    return np.array([O.dot2(np.array([float(x), 1.0]), np.array([float(u), float(v)]))
                     for x, u, v in np.broadcast(a, b, c)])


def _allgather(obj, W):
    out = [None] * W
    dist.all_gather_object(out, obj)
    return out


class ShardedK:
    """Rank `rank`'s share of the symmetric K apply, from the library's planner."""

    def __init__(self, K, lam, rank, W):
        from paper_2604_25138_b200 import laker as L
        self.K, self.lam, self.rank, self.W = K, lam, rank, W
        n = K.shape[0]
        self.n, self.nloc = n, n // W
        p = L.laker_debug_dist_tiles(n, BR, TC, rank, W)
        self.tiles = []
        for I in range(len(p["toff"]) - 1):
            Ig = rank * (len(p["toff"]) - 1) + I
            for jt in p["jt"][p["toff"][I]:p["toff"][I + 1]]:
                self.tiles.append((Ig, int(jt)))

    def apply(self, p):
        """q_loc = (lambda I + K) p on the own rows through the tile partials and the
        send / receive pattern of pcg_dist.cu; returns (q_loc, exact p_loc.q_loc)."""
        n, nloc, W, w = self.n, self.nloc, self.W, self.rank
        part = [Fraction(0)] * n
        for Ig, jt in self.tiles:
            for i in range(Ig * BR, (Ig + 1) * BR):
                for j in range(jt * TC, (jt + 1) * TC):
                    kij = _F(self.K[i, j])
                    part[i] += kij * _F(p[j])
                    if jt // (BR // TC) != Ig:
                        part[j] += kij * _F(p[i])
        D = W // 2
        sends = {(w + d) % W: part[((w + d) % W) * nloc:((w + d) % W + 1) * nloc] for d in range(1, D + 1)}
        got = _allgather(sends, W)            # rank s's messages; we take the one addressed to w
        own = part[w * nloc:(w + 1) * nloc]
        for d in range(1, D + 1):
            src = (w - d) % W
            own = [a + b for a, b in zip(own, got[src][w])]
        r0 = w * nloc
        q = np.array([float(own[i] + _F(self.lam) * _F(p[r0 + i])) for i in range(nloc)])
        return q, _exact_dot(p[r0:r0 + nloc], q)


def sharded_pcg(rank, W, K, lam, y, pkind, P, tol, max_iters):
    """The rank-`rank` view of the row-sharded PCG (the host logic of pcg_dist.cu)."""
    n = K.shape[0]
    nloc = n // W
    r0, r1 = nloc * rank, nloc * (rank + 1)
    Kop = ShardedK(K, lam, rank, W)
    fac = pkind in (P_FACTORED, P_FACTORED_QM)
    if fac:
        Q, M, ainv = P
        Q_loc = Q[r0:r1]
        QM_loc = (Q @ M)[r0:r1] if pkind == P_FACTORED_QM else None
        m = Q.shape[1]
    P_loc = P[r0:r1] if pkind == O.P_DENSE else None
    alpha_loc = np.zeros(nloc)
    r_loc = y[r0:r1].copy()
    r_full = y.copy()
    ynorm = float(np.sqrt(float(_exact_dot(y, y))))

    def z_of(r_loc, extra):
        zp = [_exact_dot(Q_loc[:, k], r_loc) for k in range(m)]
        got = _allgather((zp, extra), W)
        z = np.array([float(sum(g[0][k] for g in got)) for k in range(m)])
        return z, sum(g[1] for g in got)

    def theta_fac(r_loc, z):
        if pkind == P_FACTORED_QM:
            rows = QM_loc
            v = z
        else:
            nk = m // W
            ks = range(nk * rank, nk * (rank + 1))
            v = np.concatenate(_allgather(np.array([O.dot2(M[k], z) for k in ks]), W))
            rows = Q_loc
        return np.array([O.dot2(np.concatenate([[ainv], rows[i]]), np.concatenate([[r_loc[i]], v]))
                         for i in range(nloc)])

    def theta_dense(r_full):
        return np.array([O.dot2(P_loc[i], r_full) for i in range(nloc)])

    if pkind == O.P_DENSE or fac:
        th_loc = theta_fac(r_loc, z_of(r_loc, Fraction(0))[0]) if fac else theta_dense(r_full)
        parts = _allgather((th_loc, _exact_dot(r_loc, th_loc)), W)
        theta = np.concatenate([t for t, _ in parts])
        rho = float(sum(p for _, p in parts))
    else:
        theta = r_full.copy() if pkind == O.P_NONE else P * r_full
        rho = float(_exact_dot(r_full, theta))
    p = theta.copy()
    iters, rel = 0, 1.0
    for k in range(max_iters):
        q_loc, pq_loc = Kop.apply(p)
        pq = float(sum(_allgather(pq_loc, W)))
        delta = rho / pq
        alpha_loc = _fma(delta, p[r0:r1], alpha_loc)
        r_loc = _fma(-delta, q_loc, r_loc)
        if fac:
            z, rr = z_of(r_loc, _exact_dot(r_loc, r_loc))
        else:
            th_loc = P[r0:r1] * r_loc if pkind == O.P_JACOBI else r_loc
            parts = _allgather((r_loc, th_loc, _exact_dot(r_loc, r_loc), _exact_dot(r_loc, th_loc)), W)
            r_full = np.concatenate([a for a, _, _, _ in parts])
            rr = sum(c for _, _, c, _ in parts)
        rel = float(np.sqrt(float(rr))) / ynorm
        iters = k + 1
        if rel <= tol:
            break
        if pkind == O.P_DENSE or fac:
            th_loc = theta_fac(r_loc, z) if fac else theta_dense(r_full)
            parts2 = _allgather((th_loc, _exact_dot(r_loc, th_loc)), W)
            theta = np.concatenate([t for t, _ in parts2])
            rho_new = float(sum(pp for _, pp in parts2))
        else:
            theta = np.concatenate([b for _, b, _, _ in parts])
            rho_new = float(sum(d for _, _, _, d in parts))
        beta = rho_new / rho
        p = _fma(beta, p, theta)
        rho = rho_new
    alpha = np.concatenate(_allgather(alpha_loc, W))
    return alpha, iters, rel


def _worker(rank, W, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=W)
    K, lam, y, pkind, P, tol = case
    try:
        out = sharded_pcg(rank, W, K, lam, y, pkind, P, tol, 200)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _case(pkind):
    from synth import make_problem
    Pb = make_problem(1, n=64, d=8, lam=1e-2, tol=1e-10)
    K, _ = O.assemble(Pb.E, Pb.scale)
    P = None
    if pkind == O.P_JACOBI:
        P = O.jacobi_diag(Pb.E, Pb.scale, Pb.lam)
    elif pkind == O.P_DENSE:
        B = np.linalg.inv(K + Pb.lam * np.eye(Pb.n) + 0.5 * np.eye(Pb.n))
        P = 0.5 * (B + B.T)
    elif pkind in (P_FACTORED, P_FACTORED_QM):  # a^{-1/2} I + Q M Q^T, Q orthonormal n x 8, M sym. PSD
        r = np.random.default_rng(3)
        Q, _ = np.linalg.qr(r.standard_normal((Pb.n, 8)))
        B = r.standard_normal((8, 8))
        M = 0.3 * (B @ B.T)
        M = 0.5 * (M + M.T)
        P = (np.ascontiguousarray(Q), M, 0.7)
    return K, Pb.lam, Pb.y, pkind, P, Pb.tol


@pytest.mark.parametrize("pkind", [O.P_NONE, O.P_JACOBI, O.P_DENSE, P_FACTORED, P_FACTORED_QM])
def test_two_rank_sharded_pcg_equals_oracle(pkind):
    case = _case(pkind)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 7 * pkind + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    K, lam, y, _, P, tol = case
    if pkind == P_FACTORED:
        ao, ro = O.pcg_factored(K, lam, y, *P, tol=tol, max_iters=200)
    elif pkind == P_FACTORED_QM:
        Q, M, ainv = P
        ao, ro = O.pcg_factored_qm(K, lam, y, Q, np.ascontiguousarray(Q @ M), ainv, tol=tol, max_iters=200)
    else:
        ao, ro = O.pcg(K, lam, y, pkind, P, tol=tol, max_iters=200)
    for r in range(2):
        alpha, iters, rel = res[r]
        assert iters == ro.iters
        assert (alpha == ao).all()
    assert (res[0][0] == res[1][0]).all()
