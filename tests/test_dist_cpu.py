"""World-size-2 CPU (gloo) test of the row-sharded PCG recurrence that
pcg_dist.cu implements: rank r owns rows
[r n/W, (r+1) n/W); per iteration the ranks exchange (1) their p.q partials,
(2) [r slice | partials], (3) [theta slice | partial], combine the partials
in rank order and form p redundantly.  Partials travel unrounded (here exact
rationals standing in for the kernel's (s, c) Dot2 pairs) and are rounded once
after the combine, so every rank takes identical decisions and the sharded
iteration equals the single-rank oracle PCG bitwise (T23)."""
import os
from fractions import Fraction

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O

P_FACTORED = 3  # test-local tag: P = a^{-1/2} I + Q M Q^T applied in factored form


def _exact_dot(x, y):
    return sum((Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y)), Fraction(0))


def _fma(a, b, c):
    """RN(a*b + c) elementwise (numpy has no fma): a two-term Dot2."""
    return np.array([O.dot2(np.array([float(x), 1.0]), np.array([float(u), float(v)]))
                     for x, u, v in np.broadcast(a, b, c)])


def _allgather(obj, W):
    out = [None] * W
    dist.all_gather_object(out, obj)
    return out


def _factored_theta(rank, W, F, r_full, r0, r1):
    """theta_loc = (a^{-1/2} I + Q M Q^T) r on rows [r0, r1) as pcg_dist.cu's sharded
    factored apply does it: rank w forms z_k = Q[:, k].r for its N_r/W entries k, all-
    gather; then w_k = M_k.z likewise; then theta_i = Dot2([a^{-1/2}, Q_i], [r_i, w])."""
    Q, M, ainv = F
    m = Q.shape[1]
    nk = m // W
    ks = range(nk * rank, nk * (rank + 1))
    z = np.concatenate(_allgather(np.array([O.dot2(Q[:, k], r_full) for k in ks]), W))
    w = np.concatenate(_allgather(np.array([O.dot2(M[k], z) for k in ks]), W))
    return np.array([O.dot2(np.concatenate([[ainv], Q[i]]), np.concatenate([[r_full[i]], w]))
                     for i in range(r0, r1)])


def sharded_pcg(rank, W, K, lam, y, pkind, P, tol, max_iters):
    """The rank-`rank` view of the row-sharded PCG (the host logic of pcg_dist.cu)."""
    n = K.shape[0]
    r0, r1 = n // W * rank, n // W * (rank + 1)
    K_loc = K[r0:r1]
    fac = pkind == P_FACTORED
    if fac:
        pkind, F = O.P_DENSE, P
    P_loc = None if pkind != O.P_DENSE or fac else P[r0:r1]
    alpha_loc = np.zeros(r1 - r0)
    r_full = y.copy()
    ynorm = float(np.sqrt(float(_exact_dot(y, y))))
    # theta^0 = P r^0 (dense: sharded GEMV + all-gather of [theta slice | partial])
    if pkind == O.P_DENSE:
        th_loc = (_factored_theta(rank, W, F, r_full, r0, r1) if fac else
                  np.array([O.dot2(P_loc[i], r_full) for i in range(r1 - r0)]))
        parts = _allgather((th_loc, _exact_dot(r_full[r0:r1], th_loc)), W)
        theta = np.concatenate([t for t, _ in parts])
        rho = float(sum(p for _, p in parts))
    else:
        theta = r_full.copy() if pkind == O.P_NONE else P * r_full
        rho = float(_exact_dot(r_full, theta))
    p = theta.copy()
    iters, rel = 0, 1.0
    for k in range(max_iters):
        q_loc = np.array([O.dot2(np.concatenate([[lam], K_loc[i]]), np.concatenate([[p[r0 + i]], p]))
                          for i in range(r1 - r0)])
        pq = float(sum(_allgather(_exact_dot(p[r0:r1], q_loc), W)))
        delta = rho / pq
        alpha_loc = _fma(delta, p[r0:r1], alpha_loc)
        r_loc = _fma(-delta, q_loc, r_full[r0:r1])
        if pkind == O.P_JACOBI:
            th_loc = P[r0:r1] * r_loc
        else:
            th_loc = r_loc
        parts = _allgather((r_loc, th_loc, _exact_dot(r_loc, r_loc), _exact_dot(r_loc, th_loc)), W)
        r_full = np.concatenate([a for a, _, _, _ in parts])
        rr = float(sum(c for _, _, c, _ in parts))
        rel = float(np.sqrt(rr)) / ynorm
        iters = k + 1
        if rel <= tol:
            break
        if pkind == O.P_DENSE:
            th_loc = (_factored_theta(rank, W, F, r_full, r0, r1) if fac else
                      np.array([O.dot2(P_loc[i], r_full) for i in range(r1 - r0)]))
            parts2 = _allgather((th_loc, _exact_dot(r_full[r0:r1], th_loc)), W)
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
    Pb = make_problem(1, n=48, d=8, lam=1e-2, tol=1e-10)
    K, _ = O.assemble(Pb.E, Pb.scale)
    P = None
    if pkind == O.P_JACOBI:
        P = O.jacobi_diag(Pb.E, Pb.scale, Pb.lam)
    elif pkind == O.P_DENSE:
        B = np.linalg.inv(K + Pb.lam * np.eye(Pb.n) + 0.5 * np.eye(Pb.n))
        P = 0.5 * (B + B.T)
    elif pkind == P_FACTORED:  # a^{-1/2} I + Q M Q^T, Q orthonormal n x 8, M symmetric PSD
        r = np.random.default_rng(3)
        Q, _ = np.linalg.qr(r.standard_normal((Pb.n, 8)))
        B = r.standard_normal((8, 8))
        M = 0.3 * (B @ B.T)
        M = 0.5 * (M + M.T)
        P = (np.ascontiguousarray(Q), M, 0.7)
    return K, Pb.lam, Pb.y, pkind, P, Pb.tol


@pytest.mark.parametrize("pkind", [O.P_NONE, O.P_JACOBI, O.P_DENSE, P_FACTORED])
def test_two_rank_sharded_pcg_equals_oracle(pkind):
    case = _case(pkind)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + 7 * pkind + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    K, lam, y, _, P, tol = case
    if pkind == P_FACTORED:
        ao, ro = O.pcg_factored(K, lam, y, *P, tol=tol, max_iters=200)
    else:
        ao, ro = O.pcg(K, lam, y, pkind, P, tol=tol, max_iters=200)
    for r in range(2):
        alpha, iters, rel = res[r]
        assert iters == ro.iters
        assert (alpha == ao).all()
    assert (res[0][0] == res[1][0]).all()
