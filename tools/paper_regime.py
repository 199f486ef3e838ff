"""The paper's own regime on one B200:
n in {50, 200, 500, 1000, 2000}, d_e = 10, G = exp(E E^T), lambda = 1e-2, PCG to
1e-10, 45 x 45 grid.  Per n and preconditioner (NONE / JACOBI / LEARNED): PCG
iterations, the Lanczos estimate of kappa(P A) (the quantity behind Table I and
P:853-858), solve / fit time, the grid RMSE against the noise-free field, and the
paper's "iterations to a target objective gap of 1e-3":
  ObjGap(alpha) = |R(alpha) - R(alpha_ref)| / |R(alpha_ref)|,
  R(alpha) = ||G alpha - y||^2 + lambda alpha^T G alpha
with alpha_ref the host LAPACK Cholesky solution of (G + lambda I) alpha = y
(standing in for the paper's convex-solver reference).  PCG is deterministic,
so the k-th iterate is the result of a solve capped at max_iters = k.
One JSON line per (n, preconditioner)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_paper_problem  # noqa: E402


def objective(G, lam, y, a):
    Ga = G @ a
    return float((Ga - y) @ (Ga - y) + lam * (a @ Ga))


def objgap_iters(c, P, G, r_ref, kmax, target=1e-3):
    """first k whose PCG iterate has ObjGap <= target, and the gap at k"""
    for k in range(1, kmax + 1):
        a, _, _ = c.pcg_solve(P.y, P.tol, max_iters=k, raise_on_breakdown=False)
        gap = abs(objective(G, P.lam, P.y, a) - r_ref) / abs(r_ref)
        if gap <= target:
            return k, gap
    return None, None


ns = [int(x) for x in sys.argv[1:]] or [50, 200, 500, 1000, 2000]
c = L.Context(0)
for n in ns:
    P = make_paper_problem(n)
    for kind in ("none", "jacobi", "learned"):
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        fit = {}
        if kind == "learned":
            fit = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        elif kind == "jacobi":
            c.fit_preconditioner(L.PRECOND_JACOBI)
        else:
            c.fit_preconditioner(L.PRECOND_NONE)
        a, reps, _ = c.pcg_solve(P.y, P.tol)
        r = reps[0]
        if kind == "none":
            G = c.get_kernel_rows()
            a_ref = np.linalg.solve(G + P.lam * np.eye(n), P.y)
            r_ref = objective(G, P.lam, P.y, a_ref)
        gap_final = abs(objective(G, P.lam, P.y, a) - r_ref) / abs(r_ref)
        k_gap, _ = objgap_iters(c, P, G, r_ref, r["iters"])
        m = c.predict(P.Eq, a)
        rmse = float(np.sqrt(np.mean((m - P.truth[:, 0]) ** 2)))
        print(json.dumps(dict(workload="paper regime", n=n, d=P.d, lam=P.lam, precond=kind, iters=r["iters"],
                              termination=r["termination"], true_rel_residual=r["true_rel_residual"],
                              kappa_PA_lanczos=r["lanczos_lmax"] / r["lanczos_lmin"], solve_ms=r["seconds"] * 1e3,
                              fit_ms=fit.get("seconds", 0.0) * 1e3, fit_cccp_steps=fit.get("iters"),
                              n_dirs=P.n_dirs if kind == "learned" else None, grid_rmse_db=rmse,
                              iters_to_objgap_1e3=k_gap, objgap_final=gap_final)), flush=True)
c.close()
