"""Debug: FAST-mode solves with the factored LEARNED P (single and block)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem, make_directions
P = make_problem(4, n=2048, nrhs=16, tol=1e-8)
for mode in (L.MODE_EXACT, L.MODE_FAST):
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
    Z = np.asfortranarray(make_directions(4, P.n, P.n_dirs))
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    a, r1, _ = c.pcg_solve(np.ascontiguousarray(P.Y[:, 0]), P.tol, raise_on_breakdown=False)
    print("mode", mode, "single", r1[0]["iters"], r1[0]["termination"], flush=True)
    for tc in ("1", "0"):
        os.environ["LAKER_BLOCK_TC"] = tc
        A, reps, h = c.pcg_solve(np.asfortranarray(P.Y[:, :2]), P.tol, raise_on_breakdown=False)
        print(" block tc", tc, [(r["iters"], r["termination"]) for r in reps], flush=True)
    c.close()
