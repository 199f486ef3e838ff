"""Short C3 run for ncu: the bench step with fewer iterations -- EXACT
assembly, LEARNED fit (factored P, device Philox Z), PCG (ITERS iterations,
default 20), predict on a 32x32 sub-grid.  Argument: learned | jacobi | dense
(dense = EXTERNAL_DENSE identity, the full-row / symmetric dense P path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
prec = sys.argv[1] if len(sys.argv) > 1 else "learned"
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
if prec == "dense":
    c.set_preconditioner(L.PRECOND_EXTERNAL_DENSE, np.eye(P.n))
elif prec == "learned":
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
else:
    c.set_preconditioner(L.PRECOND_JACOBI)
a, reps, _ = c.pcg_solve(P.y, P.tol, max_iters=int(os.environ.get("ITERS", "20")))
m = c.predict(np.ascontiguousarray(P.Eq[::64]), a)
print(reps[0], float(m[0]), c.stats()["p_factored"], c.stats()["symmetric_k"])
c.close()
