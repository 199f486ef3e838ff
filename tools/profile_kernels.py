"""Short runs of the compute kernels for ncu (one launch of each is captured):
assemble_exact/assemble_fast at C3, the DMMA GEMM inside a C2 fit, the FAST
on-the-fly operator (n = 16384), the EXACT block GEMM (8 RHS)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem

c = L.Context(0)
P = make_problem(3)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_FAST)
c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
y = c.apply_operator(P.y)
P4 = make_problem(4, nrhs=8)
c.assemble_kernel(P4.E, P4.scale, P4.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
c.set_preconditioner(L.PRECOND_JACOBI)
a, reps, _ = c.pcg_solve(np.asfortranarray(P4.Y), P4.tol, max_iters=2)
print("ok", float(y[0]), reps[0]["iters"])
c.close()
