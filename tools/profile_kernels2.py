"""Short C3 run for `ncu --set full` captures of the round-1 kernels: EXACT
assembly, LEARNED fit (its first ozaki_fused_kernel is the directions GEMM
U^T = Z^T (lambda I + K), 4096 x 16384 x 16384), PCG for 3 iterations (the first
gemv_dot2_kernel is pass 1 of the factored P, z = Q^T r; symv_dot2_kernel is K.p)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
a, reps, _ = c.pcg_solve(P.y, P.tol, max_iters=3)
print(reps[0]["iters"], c.stats()["symmetric_k"], c.stats()["p_factored"])
c.close()
