"""One C3 LEARNED fit (for ncu launch lists of the fit kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(int(os.environ.get("CFG", "3")))
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
rep = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
print(rep, c.stats()["fit_ms"], flush=True)
c.close()
