"""C3 LEARNED fit (bench configuration: seed 7, N_r = 4096) with LAKER_DEBUG_FIT=1: the
library prints the device time of each fit phase to stderr (fit.cu tick())."""
import os, sys
os.environ.setdefault("LAKER_DEBUG_FIT", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
for _ in range(2):
    rep = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
    print("fit", rep["iters"], "steps", rep["seconds"] if "seconds" in rep else "", file=sys.stderr)
c.close()
