"""A short C4 block solve (64 right-hand sides, LEARNED P, MODE from argv: fast | exact)
for ncu launch lists: assemble, fit, ITERS block iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

mode = L.MODE_FAST if (sys.argv[1] if len(sys.argv) > 1 else "fast") == "fast" else L.MODE_EXACT
P = make_problem(4)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
A, reps, _ = c.pcg_solve(np.asfortranarray(P.Y), P.tol, max_iters=int(os.environ.get("ITERS", "8")))
print(reps[0]["iters"], reps[0]["seconds"])
c.close()
