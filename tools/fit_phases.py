"""C3 LEARNED fit phase breakdown (LAKER_DEBUG_FIT=1 timers; the second of REPS fits,
after warm-up) -- the fit is ~40% of the bench's end-to-end step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LAKER_DEBUG_FIT", "1")
from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

P = make_problem(int(os.environ.get("CFG", "3")))
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
for k in range(int(os.environ.get("REPS", "2"))):
    print(f"--- fit {k}", file=sys.stderr, flush=True)
    rep = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
    print(k, rep["iters"], c.stats()["fit_ms"], flush=True)
c.close()
