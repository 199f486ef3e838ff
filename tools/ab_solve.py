"""Repeated C3 LEARNED solves in one process (the bench's solve stage): min / median
time-to-solution and iterations/s over REPS solves, for A/B comparisons of kernel
variants selected by environment variables (read once per process)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

reps = int(os.environ.get("REPS", "8"))
P = make_problem(3)
dev = torch.device("cuda", 0)
c = L.Context(0)
c.assemble_kernel(torch.from_numpy(P.E).to(dev), P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
y = torch.from_numpy(P.y).to(dev)
ts, its = [], []
fit_each = os.environ.get("FIT_EACH", "0") == "1"  # the bench step's order: fit, then solve
for _ in range(reps + 1):
    if fit_each:
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
    a, r, _ = c.pcg_solve(y, P.tol)
    ts.append(r[0]["seconds"])
    its.append(r[0]["iters"])
ts, its = ts[1:], its[1:]
print(json.dumps(dict(tag=os.environ.get("TAG", ""), iters=its[0], tts_min=min(ts), tts_med=float(np.median(ts)),
                      its_per_s_best=its[0] / min(ts), its_per_s_med=its[0] / float(np.median(ts)))))
c.close()
