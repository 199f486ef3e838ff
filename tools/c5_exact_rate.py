"""Per-iteration rate of the EXACT on-the-fly operator at C5 (n = 65536, d = 64):
three capped PCG iterations with the Jacobi P.  LAKER_OTF_SYM=0 selects the
full-square kernel instead of the symmetric one (otf_sym.cu)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

P = make_problem(5)
dev = torch.device("cuda", 0)
c = L.Context(0)
c.assemble_kernel(torch.from_numpy(P.E).to(dev), P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_EXACT)
c.fit_preconditioner(L.PRECOND_JACOBI)
a, reps, _ = c.pcg_solve(torch.from_numpy(P.y).to(dev), P.tol, max_iters=3)
r = reps[0]
print(json.dumps(dict(config="C5", mode="exact", otf_sym=os.environ.get("LAKER_OTF_SYM", "1"), iters=r["iters"],
                      ms_per_iter=r["seconds"] / r["iters"] * 1e3, rel_residual=r["rel_residual"])))
c.close()
