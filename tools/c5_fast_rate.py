"""Per-iteration rate of the FAST on-the-fly operator at C5 (n = 65536, d = 64) and
the 1024^2-grid prediction: 20 capped PCG iterations with the Jacobi P.
LAKER_OTF_SYM=0 selects the full-square kernel instead of the symmetric one."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

grid = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
P = make_problem(5, grid=grid)
dev = torch.device("cuda", 0)
c = L.Context(0)
c.assemble_kernel(torch.from_numpy(P.E).to(dev), P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
c.fit_preconditioner(L.PRECOND_JACOBI)
a, reps, _ = c.pcg_solve(torch.from_numpy(P.y).to(dev), P.tol, max_iters=20)
r = reps[0]
alpha = torch.from_numpy(np.random.default_rng(0).standard_normal(P.n)).to(dev)
out = c.predict(torch.from_numpy(P.Eq).to(dev), alpha, mode=L.MODE_FAST)
st = c.stats()
print(json.dumps(dict(config="C5", mode="fast", otf_sym=os.environ.get("LAKER_OTF_SYM", "1"), iters=r["iters"],
                      ms_per_iter=r["seconds"] / r["iters"] * 1e3, rel_residual=r["rel_residual"],
                      predict_grid=P.Eq.shape[0], predict_ms=st["predict_ms"])))
c.close()
