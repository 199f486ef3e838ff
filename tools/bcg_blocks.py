"""C4 (n = 16384, 64 maps, LEARNED P): the block-CG variant (B14) by column-group size,
FAST and EXACT, beside the batched Alg. 1 solve: steps, seconds, termination, worst true
residual."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402

P = make_problem(4)
Y = np.asfortranarray(P.Y)
modes = [("fast", L.MODE_FAST)] + ([("exact", L.MODE_EXACT)] if os.environ.get("EXACT", "1") == "1" else [])
c = L.Context(0)
for name, mode in modes:
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, mode)
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
    _, rb, _ = c.pcg_solve(Y, P.tol)
    print(json.dumps({"mode": name, "solver": "batched", "steps_max": max(r["iters"] for r in rb),
                      "seconds": rb[0]["seconds"], "worst_true": max(r["true_rel_residual"] for r in rb)}), flush=True)
    for b in (4, 8, 16, 32, 64):
        _, r, _ = c.block_cg_solve(Y, P.tol, block=b, raise_on_breakdown=False)
        print(json.dumps({"mode": name, "solver": f"block_cg/{b}", "steps": r[0]["iters"], "seconds": r[0]["seconds"],
                          "termination": r[0]["termination"],
                          "worst_true": max(x["true_rel_residual"] for x in r)}), flush=True)
c.close()
