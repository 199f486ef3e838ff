"""Per-iteration time of the C3 LEARNED solve against the event-timed K and P applies:
the remainder is kernel-boundary time (tails, launches) inside the captured chunks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
y = torch.from_numpy(P.y).cuda()
a = torch.zeros(P.n, dtype=torch.float64, device="cuda")
out = {}
for inst in (0, 0, 0, 1, 2, 2):
    if inst == 2:  # as bench.py's step: assemble + fit right before the solve
        c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        torch.cuda.synchronize()
        r = L.laker_pcg_solve(c.h, 1, y, a, P.tol, 0, 0, None)[0]
        out.setdefault("after_fit_us_per_iter", []).append(r["seconds"] / r["iters"] * 1e6)
        continue
    s0 = c.stats()
    r = L.laker_pcg_solve(c.h, 1, y, a, P.tol, 0, inst, None)[0]
    s1 = c.stats()
    per = r["seconds"] / r["iters"] * 1e6
    if inst:
        op = (s1["op_ms"] - s0["op_ms"]) / max(s1["op_launches"] - s0["op_launches"], 1) * 1e3
        pr = (s1["prec_ms"] - s0["prec_ms"]) / max(s1["prec_launches"] - s0["prec_launches"], 1) * 1e3
        out["instrumented_us_per_iter"] = per
        out["op_us"], out["prec_us"] = op, pr
    else:
        out.setdefault("us_per_iter", []).append(per)
print(out, "k_tc", c.stats()["k_tensor_core"])
c.close()
