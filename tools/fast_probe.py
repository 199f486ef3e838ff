"""FAST-mode K accuracy and iteration counts at the C5 downscale (n = 8192, lambda = 1e-5):
materialized FAST (DMMA) vs on-the-fly FAST (tcgen05) vs EXACT, each with its own LAKER fit
on the harness Z; per-entry error statistics of the FAST entries against the oracle's."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle as O  # noqa: E402
from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem, make_directions  # noqa: E402

P = make_problem(5, n=8192)
K, _ = O.assemble(P.E, P.scale)
nr = O.nr_schedule(P.n)
Z = np.asfortranarray(make_directions(5, P.n, nr))
out = {}
for name, storage, mode in [("exact_mat", L.STORE_MATERIALIZED, L.MODE_EXACT),
                            ("fast_mat", L.STORE_MATERIALIZED, L.MODE_FAST),
                            ("fast_otf", L.STORE_ON_THE_FLY, L.MODE_FAST),
                            ("exact_otf", L.STORE_ON_THE_FLY, L.MODE_EXACT)]:
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, storage, mode)
    rec = {}
    if storage == L.STORE_MATERIALIZED:
        Kg = c.get_kernel_rows()
        rel = (Kg - K) / K
        rec.update(max_rel=float(np.abs(rel).max()), mean_rel=float(rel.mean()), rms_rel=float(np.sqrt((rel ** 2).mean())))
    one = np.ones(P.n)
    q1 = c.apply_operator(one)
    q1o = O.apply(K, P.lam, one)
    rec["ones_rel_bias"] = float(np.mean((q1 - q1o) / q1o))
    x = np.random.default_rng(1).standard_normal(P.n)
    qx = c.apply_operator(x)
    qxo = O.apply(K, P.lam, x)
    rec["rand_rel_err_rms"] = float(np.sqrt(np.mean(((qx - qxo) / (np.abs(K) @ np.abs(x))) ** 2)))
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=nr, Z=Z)
    a, r, _ = c.pcg_solve(P.y, P.tol)
    rec["iters"] = r[0]["iters"]
    c.set_preconditioner(L.PRECOND_JACOBI)
    a, r, _ = c.pcg_solve(P.y, P.tol)
    rec["jacobi_iters"] = r[0]["iters"]
    c.close()
    out[name] = rec
    print(name, rec, flush=True)
json.dump(out, open("gpurun_out/fast_probe.json", "w"), indent=1)
