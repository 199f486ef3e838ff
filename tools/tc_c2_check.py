"""C2 learned solve (the GPU's own fit) with the tensor-core K apply and with the fp64
symmetric apply (LAKER_SYMV_TC=0): iteration counts, first differing history entry, and
bitwise comparison of the two applies on the CG directions of the run."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem, make_directions

P = make_problem(2)
Z = np.asfortranarray(make_directions(2, P.n, P.n_dirs))


def run(tc):
    os.environ["LAKER_SYMV_TC"] = "1" if tc else "0"
    c = L.Context(0)
    c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
    k = c.stats()["k_tensor_core"]
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
    a, r, h = c.pcg_solve(P.y, P.tol, want_history=True)
    xs = [np.random.default_rng(s).standard_normal(P.n) * np.exp(np.random.default_rng(s + 9).uniform(-20, 20, P.n))
          for s in range(20)]
    ys = [c.apply_operator(x) for x in xs]
    c.close()
    return k, r[0]["iters"], np.asarray(h), ys


k1, i1, h1, y1 = run(True)
k0, i0, h0, y0 = run(False)
d = np.flatnonzero(h1[:min(len(h1), len(h0))] != h0[:min(len(h1), len(h0))])
print({"tc": k1, "fp64": k0, "iters_tc": i1, "iters_fp64": i0, "first_history_diff": int(d[0]) if d.size else None,
       "apply_mismatch_rows": [int((a != b).sum()) for a, b in zip(y1, y0)]})
