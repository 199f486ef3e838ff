"""Debug: GPU fit vs oracle on a given config (P rows, eigenvalues)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem, make_directions
import oracle as O
cid, n = int(sys.argv[1]), int(sys.argv[2])
P = make_problem(cid, n=n)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
rep = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z)
Pg = c.get_preconditioner_rows()
K, _ = O.assemble(P.E, P.scale)
Po, ro, st = O.cccp_fit_structured(K, P.lam, Z)
print(rep)
print("oracle iters", ro.iters, "a", st.a, "rel diff P", np.linalg.norm(Pg - Po) / np.linalg.norm(Po))
print("eig P gpu", np.linalg.eigvalsh(0.5 * (Pg + Pg.T))[:3], "eig P oracle", np.linalg.eigvalsh(Po)[:3])
c.close()
