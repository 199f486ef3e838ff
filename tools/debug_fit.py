import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LAKER_DEBUG_FIT"] = "1"
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem, make_directions
cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
P = make_problem(cid)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam)
Z = np.asfortranarray(make_directions(cid, P.n, P.n_dirs))
print(c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, Z=Z))
