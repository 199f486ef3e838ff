import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LAKER_DEBUG_FIT"] = "1"
from paper_2604_25138_b200 import laker as L
from synth import make_problem
P = make_problem(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam)
for _ in range(2):
    print(c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7), file=sys.stderr)
