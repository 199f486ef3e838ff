import numpy as np, sys
sys.path.insert(0, '.')
from paper_2604_25138_b200 import laker as L
from synth import make_problem
P = make_problem(1)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam)
c.set_preconditioner(L.PRECOND_JACOBI)
a, reps, _ = c.pcg_solve(P.y, P.tol, instrument=True)
print(reps, c.stats())
try:
    print(c.predict(P.Eq[:10], a))
except Exception as e:
    print("predict after instr:", e)
c2 = L.Context(0)
c2.assemble_kernel(P.E, P.scale, P.lam)
a, reps, _ = c2.pcg_solve(P.y, P.tol, instrument=False)
print(c2.predict(P.Eq[:3], a))
P = make_problem(3)
c2.assemble_kernel(P.E, P.scale, P.lam)
out = c2.predict(P.Eq, a[:1].repeat(P.n)*0+1.0)
print(out[:3])
