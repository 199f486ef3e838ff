"""One FAST on-the-fly operator apply at C5 size (n = 65536, d = 64) for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(5, grid=16)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
q = c.apply_operator(P.y)
print(float(q[0]))
c.close()
