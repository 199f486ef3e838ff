"""C3 K applies for kernel timing under ncu (tools/tc_variants.sh): assemble the C3 kernel
(EXACT, materialized) and run y = (lambda I + K) x five times through the C ABI."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
c = L.Context(0)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
x = np.random.default_rng(1).standard_normal(P.n)
for _ in range(5):
    y = c.apply_operator(x)
print(c.stats()["k_tensor_core"], float(y[0]))
c.close()
