"""Short run of the symmetric GEMV (csrc/symv.cu) at C3 (n = 16384) for ncu and
a quick timing: assemble EXACT, a few operator applies (each = symv_dot2_kernel
+ symv_finalize_kernel), then an instrumented Jacobi PCG of ITERS iterations
whose per-apply CUDA-event time is printed.  LAKER_SYMV=0 runs gemv.cu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2604_25138_b200 import laker as L
from synth import make_problem

c = L.Context(0)
P = make_problem(3)
c.assemble_kernel(P.E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
for _ in range(int(os.environ.get("REPS", "3"))):
    y = c.apply_operator(P.y)
it = int(os.environ.get("ITERS", "0"))
if it:
    c.set_preconditioner(L.PRECOND_JACOBI)
    c.pcg_solve(P.y, 1e-30, max_iters=it, instrument=True)
    s = c.stats()
    ms = s["op_ms"] / max(1, s["op_launches"])
    n = P.n
    alg = 8.0 * n * (n + 1) / 2 + 16 * n if s["symmetric_k"] else 8.0 * n * n + 16 * n
    print(f"apply: {ms * 1e3:.1f} us over {s['op_launches']} launches, symmetric={s['symmetric_k']}, "
          f"{alg / ms / 1e6:.0f} GB/s algorithmic ({alg / 1e9:.3f} GB)")
print("ok", float(y[0]), c.stats()["symmetric_k"])
c.close()
