"""Host wall-clock per call of the bench step (C3, device buffers), with the
library's own event times beside it -- to find host-side gaps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_25138_b200 import laker as L
from synth import make_problem

P = make_problem(3)
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
c = L.Context(0, 0, 1, None, stream.cuda_stream)
E = torch.from_numpy(P.E).to(dev); y = torch.from_numpy(P.y).to(dev); Eq = torch.from_numpy(P.Eq).to(dev)
alpha = torch.zeros(P.n, dtype=torch.float64, device=dev); out = torch.zeros(P.Eq.shape[0], dtype=torch.float64, device=dev)
for it in range(int(os.environ.get('STEPS', '6'))):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    c.assemble_kernel(E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT); torch.cuda.synchronize(); t.append(time.perf_counter())
    c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7); torch.cuda.synchronize(); t.append(time.perf_counter())
    reps = L.laker_pcg_solve(c.h, 1, y, alpha, P.tol, 0, False, None); t_call = time.perf_counter(); torch.cuda.synchronize(); t.append(time.perf_counter())
    L.laker_predict(c.h, Eq, alpha, out, L.MODE_EXACT); torch.cuda.synchronize(); t.append(time.perf_counter())
    st = c.stats()
    w = [1e3 * (t[i + 1] - t[i]) for i in range(4)]
    print(f"wall ms: assemble {w[0]:.1f} (ev {st['assemble_ms']:.1f}) fit {w[1]:.1f} (ev {st['fit_ms']:.1f}) "
          f"solve {w[2]:.1f} (call {1e3 * (t_call - t[2]):.1f}, ev {st['solve_ms']:.1f}) predict {w[3]:.1f} (ev {st['predict_ms']:.1f}) total {sum(w):.1f}", flush=True)
c.close()
