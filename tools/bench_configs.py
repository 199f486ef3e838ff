"""Per-config measurements of the hot path on one B200 (BASELINE.json configs
C1..C5), through the C ABI.  Prints one JSON line per (config, variant).

    python tools/bench_configs.py [C1 C2 C3 C4 C5 C5L ...]   (C5L: LEARNED at C5, on the fly)

C1/C2/C3: assemble (EXACT) -> fit (LEARNED, device Philox Z) -> PCG -> predict,
plus NONE/JACOBI solves; C4: 64-RHS block solve with the learned P, EXACT
(Dot2 GEMM) and FAST (DMMA GEMM) applies; C5: n = 65536 on the fly with
Jacobi (FAST DMMA operator) -- iterations capped, per-iteration rate reported
(the config is quoted on 8 GPUs), plus the 1024^2 FAST predict.
Device times come from the library's CUDA events (laker_get_stats).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2604_25138_b200 import laker as L  # noqa: E402
from synth import make_problem  # noqa: E402


def emit(**kw):
    print(json.dumps(kw), flush=True)


def run_std(cid, kinds=("learned", "jacobi", "none")):
    import torch
    P = make_problem(cid)
    dev = torch.device("cuda", 0)
    c = L.Context(0)
    E = torch.from_numpy(P.E).to(dev)
    y = torch.from_numpy(P.y).to(dev)
    Eq = torch.from_numpy(P.Eq).to(dev)
    for kind in kinds:
        c.assemble_kernel(E, P.scale, P.lam, L.STORE_MATERIALIZED, L.MODE_EXACT)
        asm = c.stats()["assemble_ms"]
        fit = {}
        if kind == "learned":
            fit = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        elif kind == "jacobi":
            c.fit_preconditioner(L.PRECOND_JACOBI)
        else:
            c.fit_preconditioner(L.PRECOND_NONE)
        a, reps, _ = c.pcg_solve(y, P.tol, instrument=True)
        st = c.stats()
        m = c.predict(Eq, a)
        pst = c.stats()
        emit(config=f"C{cid}", n=P.n, d=P.d, precond=kind, iters=reps[0]["iters"],
             termination=reps[0]["termination"], true_rel_residual=reps[0]["true_rel_residual"],
             time_to_solution_s=reps[0]["seconds"], iters_per_s=reps[0]["iters"] / reps[0]["seconds"],
             assemble_ms=asm, fit_ms=st["fit_ms"] if kind == "learned" else 0.0,
             fit_cccp_steps=fit.get("iters"), predict_ms=pst["predict_ms"], grid=P.Eq.shape[0],
             k_apply="symv" if st["symmetric_k"] else "gemv", p_factored=st["p_factored"],
             k_apply_ms=st["op_ms"] / max(st["op_launches"], 1),
             k_apply_gbs=((4.0 * P.n * (P.n + 1) if st["symmetric_k"] else 8.0 * P.n * P.n) + 16 * P.n)
             / (st["op_ms"] / max(st["op_launches"], 1)) / 1e6,
             p_apply_ms=st["prec_ms"] / max(st["prec_launches"], 1) if st["prec_launches"] else None,
             kappa_PA_lanczos=reps[0]["lanczos_lmax"] / reps[0]["lanczos_lmin"] if reps[0]["lanczos_lmin"] > 0
             else None,
             exp_inconclusive=pst["exp_inconclusive"])
    c.close()


def run_c4(modes=("fast", "exact"), nrhs=64):
    import torch
    P = make_problem(4, nrhs=nrhs)
    dev = torch.device("cuda", 0)
    c = L.Context(0)
    for mode in modes:
        md = L.MODE_FAST if mode == "fast" else L.MODE_EXACT
        c.assemble_kernel(torch.from_numpy(P.E).to(dev), P.scale, P.lam, L.STORE_MATERIALIZED, md)
        c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
        Yt = torch.from_numpy(np.ascontiguousarray(P.Y.T)).to(dev)   # (nrhs, n) = column-major n x nrhs
        t0 = time.perf_counter()
        A, reps, _ = c.pcg_solve(Yt, P.tol)
        wall = time.perf_counter() - t0
        its = [r["iters"] for r in reps]
        secs = reps[0]["seconds"]
        emit(config="C4", n=P.n, nrhs=nrhs, mode=mode, precond="learned", iters_max=max(its),
             iters_min=min(its), all_converged=all(r["termination"] == 0 for r in reps),
             worst_true_rel=max(r["true_rel_residual"] for r in reps), time_to_solution_s=secs,
             block_iters_per_s=max(its) / secs, rhs_iters_per_s=sum(its) / secs, wall_s=wall)
    c.close()


def run_c5(iters=20, grid=True):
    import torch
    P = make_problem(5)
    dev = torch.device("cuda", 0)
    c = L.Context(0)
    E = torch.from_numpy(P.E).to(dev)
    for mode in ("fast", "exact"):
        md = L.MODE_FAST if mode == "fast" else L.MODE_EXACT
        c.assemble_kernel(E, P.scale, P.lam, L.STORE_ON_THE_FLY, md)
        c.fit_preconditioner(L.PRECOND_JACOBI)
        k = iters if mode == "fast" else 2
        a, reps, _ = c.pcg_solve(torch.from_numpy(P.y).to(dev), P.tol, max_iters=k)
        per_it = reps[0]["seconds"] / reps[0]["iters"]
        flops = P.n * P.n * (2 * P.d + 2)
        emit(config="C5", n=P.n, d=P.d, mode=mode, precond="jacobi", storage="on_the_fly", iters=reps[0]["iters"],
             rel_residual=reps[0]["rel_residual"], ms_per_iter=per_it * 1e3, iters_per_s=1.0 / per_it,
             entries_per_s=P.n * P.n / per_it, tflops_dots=flops / per_it / 1e12, n_gpus=1,
             note="iterations capped: per-iteration rate of the matrix-free operator on 1 GPU")
    if grid:
        c.assemble_kernel(E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
        alpha = torch.from_numpy(np.random.default_rng(0).standard_normal(P.n)).to(dev)
        Eq = torch.from_numpy(P.Eq).to(dev)
        out = c.predict(Eq, alpha, mode=L.MODE_FAST)
        st = c.stats()
        ent = P.Eq.shape[0] * P.n
        emit(config="C5", what="predict", grid=P.Eq.shape[0], mode="fast", predict_ms=st["predict_ms"],
             entries_per_s=ent / (st["predict_ms"] * 1e-3), n_gpus=1)
    c.close()


def run_c5_learned(max_iters=4000):
    """LAKER at C5: K on the fly, LEARNED P fitted through the
    chunked directions GEMM and applied factored; full solve to the tolerance."""
    import torch
    P = make_problem(5)
    dev = torch.device("cuda", 0)
    c = L.Context(0)
    E = torch.from_numpy(P.E).to(dev)
    c.assemble_kernel(E, P.scale, P.lam, L.STORE_ON_THE_FLY, L.MODE_FAST)
    fit = c.fit_preconditioner(L.PRECOND_LEARNED, n_dirs=P.n_dirs, seed=7)
    a, reps, _ = c.pcg_solve(torch.from_numpy(P.y).to(dev), P.tol, max_iters=max_iters, instrument=True)
    r = reps[0]
    st = c.stats()
    emit(config="C5", n=P.n, d=P.d, mode="fast", precond="learned (factored)", storage="on_the_fly",
         n_dirs=fit["n_dirs"], fit_s=fit["seconds"], fit_cccp_steps=fit["iters"], iters=r["iters"],
         termination=r["termination"], rel_residual=r["rel_residual"], true_rel_residual=r["true_rel_residual"],
         solve_s=r["seconds"], ms_per_iter=r["seconds"] / max(r["iters"], 1) * 1e3,
         kappa_PA_lanczos=r["lanczos_lmax"] / r["lanczos_lmin"],
         k_apply_ms=st["op_ms"] / max(st["op_launches"], 1), p_apply_ms=st["prec_ms"] / max(st["prec_launches"], 1),
         n_gpus=1)
    c.close()


if __name__ == "__main__":
    which = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    for w in which:
        if w in ("C1", "C2", "C3"):
            run_std(int(w[1]))
        elif w == "C4":
            run_c4()
        elif w == "C4E":
            run_c4(modes=("exact",))
        elif w == "C5":
            run_c5()
        elif w == "C5L":
            run_c5_learned()
