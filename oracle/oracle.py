"""fp64 CPU oracle for the LAKER hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference for what the CUDA library computes.
Line citations "P:n" are to /root/reference/PAPER.md (LaTeX of arXiv
2604.25138); "S:n" to SPEC.md; readings R1..R23 are listed in DESIGN.md §3.

* Exact-arithmetic parts (kernel entries with a correctly rounded exp, Dot2
  inner products, the PCG recursion of Alg. 1) are in liblaker_oracle.so
  (oracle/laker_oracle.c), called through ctypes.
* The CCCP preconditioner fit (Alg. 1 l.5-14; Eqs.
  kernel_shrinkage_cccp_F/_Sigma/_normalization) is written here in
  numpy, with LAPACK primitives (matmul, Cholesky, triangular solve, QR,
  symmetric eigendecomposition) as single steps and no blocking or fusion:
    - `cccp_fit_literal`: the iteration on the dense n x n Sigma_t exactly as
      written (the definition);
    - `cccp_fit_structured`: an exact algebraic restatement (DESIGN.md §3,
      reading O4'): Sigma_t = a_t I + U diag(b_t) U^T for t >= 1, so the
      iteration runs on (a_t, b_t) with the N_r x N_r matrix
      T_t = a_t I + R diag(b_t) R^T after one thin QR U = Q R.  Pinned against
      the literal form in tests/test_oracle_fit.py.
* `block_pcg`: O'Leary's block PCG (1980) for the C4 block-CG variant, plain numpy;
  pinned by its one-column case (= Alg. 1's PCG, `pcg`), finite termination on a
  spectrum of k distinct eigenvalues (<= ceil(k/m) steps), an exact preconditioner
  (one step) and the dense solve (tests/test_oracle_block_cg.py).
* `reference_solve`: dense Cholesky solve of (lambda I + K) alpha = y, the
  stand-in for the paper's CVXPY reference.
"""
from __future__ import annotations

import ctypes
from collections import namedtuple
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.linalg as sla

__all__ = [
    "lib", "exp_cr", "dot2", "assemble", "assemble_rows", "cross_kernel", "predict",
    "apply", "dense_apply", "factored_apply", "factored_qm_apply", "pcg_factored_qm", "jacobi_diag", "pcg", "pcg_factored", "PcgReport",
    "P_NONE", "P_JACOBI", "P_DENSE", "factors", "TERM_RESIDUAL_TOL", "TERM_MAX_ITERS", "TERM_ZERO_RHS", "TERM_BREAKDOWN",
    "TERM_INDEFINITE", "rho_schedule", "nr_schedule", "directions", "cccp_step_literal",
    "cccp_fit_literal",
    "cccp_fit_structured", "FitReport", "reference_solve", "cond_spd", "cond_precond",
    "objective", "residual", "num_threads", "block_pcg", "BlockPcgReport",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liblaker_oracle.so")


def _load():
    src = os.path.join(_HERE, "laker_oracle.c")
    if (not os.path.exists(_SO)) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    L = ctypes.CDLL(_SO)
    D = ctypes.POINTER(ctypes.c_double)
    i64, i32, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    L.orc_dot2.argtypes = [i64, D, D]; L.orc_dot2.restype = dbl
    L.orc_exp_cr.argtypes = [dbl]; L.orc_exp_cr.restype = dbl
    L.orc_assemble.argtypes = [i64, i32, D, dbl, D]; L.orc_assemble.restype = i64
    L.orc_assemble_rows.argtypes = [i64, i32, D, dbl, i64, i64, D]; L.orc_assemble_rows.restype = i64
    L.orc_cross_kernel.argtypes = [i64, i64, i32, D, D, dbl, D]; L.orc_cross_kernel.restype = i64
    L.orc_predict.argtypes = [i64, i64, i32, D, D, dbl, D, D]; L.orc_predict.restype = i64
    L.orc_apply.argtypes = [i64, D, dbl, D, D]; L.orc_apply.restype = None
    L.orc_dense_apply.argtypes = [i64, D, D, D]; L.orc_dense_apply.restype = None
    L.orc_jacobi_diag.argtypes = [i64, i32, D, dbl, dbl, D]; L.orc_jacobi_diag.restype = i64
    L.orc_pcg.argtypes = [i64, D, dbl, D, ctypes.c_int, D, dbl, i32, D, ctypes.c_void_p, D]
    L.orc_pcg.restype = ctypes.c_int
    L.orc_factored_apply.argtypes = [i64, i64, D, D, dbl, D, D]; L.orc_factored_apply.restype = None
    L.orc_pcg_factored.argtypes = [i64, D, dbl, D, i64, D, D, dbl, dbl, i32, D, ctypes.c_void_p, D]
    L.orc_pcg_factored.restype = ctypes.c_int
    L.orc_factored_qm_apply.argtypes = [i64, i64, D, D, dbl, D, D]; L.orc_factored_qm_apply.restype = None
    L.orc_pcg_factored_qm.argtypes = [i64, D, dbl, D, i64, D, D, dbl, dbl, i32, D, ctypes.c_void_p, D]
    L.orc_pcg_factored_qm.restype = ctypes.c_int
    L.orc_num_threads.argtypes = []; L.orc_num_threads.restype = ctypes.c_int
    return L


lib = _load()


def _p(a: Optional[np.ndarray]):
    if a is None:
        return ctypes.POINTER(ctypes.c_double)()
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return int(lib.orc_num_threads())


# ------------------------------------------------------------- exact pieces
def exp_cr(x: float) -> float:
    """Correctly rounded exp (binary128 expq rounded once; reading R18)."""
    return float(lib.orc_exp_cr(float(x)))


def dot2(x, y) -> float:
    """Dot2 (Ogita-Rump-Oishi 2005, Alg. 5.3) in index order (reading R17)."""
    x, y = _c(x), _c(y)
    assert x.shape == y.shape and x.ndim == 1
    return float(lib.orc_dot2(x.size, _p(x), _p(y)))


def assemble(E, scale: float):
    """K = exp(scale E E^T) elementwise, P:141-147 / Alg. 1 l.3; scale
    per reading R1.  Returns (K, n_overflow)."""
    E = _c(E)
    n, d = E.shape
    K = np.empty((n, n))
    nov = lib.orc_assemble(n, d, _p(E), float(scale), _p(K))
    return K, int(nov)


def assemble_rows(E, scale: float, r0: int, r1: int) -> np.ndarray:
    E = _c(E)
    n, d = E.shape
    K = np.empty((r1 - r0, n))
    lib.orc_assemble_rows(n, d, _p(E), float(scale), r0, r1, _p(K))
    return K


def cross_kernel(Eq, E, scale: float) -> np.ndarray:
    """k(x_m, x_i) = exp(scale <e(x_m), e_i>)."""
    Eq, E = _c(Eq), _c(E)
    m, d = Eq.shape
    n = E.shape[0]
    Kx = np.empty((m, n))
    lib.orc_cross_kernel(m, n, d, _p(Eq), _p(E), float(scale), _p(Kx))
    return Kx


def predict(Eq, E, scale: float, alpha) -> np.ndarray:
    """r_hat(x) = sum_i k(x, x_i) alpha_i, Eq. sc-radio-map-reconstruction
    (P:164-172), Alg. 1 l.24; Dot2 over i."""
    Eq, E, alpha = _c(Eq), _c(E), _c(alpha)
    m, d = Eq.shape
    n = E.shape[0]
    out = np.empty(m)
    lib.orc_predict(m, n, d, _p(Eq), _p(E), float(scale), _p(alpha), _p(out))
    return out


def apply(K, lam: float, p) -> np.ndarray:
    """q = (lambda I + K) p, one Dot2 per row over n+1 terms."""
    K, p = _c(K), _c(p)
    q = np.empty(K.shape[0])
    lib.orc_apply(K.shape[0], _p(K), float(lam), _p(p), _p(q))
    return q


def dense_apply(P, r) -> np.ndarray:
    P, r = _c(P), _c(r)
    th = np.empty(P.shape[0])
    lib.orc_dense_apply(P.shape[0], _p(P), _p(r), _p(th))
    return th


def factored_apply(Q, M, ainv: float, r) -> np.ndarray:
    """theta = P r with P = ainv I + Q M Q^T held in factored form (P:273-278 via
    O4'): z = Q^T r, w = M z, theta_i = ainv r_i + Q_i. w, each entry one Dot2."""
    Q, M, r = _c(Q), _c(M), _c(r)
    n, m = Q.shape
    th = np.empty(n)
    lib.orc_factored_apply(n, m, _p(Q), _p(M), float(ainv), _p(r), _p(th))
    return th


def factored_qm_apply(Q, QM, ainv: float, r) -> np.ndarray:
    """theta = P r with P = ainv I + Q M Q^T applied as ainv r + QM (Q^T r), QM = Q M given
    (the same product associated (Q M) z instead of Q (M z); R21): z = Q^T r and
    theta_i = ainv r_i + QM_i. z, each entry one Dot2."""
    Q, QM, r = _c(Q), _c(QM), _c(r)
    n, m = Q.shape
    th = np.empty(n)
    lib.orc_factored_qm_apply(n, m, _p(Q), _p(QM), float(ainv), _p(r), _p(th))
    return th


def jacobi_diag(E, scale: float, lam: float) -> np.ndarray:
    """P_J = diag(lambda I + G)^{-1}."""
    E = _c(E)
    n, d = E.shape
    dv = np.empty(n)
    lib.orc_jacobi_diag(n, d, _p(E), float(scale), float(lam), _p(dv))
    return dv


P_NONE, P_JACOBI, P_DENSE = 0, 1, 2
TERM_RESIDUAL_TOL, TERM_MAX_ITERS, TERM_ZERO_RHS, TERM_BREAKDOWN, TERM_INDEFINITE = 0, 1, 2, 3, 4


class _CReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("termination", ctypes.c_int32),
                ("rel_residual", ctypes.c_double), ("true_rel_residual", ctypes.c_double)]


@dataclass
class PcgReport:
    iters: int
    termination: int
    rel_residual: float
    true_rel_residual: float
    history: np.ndarray = field(repr=False, default=None)


def pcg(K, lam: float, y, pkind: int = P_NONE, P=None, tol: float = 1e-10,
        max_iters: Optional[int] = None):
    """Alg. 1 PCG block verbatim.  P: None / diag (n) / dense n x n.
    Returns (alpha, PcgReport)."""
    K, y = _c(K), _c(y)
    n = K.shape[0]
    max_iters = 10 * n if max_iters is None else int(max_iters)
    Pa = None if pkind == P_NONE else _c(P)
    alpha = np.empty(n)
    hist = np.zeros(max(max_iters, 1))
    rep = _CReport()
    lib.orc_pcg(n, _p(K), float(lam), _p(y), int(pkind), _p(Pa), float(tol), max_iters,
                _p(alpha), ctypes.byref(rep), _p(hist))
    return alpha, PcgReport(rep.iters, rep.termination, rep.rel_residual, rep.true_rel_residual,
                            hist[: rep.iters].copy())


# --------------------------------------------------------------- CCCP fit
def pcg_factored(K, lam: float, y, Q, M, ainv: float, tol: float = 1e-10,
                 max_iters: Optional[int] = None):
    """`pcg` with the factored preconditioner of `factored_apply`."""
    K, y, Q, M = _c(K), _c(y), _c(Q), _c(M)
    n = K.shape[0]
    max_iters = 10 * n if max_iters is None else int(max_iters)
    alpha = np.empty(n)
    hist = np.zeros(max(max_iters, 1))
    rep = _CReport()
    lib.orc_pcg_factored(n, _p(K), float(lam), _p(y), Q.shape[1], _p(Q), _p(M), float(ainv), float(tol),
                         max_iters, _p(alpha), ctypes.byref(rep), _p(hist))
    return alpha, PcgReport(rep.iters, rep.termination, rep.rel_residual, rep.true_rel_residual,
                            hist[: rep.iters].copy())


def pcg_factored_qm(K, lam: float, y, Q, QM, ainv: float, tol: float = 1e-10,
                    max_iters: Optional[int] = None):
    """`pcg` with the factored preconditioner in the QM form of `factored_qm_apply`."""
    K, y, Q, QM = _c(K), _c(y), _c(Q), _c(QM)
    n = K.shape[0]
    max_iters = 10 * n if max_iters is None else int(max_iters)
    alpha = np.empty(n)
    hist = np.zeros(max(max_iters, 1))
    rep = _CReport()
    lib.orc_pcg_factored_qm(n, _p(K), float(lam), _p(y), Q.shape[1], _p(Q), _p(QM), float(ainv), float(tol),
                            max_iters, _p(alpha), ctypes.byref(rep), _p(hist))
    return alpha, PcgReport(rep.iters, rep.termination, rep.rel_residual, rep.true_rel_residual,
                            hist[: rep.iters].copy())


def nr_schedule(n: int) -> int:
    """N_r = min(n, max(ceil(8 sqrt n), ceil(n/4))) (P:743 shape)."""
    return int(min(n, max(math.ceil(8.0 * math.sqrt(n)), math.ceil(n / 4.0))))


def rho_schedule(n_dirs: int, n: int, gamma: float, lmin: float, rho_floor: float = 1e-3) -> float:
    """Reading R6 (P:508 vs P:743): rho = eps_rho when N_r >= n, else
    clamp(eps_rho + 0.5 (1 - N_r/n) min(1, 10 gamma), eps_rho, 0.9); and
    rho <- max(rho, 0.2) when lambda_min(Sigma_t) < 1e-6."""
    if n_dirs >= n:
        rho = rho_floor
    else:
        rho = min(max(rho_floor + 0.5 * (1.0 - n_dirs / n) * min(1.0, 10.0 * gamma), rho_floor), 0.9)
    if lmin < 1e-6:
        rho = max(rho, 0.2)
    return rho


def directions(K, lam: float, Z):
    """u_k = (lambda I + K) z_k, ubar_k = u_k / ||u_k|| (Eq. random_directions,
    P:236-245; Alg. 1 l.6).  Plain fp64 matmul (library primitive)."""
    K = np.asarray(K, dtype=np.float64)
    Z = np.asarray(Z, dtype=np.float64)
    U = lam * Z + K @ Z
    norms = np.sqrt((U * U).sum(axis=0))
    return U / norms, norms


@dataclass
class FitReport:
    iters: int
    n_dirs: int
    converged: bool
    final_change: float
    rho_used: float
    sigma_min_eig: float
    trace: float
    changes: list = field(default_factory=list, repr=False)
    rhos: list = field(default_factory=list, repr=False)


def _inv_sqrt_spd(S: np.ndarray) -> np.ndarray:
    """S^{-1/2} = V diag(w^{-1/2}) V^T by symmetric eigendecomposition, symmetrized."""
    w, V = np.linalg.eigh(S)
    if w[0] <= 0:
        raise np.linalg.LinAlgError("not positive definite")
    P = (V * (1.0 / np.sqrt(w))) @ V.T
    return 0.5 * (P + P.T)


def cccp_step_literal(Sigma, Ubar, gamma: float, eps: float, rho: float,
                      return_tilde: bool = False):
    """One map T(Sigma) of Theorem 1: F_gamma,eps, the
    shrinkage and the trace normalization.
    ubar_k^T Sigma^{-1} ubar_k via one Cholesky of Sigma and a triangular solve."""
    n, Nr = Ubar.shape
    I = np.eye(n)
    L = np.linalg.cholesky(Sigma)
    X = sla.solve_triangular(L, Ubar, lower=True)
    qf = (X * X).sum(axis=0)
    w = 1.0 / (qf + eps)
    F = ((n / Nr) * ((Ubar * w) @ Ubar.T) + gamma * I) / (1.0 + gamma / n)
    St = (1.0 - rho) * F + rho * I
    Snew = St / (np.trace(St) / n)
    if return_tilde:
        return Snew, St
    return Snew


def cccp_fit_literal(K, lam: float, Z, gamma: float = 0.1, eps: float = 1e-12,
                     rho: Optional[float] = None, rho_floor: float = 1e-3,
                     max_iters: int = 200, fp_tol: float = 1e-8, Ubar=None,
                     return_sigma: bool = False):
    """Alg. 1 l.5-14 on the dense n x n Sigma, as written:
        F_gamma(Sigma_t) = (1+gamma/n)^{-1} [ (n/N_r) sum_k ubar_k ubar_k^T /
                           (ubar_k^T Sigma_t^{-1} ubar_k + eps) + gamma I ]
        Sigma~ = (1-rho) F + rho I
        Sigma_{t+1} = Sigma~ / (tr Sigma~ / n)
    until ||Sigma_{t+1} - Sigma_t||_F / ||Sigma_t||_F <= fp_tol (reading R8);
    P = Sigma*^{-1/2} (Eq. preconditioner-Sigmma).
    Quadratic forms via one Cholesky of Sigma_t and a triangular solve.
    rho=None -> rho_schedule with lambda_min(Sigma_t) from eigvalsh."""
    if Ubar is None:
        Ubar, _ = directions(K, lam, Z)
    n, Nr = Ubar.shape
    Sigma = np.eye(n)
    rep = FitReport(0, Nr, False, float("nan"), float("nan"), float("nan"), float("nan"))
    for t in range(max_iters):
        lmin = float(np.linalg.eigvalsh(Sigma)[0])
        rho_t = rho_schedule(Nr, n, gamma, lmin, rho_floor) if rho is None else float(rho)
        Snew = cccp_step_literal(Sigma, Ubar, gamma, eps, rho_t)
        change = float(np.linalg.norm(Snew - Sigma, "fro") / np.linalg.norm(Sigma, "fro"))
        Sigma = Snew
        rep.iters, rep.final_change, rep.rho_used = t + 1, change, rho_t
        rep.changes.append(change)
        rep.rhos.append(rho_t)
        if change <= fp_tol:
            rep.converged = True
            break
    rep.sigma_min_eig = float(np.linalg.eigvalsh(Sigma)[0])
    rep.trace = float(np.trace(Sigma))
    P = _inv_sqrt_spd(Sigma)
    if return_sigma:
        return P, rep, Sigma
    return P, rep


@dataclass
class StructuredState:
    a: float
    b: np.ndarray
    Q: np.ndarray
    R: np.ndarray
    C: np.ndarray
    T: np.ndarray
    Ubar: np.ndarray


def cccp_fit_structured(K, lam: float, Z, gamma: float = 0.1, eps: float = 1e-12,
                        rho: Optional[float] = None, rho_floor: float = 1e-3,
                        max_iters: int = 200, fp_tol: float = 1e-8, Ubar=None,
                        form_P: bool = True):
    """The same iteration as `cccp_fit_literal`, restated exactly (O4'):
    Sigma_t = a_t I + Ubar diag(b_t) Ubar^T (Sigma_0 = I: a_0 = 1, b_0 = 0).
    With Ubar = Q R (Householder thin QR, diag R >= 0) and
    T_t = a_t I + R diag(b_t) R^T: Sigma_t Q = Q T_t, hence
        qf_k = ubar_k^T Sigma_t^{-1} ubar_k = (R e_k)^T T_t^{-1} (R e_k),
    Sigma~ = a' I + Ubar diag(b') Ubar^T with a' = (1-rho) gamma/(1+gamma/n) + rho,
    b'_k = (1-rho)(n/N_r) w_k/(1+gamma/n), tr Sigma~ = n a' + sum_k b'_k C_kk
    (C = Ubar^T Ubar), and (a_{t+1}, b_{t+1}) = n (a', b') / tr Sigma~.
    ||Sigma_{t+1}-Sigma_t||_F^2 = n da^2 + 2 da sum_k db_k C_kk + db^T (C o C) db.
    lambda_min(Sigma_t) = a_t when rank(Ubar) < n.
    P = Sigma*^{-1/2} = a^{-1/2} I + Q (T^{-1/2} - a^{-1/2} I) Q^T."""
    if Ubar is None:
        Ubar, _ = directions(K, lam, Z)
    n, Nr = Ubar.shape
    Q, R = np.linalg.qr(Ubar, mode="reduced")
    s = np.sign(np.diag(R))
    s[s == 0] = 1.0
    Q, R = Q * s, R * s[:, None]
    m = R.shape[0]
    C = Ubar.T @ Ubar
    cd = np.diag(C).copy()
    C2 = C * C
    a, b = 1.0, np.zeros(Nr)
    rep = FitReport(0, Nr, False, float("nan"), float("nan"), float("nan"), float("nan"))
    Im = np.eye(m)
    for t in range(max_iters):
        T = a * Im + (R * b) @ R.T
        lmin = a if m < n else float(np.linalg.eigvalsh(T)[0])
        rho_t = rho_schedule(Nr, n, gamma, lmin, rho_floor) if rho is None else float(rho)
        L = np.linalg.cholesky(T)
        X = sla.solve_triangular(L, R, lower=True)
        qf = (X * X).sum(axis=0)
        w = 1.0 / (qf + eps)
        a1 = (1.0 - rho_t) * gamma / (1.0 + gamma / n) + rho_t
        b1 = (1.0 - rho_t) * (n / Nr) * w / (1.0 + gamma / n)
        tr = n * a1 + float((b1 * cd).sum())
        an, bn = n * a1 / tr, n * b1 / tr
        da, db = an - a, bn - b
        d2 = n * da * da + 2.0 * da * float((db * cd).sum()) + float(db @ C2 @ db)
        s2 = n * a * a + 2.0 * a * float((b * cd).sum()) + float(b @ C2 @ b)
        change = math.sqrt(max(d2, 0.0)) / math.sqrt(s2)
        a, b = an, bn
        rep.iters, rep.final_change, rep.rho_used = t + 1, change, rho_t
        rep.changes.append(change)
        rep.rhos.append(rho_t)
        if change <= fp_tol:
            rep.converged = True
            break
    T = a * Im + (R * b) @ R.T
    rep.sigma_min_eig = a if m < n else float(np.linalg.eigvalsh(T)[0])
    rep.trace = n * a + float((b * cd).sum())
    state = StructuredState(a=a, b=b, Q=Q, R=R, C=C, T=T, Ubar=Ubar)
    if not form_P:
        return None, rep, state
    Ti = _inv_sqrt_spd(T)
    M = Ti - Im / math.sqrt(a)
    P = np.eye(n) / math.sqrt(a) + Q @ M @ Q.T
    return 0.5 * (P + P.T), rep, state


def factors(state) -> tuple:
    """(Q, M, a^{-1/2}) of P = Sigma*^{-1/2} = a^{-1/2} I + Q (T^{-1/2} - a^{-1/2} I) Q^T
    from a `cccp_fit_structured` state (O4')."""
    a = state.a
    M = _inv_sqrt_spd(state.T) - np.eye(state.T.shape[0]) / math.sqrt(a)
    return state.Q, 0.5 * (M + M.T), 1.0 / math.sqrt(a)


# ------------------------------------------------------- reference + metrics
def reference_solve(K, lam: float, y) -> np.ndarray:
    """alpha = (lambda I + K)^{-1} y by dense Cholesky (O5; stand-in for the
    paper's CVXPY reference)."""
    A = np.asarray(K, dtype=np.float64) + lam * np.eye(K.shape[0])
    return sla.cho_solve(sla.cho_factor(A, lower=True), np.asarray(y, dtype=np.float64))


def cond_spd(A) -> float:
    w = np.linalg.eigvalsh(A)
    return float(w[-1] / w[0])


def cond_precond(P, A) -> float:
    """kappa(P A) evaluated on P^{1/2} A P^{1/2}."""
    w, V = np.linalg.eigh(P)
    Ph = (V * np.sqrt(w)) @ V.T
    return cond_spd(Ph @ A @ Ph)


def objective(K, lam: float, alpha, y) -> float:
    """R(alpha) = ||G alpha - y||^2 + lambda alpha^T G alpha (Eq. simu-R)."""
    Ga = K @ alpha
    return float((Ga - y) @ (Ga - y) + lam * (alpha @ Ga))


def residual(K, lam: float, alpha, y) -> float:
    """Res = ||(lambda I + G) alpha - y|| / ||y|| (Eq. residual)."""
    r = K @ alpha + lam * alpha - y
    return float(np.linalg.norm(r) / np.linalg.norm(y))


BlockPcgReport = namedtuple("BlockPcgReport", "iters termination rel_residual true_rel_residual")


def block_pcg(K, lam: float, Y, precond=None, tol: float = 1e-8, max_iters: Optional[int] = None,
              plain: bool = False):
    """Block PCG (O'Leary, "The block conjugate gradient algorithm and related methods",
    Linear Algebra Appl. 29, 1980, Alg. BPCG) for (lambda I + K) X = Y with the m columns
    of Y sharing one block Krylov space -- the block-CG variant of C4 (SURVEY §8(f)
    NEXT-4, reading R13's alternative).  `precond(R)` returns P R (None: P = I).
    Written out as published, with m x m solves by Cholesky:
        X0 = 0, R0 = Y, Z0 = P R0, D0 = Z0
        Q = A D_k;  alpha_k = (D_k^T Q)^{-1} (Z_k^T R_k)
        X_{k+1} = X_k + D_k alpha_k;  R_{k+1} = R_k - Q alpha_k
        Z_{k+1} = P R_{k+1};  beta_k = (Z_k^T R_k)^{-1} (Z_{k+1}^T R_{k+1})
        D_{k+1} = Z_{k+1} + D_k beta_k
    stopping when every column has ||R_c|| / ||Y_c|| <= tol.  Termination: RESIDUAL_TOL,
    MAX_ITERS, or BREAKDOWN when an m x m Gram matrix is not numerically positive definite.
    The operator applies A D column by column with `apply` (one Dot2 per row, as Alg. 1's
    products, R17) unless `plain` (numpy K @ D); Gram matrices and m x m solves plain numpy.
    Block CG's step count is sensitive to the products' rounding (n = 1024, m = 8, Jacobi:
    168 steps with Dot2 products, 203 with plain ones), so the GPU is compared within an
    envelope, never bitwise."""
    K = np.asarray(K, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    if Y.ndim == 1:
        Y = Y[:, None]
    n, m = Y.shape
    max_iters = 10 * n if max_iters is None else int(max_iters)
    if plain:
        A = lambda V: K @ V + lam * V  # noqa: E731
    else:
        A = lambda V: np.column_stack([apply(K, lam, np.ascontiguousarray(V[:, c]))  # noqa: E731
                                       for c in range(V.shape[1])])
    P = (lambda V: V) if precond is None else precond  # noqa: E731
    ynorm = np.linalg.norm(Y, axis=0)
    X = np.zeros((n, m))
    R = Y.copy()
    Z = P(R)
    D = Z.copy()
    Gzr = Z.T @ R
    term, it = TERM_MAX_ITERS, 0
    rel = np.linalg.norm(R, axis=0) / ynorm
    for it in range(1, max_iters + 1):
        Q = A(D)
        try:
            alpha = sla.cho_solve(sla.cho_factor(D.T @ Q, lower=True), Gzr)
        except np.linalg.LinAlgError:
            term = TERM_BREAKDOWN
            break
        X = X + D @ alpha
        R = R - Q @ alpha
        rel = np.linalg.norm(R, axis=0) / ynorm
        if np.all(rel <= tol):
            term = TERM_RESIDUAL_TOL
            break
        Z = P(R)
        Gzr_new = Z.T @ R
        try:
            beta = sla.cho_solve(sla.cho_factor(Gzr, lower=True), Gzr_new)
        except np.linalg.LinAlgError:
            term = TERM_BREAKDOWN
            break
        D = Z + D @ beta
        Gzr = Gzr_new
    true = np.linalg.norm(Y - A(X), axis=0) / ynorm
    return X, BlockPcgReport(it, term, rel, true)
