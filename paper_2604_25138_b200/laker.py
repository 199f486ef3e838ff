"""Thin ctypes binding of liblaker.so (include/laker.h) -- argument marshalling
only; every step of the hot path runs in the library's CUDA kernels.

Module-level functions carry the C names (laker_create, laker_assemble_kernel,
laker_fit_preconditioner, laker_pcg_solve, laker_predict, ...).  `Context`
is a convenience wrapper over them.  Arrays may be numpy (host) or torch
tensors (host or CUDA); fp64, C-contiguous (multi-RHS blocks: n x nrhs
column-major, i.e. numpy order='F' or a torch tensor of shape (nrhs, n)).

There is no CPU fallback: importing this module fails loudly if liblaker.so
is missing or cannot be loaded, and laker_create fails without a GPU.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# LAKER_LIB_PATH: an alternative build of the same library (tools/ A/B experiments only)
LIB_PATH = os.environ.get("LAKER_LIB_PATH") or os.path.join(_HERE, "liblaker.so")

LAKER_OK = 0
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "DIMENSION_MISMATCH", 3: "NOT_READY", 4: "CUDA", 5: "NCCL",
          6: "OUT_OF_MEMORY", 7: "NOT_POSITIVE_DEFINITE", 8: "INDEFINITE_PRECONDITIONER",
          9: "BREAKDOWN_ZERO_CURVATURE", 10: "OVERFLOW", 11: "INTERNAL"}
STORE_MATERIALIZED, STORE_ON_THE_FLY = 0, 1
MODE_FAST, MODE_EXACT = 0, 1
PRECOND_NONE, PRECOND_JACOBI, PRECOND_LEARNED, PRECOND_EXTERNAL_DENSE = 0, 1, 2, 3
P_AUTO, P_DENSE, P_FACTORED, P_FACTORED_QM = 0, 1, 2, 3
TERM_RESIDUAL_TOL, TERM_MAX_ITERS, TERM_ZERO_RHS, TERM_BREAKDOWN, TERM_INDEFINITE = 0, 1, 2, 3, 4

EXPORTED = ["laker_get_unique_id", "laker_create", "laker_destroy", "laker_status_string",
            "laker_last_error", "laker_assemble_kernel", "laker_fit_preconditioner", "laker_pcg_solve",
            "laker_block_cg_solve",
            "laker_predict", "laker_load_kernel_rows", "laker_get_kernel_rows", "laker_set_preconditioner",
            "laker_get_preconditioner_rows", "laker_get_preconditioner_factors", "laker_get_preconditioner_qm",
            "laker_apply_operator",
            "laker_get_stats", "laker_debug_igemm_s8", "laker_debug_ozaki_gemm", "laker_debug_dist_tiles",
            "laker_debug_dist_symv_partials", "laker_debug_dist_symv_combine", "laker_debug_tc_groups"]


class LakerError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class FitOpts(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_dirs", ctypes.c_int32), ("gamma", ctypes.c_double),
                ("eps", ctypes.c_double), ("rho", ctypes.c_double), ("rho_floor", ctypes.c_double),
                ("max_iters", ctypes.c_int32), ("fp_tol", ctypes.c_double), ("Z", ctypes.c_void_p),
                ("seed", ctypes.c_uint64), ("p_layout", ctypes.c_int32)]


class FitReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("n_dirs", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("final_change", ctypes.c_double), ("rho_used", ctypes.c_double),
                ("sigma_min_eig", ctypes.c_double), ("trace", ctypes.c_double), ("seconds", ctypes.c_double)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iters", ctypes.c_int32), ("instrument", ctypes.c_int32)]


class SolveReport(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("termination", ctypes.c_int32), ("rel_residual", ctypes.c_double),
                ("true_rel_residual", ctypes.c_double), ("seconds", ctypes.c_double),
                ("lanczos_lmin", ctypes.c_double), ("lanczos_lmax", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("local_rows", ctypes.c_int64), ("ld", ctypes.c_int64),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("precond_kind", ctypes.c_int32),
                ("storage", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("exp_inconclusive", ctypes.c_uint64), ("exp_overflow", ctypes.c_uint64),
                ("op_ms", ctypes.c_double), ("prec_ms", ctypes.c_double),
                ("op_launches", ctypes.c_int64), ("prec_launches", ctypes.c_int64),
                ("assemble_ms", ctypes.c_double), ("fit_ms", ctypes.c_double),
                ("solve_ms", ctypes.c_double), ("predict_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64),
                ("symmetric_k", ctypes.c_int32), ("symmetric_p", ctypes.c_int32),
                ("p_factored", ctypes.c_int32), ("n_dirs", ctypes.c_int32),
                ("k_tensor_core", ctypes.c_int32), ("pad0", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_25138_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, dbl, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    sig = {
        "laker_get_unique_id": [vp],
        "laker_create": [ctypes.POINTER(vp), st, st, st, vp, vp],
        "laker_destroy": [vp],
        "laker_assemble_kernel": [vp, i64, i32, vp, dbl, dbl, st, st],
        "laker_fit_preconditioner": [vp, ctypes.POINTER(FitOpts), ctypes.POINTER(FitReport)],
        "laker_pcg_solve": [vp, i32, vp, vp, ctypes.POINTER(SolveOpts), ctypes.POINTER(SolveReport), vp],
        "laker_block_cg_solve": [vp, i32, i32, vp, vp, ctypes.POINTER(SolveOpts), ctypes.POINTER(SolveReport), vp],
        "laker_predict": [vp, i64, vp, vp, vp, st],
        "laker_load_kernel_rows": [vp, vp],
        "laker_get_kernel_rows": [vp, vp],
        "laker_set_preconditioner": [vp, st, vp],
        "laker_get_preconditioner_rows": [vp, vp],
        "laker_get_preconditioner_factors": [vp, vp, vp, vp],
        "laker_get_preconditioner_qm": [vp, vp],
        "laker_apply_operator": [vp, vp, vp],
        "laker_get_stats": [vp, ctypes.POINTER(Stats)],
        "laker_debug_igemm_s8": [vp, vp, vp, i64, i64, i64],
        "laker_debug_ozaki_gemm": [vp, vp, vp, i64, i64, i64, i32, i32],
        "laker_debug_dist_tiles": [i64, i32, i32, i32, i32, vp, vp, vp, vp, vp],
        "laker_debug_dist_symv_partials": [vp, vp, vp, vp],
        "laker_debug_dist_symv_combine": [vp, vp, vp, vp, vp, vp],
        "laker_debug_tc_groups": [vp, vp, vp, vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = st
    L.laker_status_string.argtypes = [st]
    L.laker_status_string.restype = ctypes.c_char_p
    L.laker_last_error.argtypes = [vp]
    L.laker_last_error.restype = ctypes.c_char_p
    return L


lib = _load()


# ------------------------------------------------------------ marshalling
def _ptr(a, dtype=np.float64) -> Optional[int]:
    """Data pointer of a numpy array or torch tensor (fp64, contiguous)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype:
            raise TypeError(f"expected {dtype}, got {a.dtype}")
        if not (a.flags.c_contiguous or a.flags.f_contiguous):
            raise ValueError("array must be contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):  # torch.Tensor
        import torch
        if a.dtype != torch.float64:
            raise TypeError(f"expected torch.float64, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported buffer type {type(a)}")


def _check(ctx, s: int):
    if s != LAKER_OK:
        msg = lib.laker_last_error(ctx).decode() if ctx else lib.laker_status_string(s).decode()
        raise LakerError(s, msg)


# ----------------------------------------------------- C-named functions
def laker_status_string(status: int) -> str:
    return lib.laker_status_string(int(status)).decode()


def laker_last_error(ctx) -> str:
    return lib.laker_last_error(ctx).decode()


def laker_get_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(None, lib.laker_get_unique_id(buf))
    return bytes(buf)


def laker_create(device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 stream: Optional[int] = None):
    h = ctypes.c_void_p()
    idbuf = (ctypes.c_ubyte * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
    s = lib.laker_create(ctypes.byref(h), device, rank, world, idbuf, stream)
    if s != LAKER_OK:
        raise LakerError(s, "laker_create failed (" + lib.laker_status_string(s).decode() + ")")
    return h


def laker_destroy(ctx):
    _check(None, lib.laker_destroy(ctx))


def laker_assemble_kernel(ctx, E, scale: float, lam: float, storage: int = STORE_MATERIALIZED,
                          mode: int = MODE_EXACT):
    n, d = E.shape
    _check(ctx, lib.laker_assemble_kernel(ctx, n, d, _ptr(E), float(scale), float(lam), storage, mode))


def laker_fit_preconditioner(ctx, kind: int, n_dirs: int = 0, gamma: float = 0.1, eps: float = 1e-12,
                             rho: float = -1.0, rho_floor: float = 1e-3, max_iters: int = 200,
                             fp_tol: float = 1e-8, Z=None, seed: int = 0, p_layout: int = P_AUTO) -> dict:
    o = FitOpts(kind, n_dirs, gamma, eps, rho, rho_floor, max_iters, fp_tol, _ptr(Z), seed, p_layout)
    r = FitReport()
    _check(ctx, lib.laker_fit_preconditioner(ctx, ctypes.byref(o), ctypes.byref(r)))
    return {f: getattr(r, f) for f, _ in FitReport._fields_}


def laker_pcg_solve(ctx, nrhs: int, Y, alpha, tol: float, max_iters: int = 0, instrument: bool = False,
                    history=None, raise_on_breakdown: bool = True):
    o = SolveOpts(tol, max_iters, 1 if instrument else 0)
    reps = (SolveReport * nrhs)()
    s = lib.laker_pcg_solve(ctx, nrhs, _ptr(Y), _ptr(alpha), ctypes.byref(o), reps, _ptr(history))
    out = [{f: getattr(r, f) for f, _ in SolveReport._fields_} for r in reps]
    if s in (8, 9) and not raise_on_breakdown:
        return out
    _check(ctx, s)
    return out


def laker_block_cg_solve(ctx, nrhs: int, Y, alpha, tol: float, max_iters: int = 0, history=None,
                         raise_on_breakdown: bool = True, block: int = 0):
    o = SolveOpts(tol, max_iters, 0)
    reps = (SolveReport * nrhs)()
    s = lib.laker_block_cg_solve(ctx, nrhs, block, _ptr(Y), _ptr(alpha), ctypes.byref(o), reps, _ptr(history))
    out = [{f: getattr(r, f) for f, _ in SolveReport._fields_} for r in reps]
    if s in (8, 9) and not raise_on_breakdown:
        return out
    _check(ctx, s)
    return out


def laker_predict(ctx, Eq, alpha, out, mode: int = MODE_EXACT):
    _check(ctx, lib.laker_predict(ctx, Eq.shape[0], _ptr(Eq), _ptr(alpha), _ptr(out), mode))


def laker_load_kernel_rows(ctx, K_rows):
    _check(ctx, lib.laker_load_kernel_rows(ctx, _ptr(K_rows)))


def laker_get_kernel_rows(ctx, K_rows):
    _check(ctx, lib.laker_get_kernel_rows(ctx, _ptr(K_rows)))


def laker_set_preconditioner(ctx, kind: int, data=None):
    _check(ctx, lib.laker_set_preconditioner(ctx, kind, _ptr(data)))


def laker_get_preconditioner_rows(ctx, P_rows):
    _check(ctx, lib.laker_get_preconditioner_rows(ctx, _ptr(P_rows)))


def laker_get_preconditioner_qm(ctx, QM) -> None:
    _check(ctx, lib.laker_get_preconditioner_qm(ctx, _ptr(QM)))


def laker_get_preconditioner_factors(ctx, Q, M, a_inv_sqrt) -> None:
    _check(ctx, lib.laker_get_preconditioner_factors(ctx, _ptr(Q), _ptr(M), _ptr(a_inv_sqrt)))


def laker_apply_operator(ctx, x, y):
    _check(ctx, lib.laker_apply_operator(ctx, _ptr(x), _ptr(y)))


def laker_get_stats(ctx) -> dict:
    s = Stats()
    _check(ctx, lib.laker_get_stats(ctx, ctypes.byref(s)))
    return {f: getattr(s, f) for f, _ in Stats._fields_}


def laker_debug_igemm_s8(A, B, C) -> None:
    """C = A B^T on the tcgen05 int8 tensor cores; torch int8 / int32 CUDA tensors."""
    M, K = A.shape
    N = B.shape[0]
    s = lib.laker_debug_igemm_s8(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K)
    if s != LAKER_OK:
        raise LakerError(s, "laker_debug_igemm_s8")


def laker_debug_ozaki_gemm(A, B, C, slices: int = 0, kernel: int = -1) -> None:
    """C = A B^T in fp64 emulated on the int8 tensor cores; torch float64 CUDA tensors."""
    M, K = A.shape
    N = B.shape[0]
    s = lib.laker_debug_ozaki_gemm(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, slices, kernel)
    if s != LAKER_OK:
        raise LakerError(s, "laker_debug_ozaki_gemm")


def laker_debug_dist_tiles(n: int, br: int, tc: int, rank: int, world: int) -> dict:
    """The tile lists of the row-sharded symmetric apply (host only, no GPU needed)."""
    cnt = np.zeros(3, dtype=np.int64)
    s = lib.laker_debug_dist_tiles(n, br, tc, rank, world, _ptr(cnt, np.int64), None, None, None, None)
    if s != LAKER_OK:
        raise LakerError(s, "laker_debug_dist_tiles")
    L, T, nct = (int(v) for v in cnt)
    toff = np.zeros(L + 1, dtype=np.int64)
    jt = np.zeros(max(T, 1), dtype=np.int32)
    lo, hi = np.zeros(nct, dtype=np.int32), np.zeros(nct, dtype=np.int32)
    s = lib.laker_debug_dist_tiles(n, br, tc, rank, world, _ptr(cnt, np.int64), _ptr(toff, np.int64),
                                   _ptr(jt, np.int32), _ptr(lo, np.int32), _ptr(hi, np.int32))
    if s != LAKER_OK:
        raise LakerError(s, "laker_debug_dist_tiles")
    return {"toff": toff, "jt": jt[:T], "cr_lo": lo, "cr_hi": hi}


def laker_debug_dist_symv_partials(ctx, x, rowmax, pairs):
    _check(ctx, lib.laker_debug_dist_symv_partials(ctx, _ptr(x), _ptr(rowmax), _ptr(pairs)))


def laker_debug_dist_symv_combine(ctx, x, own, recv, q_loc, pq_pair=None):
    _check(ctx, lib.laker_debug_dist_symv_combine(ctx, _ptr(x), _ptr(own), _ptr(recv), _ptr(q_loc), _ptr(pq_pair)))


def laker_debug_tc_groups(ctx, x, rowmax, groups):
    _check(ctx, lib.laker_debug_tc_groups(ctx, _ptr(x), _ptr(rowmax), _ptr(groups, np.int64)))


# ------------------------------------------------------------ convenience
class Context:
    """Owns one laker_ctx.  Methods are the C calls without the `laker_` prefix."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 stream: Optional[int] = None):
        self.h = laker_create(device, rank, world, nccl_id, stream)
        self.n = 0
        self.rank, self.world = rank, world

    def close(self):
        if self.h:
            laker_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def local_rows(self):
        return self.n // self.world

    def assemble_kernel(self, E, scale, lam, storage=STORE_MATERIALIZED, mode=MODE_EXACT):
        laker_assemble_kernel(self.h, E, scale, lam, storage, mode)
        self.n = E.shape[0]

    def fit_preconditioner(self, kind, **kw):
        return laker_fit_preconditioner(self.h, kind, **kw)

    def pcg_solve(self, Y, tol, max_iters=0, instrument=False, want_history=False, raise_on_breakdown=True):
        Y = np.asarray(Y, dtype=np.float64) if isinstance(Y, (list, tuple)) else Y
        if isinstance(Y, np.ndarray):
            nrhs = 1 if Y.ndim == 1 else Y.shape[1]
            Yc = np.asfortranarray(Y)
            alpha = np.zeros_like(Yc, order="F")
        else:  # torch: (n,) or (nrhs, n) contiguous
            nrhs = 1 if Y.dim() == 1 else Y.shape[0]
            Yc = Y.contiguous()
            alpha = Yc.new_zeros(Yc.shape)
        hist = None
        if want_history:
            mi = max_iters if max_iters > 0 else 10 * self.n
            hist = np.zeros(mi)
        reps = laker_pcg_solve(self.h, nrhs, Yc, alpha, tol, max_iters, instrument, hist, raise_on_breakdown)
        if hist is not None:
            hist = hist[: reps[0]["iters"]].copy()
        return alpha, reps, hist

    def block_cg_solve(self, Y, tol, max_iters=0, want_history=False, raise_on_breakdown=True, block=0):
        """O'Leary block PCG over the columns of Y (n x nrhs, nrhs <= 64) in groups of `block`
        columns (0: one group): laker_block_cg_solve."""
        Yc = np.asfortranarray(np.asarray(Y, dtype=np.float64)) if not hasattr(Y, "dim") else Y.contiguous()
        nrhs = (1 if Yc.ndim == 1 else Yc.shape[1]) if isinstance(Yc, np.ndarray) else \
            (1 if Yc.dim() == 1 else Yc.shape[0])
        alpha = np.zeros_like(Yc, order="F") if isinstance(Yc, np.ndarray) else Yc.new_zeros(Yc.shape)
        hist = np.zeros(max_iters if max_iters > 0 else 10 * self.n) if want_history else None
        reps = laker_block_cg_solve(self.h, nrhs, Yc, alpha, tol, max_iters, hist, raise_on_breakdown, block)
        if hist is not None:
            hist = hist[: reps[0]["iters"]].copy()
        return alpha, reps, hist

    def predict(self, Eq, alpha, mode=MODE_EXACT, out=None):
        if out is None:
            out = np.zeros(Eq.shape[0]) if isinstance(Eq, np.ndarray) else Eq.new_zeros(Eq.shape[0])
        laker_predict(self.h, Eq, alpha, out, mode)
        return out

    def get_kernel_rows(self):
        K = np.empty((self.local_rows, self.n))
        laker_get_kernel_rows(self.h, K)
        return K

    def load_kernel_rows(self, K_rows):
        laker_load_kernel_rows(self.h, np.ascontiguousarray(K_rows, dtype=np.float64))

    def set_preconditioner(self, kind, data=None):
        if isinstance(data, np.ndarray):
            data = np.ascontiguousarray(data, dtype=np.float64)
        laker_set_preconditioner(self.h, kind, data)

    def get_preconditioner_rows(self):
        P = np.empty((self.local_rows, self.n))
        laker_get_preconditioner_rows(self.h, P)
        return P

    def get_preconditioner_factors(self):
        """(Q n x N_r, M N_r x N_r, a^{-1/2}) of a factored LEARNED P."""
        nr = self.stats()["n_dirs"]
        Q, M, ai = np.empty((self.local_rows, nr)), np.empty((nr, nr)), np.zeros(1)
        laker_get_preconditioner_factors(self.h, Q, M, ai)
        return Q, M, float(ai[0])

    def get_preconditioner_qm(self):
        """QM = Q M (n x N_r) of a factored LEARNED P in the QM form (R21), or None."""
        if self.stats()["p_factored"] != 2:
            return None
        QM = np.empty((self.local_rows, self.stats()["n_dirs"]))
        laker_get_preconditioner_qm(self.h, QM)
        return QM

    def apply_operator(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64) if isinstance(x, np.ndarray) else x
        y = np.zeros(self.n) if isinstance(x, np.ndarray) else x.new_zeros(self.n)
        laker_apply_operator(self.h, x, y)
        return y

    def stats(self) -> dict:
        return laker_get_stats(self.h)
