"""Synthetic radio-map workloads standing in for the paper's unpublished §V
generator ("superposing multiple transmitters with
spatially decaying power profiles and log-normal shadowing") at the sizes of
BASELINE.json's five configs.  Readings R3/R4/R5/R19 of DESIGN.md §3.

Everything here is input construction: locations x_i, RSS values y_i (dBm),
embeddings e_i = q(x_i) = k(x_i) (BASELINE.json: q = k = W.[x; RFF(x)]),
grid points and random directions z_k.  The method's arithmetic (kernel,
operator, PCG, CCCP) lives in oracle/ (CPU, test-only) and in the CUDA
library; neither is imported here.

Seeds: numpy PCG64 from SeedSequence((25138, config_id, stream)) with streams
0 locations, 1 Tx positions, 2 Tx powers, 3 shadowing, 4 RFF Omega, 5 RFF
phase, 6 W, 7 Z, 8 cluster centres, 16+b band b (C4).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

SEED_ROOT = 25138
C_LIGHT = 299_792_458.0
F_CARRIER = 3.5e9


def rng(config_id: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence((SEED_ROOT, config_id, stream))))


@dataclasses.dataclass(frozen=True)
class ConfigSpec:
    cid: int
    n: int
    d: int
    lam: float
    tol: float
    layout: str          # "uniform" | "clusters"
    n_tx: int
    nrhs: int
    grid: int            # g -> g x g evaluation grid
    n_dirs: int          # N_r (0: no learned fit)
    precond: str         # "learned" | "jacobi" | "none"
    storage: str         # "materialized" | "on_the_fly"
    world: int           # GPUs the config is quoted on


# BASELINE.json configs[0..4] with the readings of SURVEY.md §8(d) M1.
CONFIGS = {
    1: ConfigSpec(1, 256, 16, 1e-3, 1e-10, "uniform", 3, 1, 64, 128, "learned", "materialized", 1),
    2: ConfigSpec(2, 2048, 32, 1e-4, 1e-8, "uniform", 3, 1, 256, 512, "learned", "materialized", 1),
    3: ConfigSpec(3, 16384, 64, 1e-4, 1e-8, "clusters", 6, 1, 256, 4096, "learned", "materialized", 1),
    4: ConfigSpec(4, 16384, 64, 1e-4, 1e-8, "clusters", 6, 64, 256, 4096, "learned", "materialized", 1),
    5: ConfigSpec(5, 65536, 64, 1e-5, 1e-8, "clusters", 6, 1, 1024, 0, "jacobi", "on_the_fly", 8),
}


@dataclasses.dataclass
class Problem:
    spec: ConfigSpec
    n: int
    d: int
    lam: float
    tol: float
    scale: float         # 1/sqrt(d) (BASELINE.json north_star; reading R1)
    X: np.ndarray        # n x 2 locations in [0,1]^2 (metres = 100 x)
    E: np.ndarray        # n x d row-major embeddings (q = k)
    Y: np.ndarray        # n x nrhs, Fortran (column-major) order, dBm
    Xq: np.ndarray       # m x 2 grid points
    Eq: np.ndarray       # m x d grid embeddings
    truth: np.ndarray    # m x nrhs shadow-free field on the grid, dBm
    n_dirs: int

    @property
    def y(self) -> np.ndarray:
        return np.ascontiguousarray(self.Y[:, 0])


# ----------------------------------------------------------------- embeddings
@dataclasses.dataclass(frozen=True)
class Embedding:
    """q(x) = W [x ; sqrt(2/D) cos(Omega x + b)], D = d (reading R3)."""
    W: np.ndarray        # d x (2 + D)
    Omega: np.ndarray    # D x 2
    b: np.ndarray        # D


def make_embedding(config_id: int, d: int, length_scale: float = 0.1) -> Embedding:
    D = d
    Omega = rng(config_id, 4).standard_normal((D, 2)) / length_scale
    b = rng(config_id, 5).uniform(0.0, 2.0 * math.pi, D)
    W = rng(config_id, 6).standard_normal((d, 2 + D)) / math.sqrt(2 + D)
    return Embedding(W=W, Omega=Omega, b=b)


def embed(emb: Embedding, X: np.ndarray) -> np.ndarray:
    D = emb.Omega.shape[0]
    phi = np.concatenate([X, math.sqrt(2.0 / D) * np.cos(X @ emb.Omega.T + emb.b)], axis=1)
    return np.ascontiguousarray(phi @ emb.W.T, dtype=np.float64)


def grid_points(g: int) -> np.ndarray:
    """Cell centres ((i+1/2)/g, (j+1/2)/g), row-major over (i, j) (reading R19)."""
    c = (np.arange(g, dtype=np.float64) + 0.5) / g
    gx, gy = np.meshgrid(c, c, indexing="ij")
    return np.ascontiguousarray(np.stack([gx.ravel(), gy.ravel()], axis=1))


# --------------------------------------------------------------------- field
def _locations(spec: ConfigSpec, n: int) -> np.ndarray:
    r = rng(spec.cid, 0)   # spec is the generator's config (C4 -> C3)
    if spec.layout == "uniform":
        return r.uniform(0.0, 1.0, (n, 2))
    centres = rng(spec.cid, 8).uniform(0.1, 0.9, (8, 2))
    lab = r.integers(0, 8, n)
    X = centres[lab] + 0.05 * r.standard_normal((n, 2))
    return np.clip(X, 0.0, 1.0)


def _rss_dbm(Xm: np.ndarray, tx_m: np.ndarray, p_dbm: np.ndarray, f_hz: float,
             shadow: Optional[np.ndarray]) -> np.ndarray:
    """Log-distance path loss, exponent 3, d0 = 1 m, free-space PL at 1 m (R4)."""
    pl0 = 20.0 * math.log10(4.0 * math.pi * f_hz / C_LIGHT)
    dist = np.sqrt(((Xm[:, None, :] - tx_m[None, :, :]) ** 2).sum(-1))
    dist = np.maximum(dist, 1.0)
    rss = p_dbm[None, :] - pl0 - 30.0 * np.log10(dist)
    if shadow is not None:
        rss = rss + shadow
    return 10.0 * np.log10((10.0 ** (rss / 10.0)).sum(axis=1))


def make_problem(cid: int, n: Optional[int] = None, d: Optional[int] = None,
                 lam: Optional[float] = None, nrhs: Optional[int] = None,
                 grid: Optional[int] = None, tol: Optional[float] = None) -> Problem:
    """Config `cid` of BASELINE.json (1..5), optionally downscaled."""
    spec = CONFIGS[cid]
    n = spec.n if n is None else int(n)
    d = spec.d if d is None else int(d)
    lam = spec.lam if lam is None else float(lam)
    nrhs = spec.nrhs if nrhs is None else int(nrhs)
    g = spec.grid if grid is None else int(grid)
    tol = spec.tol if tol is None else float(tol)

    gid = 3 if cid == 4 else cid   # C4 reuses C3's sensors, Tx sites and embeddings (R5)
    X = _locations(CONFIGS[gid], n)
    Xq = grid_points(g)
    tx = rng(gid, 1).uniform(0.0, 1.0, (spec.n_tx, 2)) * 100.0
    Y = np.empty((n, nrhs), dtype=np.float64, order="F")
    T = np.empty((Xq.shape[0], nrhs), dtype=np.float64, order="F")
    for b in range(nrhs):
        if nrhs == 1:
            f = F_CARRIER
            p = rng(cid, 2).uniform(20.0, 30.0, spec.n_tx)
            sh = 6.0 * rng(cid, 3).standard_normal((n, spec.n_tx))
        else:  # C4: 64 bands, f_b = 3.5 GHz + (b - 31.5) * 5 MHz (reading R5)
            f = F_CARRIER + (b - (nrhs - 1) / 2.0) * 5e6
            rb = rng(cid, 16 + b)
            p = rb.uniform(20.0, 30.0, spec.n_tx)
            sh = 6.0 * rb.standard_normal((n, spec.n_tx))
        Y[:, b] = _rss_dbm(100.0 * X, tx, p, f, sh)
        T[:, b] = _rss_dbm(100.0 * Xq, tx, p, f, None)

    emb = make_embedding(gid, d)
    E = embed(emb, X)
    Eq = embed(emb, Xq)
    n_dirs = min(spec.n_dirs, n) if spec.n_dirs else 0
    if n != spec.n and spec.n_dirs:
        n_dirs = nr_schedule(n)
    return Problem(spec=spec, n=n, d=d, lam=lam, tol=tol, scale=1.0 / math.sqrt(d),
                   X=X, E=E, Y=Y, Xq=Xq, Eq=Eq, truth=T, n_dirs=n_dirs)


def make_paper_problem(n: int, grid: int = 45, d: int = 10, lam: float = 1e-2, tol: float = 1e-10,
                       noise_db: float = 1.5, n_tx: int = 3) -> Problem:
    """The paper's own regime (Table "Key simulation parameters";
    SURVEY §8(f) NEXT-4): n locations uniform on [0,100]^2 m, superposed
    transmitters with log-distance decay (R4 model, no shadowing) plus i.i.d.
    N(0, 1.5^2) dB measurement noise, d_e = 10 embeddings, G = exp(E E^T)
    (scale 1, as in the worked example), lambda = 1e-2, a 45 x 45 evaluation grid,
    PCG tolerance 1e-10.  Config id 0 seeds it (streams as in make_problem, noise
    on stream 3)."""
    X = rng(0, 0).uniform(0.0, 1.0, (n, 2))
    Xq = grid_points(grid)
    tx = rng(0, 1).uniform(0.0, 1.0, (n_tx, 2)) * 100.0
    p = rng(0, 2).uniform(20.0, 30.0, n_tx)
    clean = _rss_dbm(100.0 * X, tx, p, F_CARRIER, None)
    y = clean + noise_db * rng(0, 3).standard_normal(n)
    T = _rss_dbm(100.0 * Xq, tx, p, F_CARRIER, None)
    emb = make_embedding(0, d)
    spec = ConfigSpec(0, n, d, lam, tol, "uniform", n_tx, 1, grid, nr_schedule(n), "learned", "materialized", 1)
    return Problem(spec=spec, n=n, d=d, lam=lam, tol=tol, scale=1.0, X=X, E=embed(emb, X),
                   Y=np.asfortranarray(y[:, None]), Xq=Xq, Eq=embed(emb, Xq),
                   truth=np.asfortranarray(T[:, None]), n_dirs=nr_schedule(n))


def nr_schedule(n: int) -> int:
    """N_r = min(n, max(ceil(8 sqrt n), ceil(n/4))) -- SPEC.md l.241 reading of
    PAPER.md l.743 ("O(sqrt n) for small n and linearly for large n")."""
    return int(min(n, max(math.ceil(8.0 * math.sqrt(n)), math.ceil(n / 4.0))))


def make_directions(cid: int, n: int, n_dirs: int) -> np.ndarray:
    """z_k ~ N(0, I_n) (Eq. random_directions) as an n x N_r
    column-major array (stream 7).  Column k is independent of N_r."""
    Zt = rng(cid, 7).standard_normal((n_dirs, n))
    return Zt.T  # Fortran-ordered view: column k contiguous


def worked_example():
    """PAPER.md l.632-673 (Example, n = 3): printed inputs and outputs."""
    return dict(
        E=np.array([[0.241, 0.444], [-0.336, 0.112], [-0.220, 0.353]]),
        y=np.array([-66.14, -65.77, -77.30]),
        lam=0.1,
        G=np.array([[1.291, 0.969, 1.109], [0.969, 1.133, 1.120], [1.109, 1.120, 1.189]]),
        alpha=np.array([0.815, 5.438, -65.406]),
        e_star=np.array([0.051, 0.452]),
        cross=np.array([1.237, 1.034, 1.160]),
        r_hat=-69.2,
    )
