"""Seeded synthetic workloads shared by the oracle tests, the GPU tests and bench.py.

This module holds the five BASELINE.json configurations and
the seeded generators of their *problem data*: grid coordinates, initial
fields, the sampled source term and random apply inputs.  It deliberately holds
none of the method's arithmetic: no spatial operator, no time-stepping matrix,
no right-hand-side assembly, no DFT, no solve.  Both the oracle (``oracle/``)
and the CUDA path (``paper_2005_09158_b200``) build everything else from these
arrays on their own.

Readings of the paper/BASELINE that fix the data:
  c8  T=1 for configs 3/4 (dt = 1/Nt).
  c9  "N(0,1e-3)" noise = standard deviation 1e-3, numpy PCG64 seeded.
  c10 Gaussian bump exp(-(x-c)^2 / (2*0.05^2)), c ~ U(0.3, 0.7).
  c11 config-1 source: sum_{k=1..8} a_k sin(k pi x) cos(t), a_k ~ N(0,1).
  c12 configs 3/4: sum_{0<|k|<=8} (a_k cos(k.x) + b_k sin(k.x)) / |k|^2.
  c13 1D Dirichlet grids hold interior nodes x_i=(i+1)h, h=1/(Nx+1);
      periodic grids have no duplicate endpoint, x_i = i h, h = 2 pi / N.
No public dataset is involved: the paper's workloads are analytic PDE data.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

# operator ids (mirror include/paradiag.h pd_operator)
ADE1D = "ade1d"      # u_t = nu u_xx - a u_x on (0,1), homogeneous Dirichlet
WAVE1D = "wave1d"    # u_tt = u_xx on (0,1), homogeneous Dirichlet
ADE2D = "ade2d"      # u_t = nu Lap u - a.grad u on [0,2pi)^2, periodic
WAVE2D = "wave2d"    # u_tt = Lap u + f on (0,1)^2, homogeneous Dirichlet (Table T4A, P:l.1309-1349)

# scheme ids (mirror pd_scheme)
BE, CN, LF = "be", "cn", "lf"


@dataclasses.dataclass(frozen=True)
class Config:
    """One all-at-once problem: grid, operator coefficients, time grid, alpha, solver."""
    name: str
    op: str
    nx: int               # 1D: interior nodes; 2D: N per dimension
    ny: int               # 1 for 1D; N for 2D
    nt: int
    T: float
    scheme: str
    alpha: float
    nu: float = 1.0
    ax: float = 0.0
    ay: float = 0.0
    solver: str = "stationary"   # "stationary" | "gmres"
    tol: float = 1e-10
    m: int = 20                  # GMRES restart length
    maxit: int = 100
    seed: int = 0
    source: str = "zero"         # "zero" | "sin8cos"
    init: str = "sin_noise"      # "sin_noise" | "bump" | "fourier8" | "exact_wave" | "gauss20"
    domain: float = 0.0          # 2D domain length; 0 = the default [0, 2pi) (configs 3-4)

    @property
    def dt(self) -> float:
        return self.T / self.nt

    @property
    def length(self) -> float:
        if self.op in (ADE1D, WAVE1D, WAVE2D):
            return 1.0
        return self.domain if self.domain > 0 else 2.0 * math.pi

    @property
    def h(self) -> float:
        if self.op in (ADE1D, WAVE1D, WAVE2D):
            return 1.0 / (self.nx + 1)
        return self.length / self.nx

    @property
    def S(self) -> int:
        """Spatial dofs per time level."""
        return self.nx * self.ny

    @property
    def D(self) -> int:
        """All-at-once dofs Nt*Nx (the metric's unit of work)."""
        return self.nt * self.S

    def scaled(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


# SURVEY.md §8(d) table; BASELINE.json "configs"
CONFIGS = [
    Config("cfg0", ADE1D, nx=63, ny=1, nt=32, T=1.0, scheme=BE, alpha=1e-2, nu=1e-2, ax=1.0,
           solver="stationary", tol=1e-10, seed=0, init="sin_noise"),
    Config("cfg1", ADE1D, nx=1023, ny=1, nt=1024, T=1.0, scheme=CN, alpha=1e-3, nu=1e-2, ax=1.0,
           solver="gmres", tol=1e-10, m=20, seed=1, init="sin_noise", source="sin8cos"),
    Config("cfg2", WAVE1D, nx=4095, ny=1, nt=4096, T=2.0, scheme=LF, alpha=1e-2,
           solver="stationary", tol=1e-9, seed=2, init="bump"),
    Config("cfg3", ADE2D, nx=256, ny=256, nt=256, T=1.0, scheme=BE, alpha=1e-3, nu=1e-2, ax=1.0, ay=0.5,
           solver="gmres", tol=1e-10, m=20, seed=3, init="fourier8"),
    Config("cfg4", ADE2D, nx=512, ny=512, nt=2048, T=1.0, scheme=CN, alpha=1e-4, nu=1e-2, ax=1.0, ay=0.5,
           solver="gmres", tol=1e-9, m=10, seed=4, init="fourier8"),
]
BY_NAME = {c.name: c for c in CONFIGS}

# Table ctp-01 (P:l.954-978): eq 2.14 on Omega = (0,1)^2 periodic, u_t - nu Lap u + grad u = 0
# (advection (1, 1), reading x1), dx = dy = dt = 1/128, Nt = 512, alpha = 0.02, tol = 1e-6, stationary eq 2.10.
CTP01_NUS = (1.0, 1e-1, 1e-2, 1e-3, 1e-4, 1e-5)
CTP01_COUNTS = {BE: (4, 4, 5, 5, 5, 5), CN: (4, 5, 5, 5, 5, 5)}   # printed iteration numbers (B-E, TR)


def ctp01_config(scheme: str, nu: float, **kw) -> Config:
    c = Config("ctp01", ADE2D, nx=128, ny=128, nt=512, T=4.0, scheme=scheme, alpha=0.02, nu=nu, ax=1.0, ay=1.0,
               solver="stationary", tol=1e-6, seed=0, init="gauss20", domain=1.0)
    return c.scaled(**kw) if kw else c


def grid(cfg: Config):
    """Node coordinates (reading c13). 1D: x[Nx]; 2D: (X, Y) each [N][N], x fastest."""
    if cfg.op in (ADE1D, WAVE1D):
        return (np.arange(cfg.nx, dtype=np.float64) + 1.0) * cfg.h
    if cfg.op == WAVE2D:  # interior nodes of (0,1)^2
        x = (np.arange(cfg.nx, dtype=np.float64) + 1.0) * cfg.h
        Y, X = np.meshgrid(x[: cfg.ny], x, indexing="ij")
        return X, Y
    x = np.arange(cfg.nx, dtype=np.float64) * cfg.h
    y = np.arange(cfg.ny, dtype=np.float64) * (cfg.length / cfg.ny)
    Y, X = np.meshgrid(y, x, indexing="ij")
    return X, Y


def initial_u0(cfg: Config) -> np.ndarray:
    """U_0 on the grid, flattened [S] (x fastest)."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    if cfg.init == "sin_noise":            # configs 0, 1 (reading c9)
        x = grid(cfg)
        return np.sin(math.pi * x) + 1e-3 * rng.standard_normal(cfg.nx)
    if cfg.init == "bump":                 # config 2 (reading c10)
        x = grid(cfg)
        c = rng.uniform(0.3, 0.7)
        return np.exp(-((x - c) ** 2) / (2.0 * 0.05 ** 2))
    if cfg.init == "exact_wave2d":         # Table T4A: u0 = sin(pi x) sin(pi y) (P:l.1311-1313)
        X, Y = grid(cfg)
        return (np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)
    if cfg.init == "gauss20":              # Table ctp-01 (P:l.910-912): exp(-20((x-1/2)^2 + (y-1/2)^2))
        X, Y = grid(cfg)
        return np.exp(-20.0 * ((X - 0.5) ** 2 + (Y - 0.5) ** 2)).reshape(-1)
    if cfg.init == "fourier8":             # configs 3, 4 (reading c12)
        X, Y = grid(cfg)
        u = np.zeros_like(X)
        for kx in range(-8, 9):
            for ky in range(-8, 9):
                k2 = kx * kx + ky * ky
                if k2 == 0 or k2 > 64:
                    continue
                a, b = rng.standard_normal(2)
                ph = kx * X + ky * Y
                u += (a * np.cos(ph) + b * np.sin(ph)) / k2
        return u.reshape(-1)
    if cfg.init == "exact_wave":           # u = sin(pi x) e^t (1D analogue of P:l.1311-1314)
        x = grid(cfg)
        return np.sin(math.pi * x)
    raise ValueError(cfg.init)


def initial_v0(cfg: Config) -> np.ndarray:
    """u_t(0) for the wave problems ([S]); zeros elsewhere."""
    if cfg.init == "exact_wave":
        return np.sin(math.pi * grid(cfg))
    if cfg.init == "exact_wave2d":         # u_1 = u_t(0) = sin(pi x) sin(pi y)
        X, Y = grid(cfg)
        return (np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)
    return np.zeros(cfg.S)


def source_samples(cfg: Config):
    """f(x, t_n) sampled at t_n = n dt, n = 0..Nt, shape [Nt+1][S]; None when f = 0."""
    if cfg.source == "zero":
        return None
    t = np.arange(cfg.nt + 1, dtype=np.float64) * cfg.dt
    if cfg.source == "sin8cos":            # config 1 (reading c11)
        rng = np.random.Generator(np.random.PCG64(1000 + cfg.seed))
        a = rng.standard_normal(8)
        x = grid(cfg)
        shape = sum(a[k - 1] * np.sin(k * math.pi * x) for k in range(1, 9))
        return np.cos(t)[:, None] * shape[None, :]
    if cfg.source == "exact_wave2d":       # f = (1 + 2 pi^2) sin(pi x) sin(pi y) e^t (P:l.1311-1313)
        X, Y = grid(cfg)
        return np.exp(t)[:, None] * ((1.0 + 2.0 * math.pi ** 2) * np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)[None, :]
    if cfg.source == "exact_wave":         # f = (1 + pi^2) sin(pi x) e^t for u = sin(pi x) e^t
        x = grid(cfg)
        return np.exp(t)[:, None] * ((1.0 + math.pi ** 2) * np.sin(math.pi * x))[None, :]
    raise ValueError(cfg.source)


def random_vector(cfg: Config, seed: int | None = None) -> np.ndarray:
    """r ~ N(0,1) iid, shape [Nt][S] (seed 100 + cfg index)."""
    if seed is None:
        seed = 100 + (CONFIGS.index(BY_NAME[cfg.name]) if cfg.name in BY_NAME else 0)
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((cfg.nt, cfg.S))


def exact_wave_solution(cfg: Config) -> np.ndarray:
    """sin(pi x) e^{t_n} (1D) / sin(pi x) sin(pi y) e^{t_n} (2D, Table T4A), n = 1..Nt ([Nt][S])."""
    t = np.arange(1, cfg.nt + 1, dtype=np.float64) * cfg.dt
    if cfg.op == WAVE2D:
        X, Y = grid(cfg)
        return np.exp(t)[:, None] * (np.sin(math.pi * X) * np.sin(math.pi * Y)).reshape(-1)[None, :]
    x = grid(cfg)
    return np.exp(t)[:, None] * np.sin(math.pi * x)[None, :]


# Table T4A (P:l.1309-1349): u_tt = Lap u + f on (0,1)^2, T = 2, exact u = sin(pi x) sin(pi y) e^t,
# implicit leapfrog (eq 3.2b), GMRES, zero initial guess, tol 1e-10.  Mesh label (Nx, Nx, Nt) read as h = 1/Nx
# (Nx - 1 interior nodes per direction) and Nt - 1 time steps (the label counts the time points incl. t = 0;
# reading x3, pinned by the printed errors).
T4A_LABELS = (32, 64, 128, 256)
T4A_ERRORS = (7.17e-3, 1.86e-3, 4.74e-4, 1.20e-4)          # alpha = 1 and alpha = 0.1 columns
T4A_ITERS = {0.1: (3, 3, 3, 3), 1.0: (3, 7, 37, None)}      # None: "> 50"


def t4a_config(label: int, alpha: float = 0.1, **kw) -> Config:
    c = Config(f"t4a_{label}", WAVE2D, nx=label - 1, ny=label - 1, nt=label, T=2.0, scheme=LF, alpha=alpha,
               nu=1.0, solver="gmres", tol=1e-10, m=30, maxit=50, seed=0, source="exact_wave2d", init="exact_wave2d")
    return c.scaled(**kw) if kw else c


# Nonlinear ParaDiag-II by simplified Newton (eq 1.4-1.5, P:l.196-227): u_t + K u + g(u) = 0 on
# (0,1), Dirichlet, K as config 1 (nu = 1e-2, a = 1), g(u) = c3 u^3 + c1 u (Allen-Cahn: c3 = 1, c1 = -1, reading
# x5), u0 as config 1, f = 0, Crank-Nicolson, alpha = 1e-2, tol 1e-10.
NL_REACTION = (1.0, -1.0)


def nl_config(nx: int = 1023, nt: int = 1024, scheme: str = CN, **kw) -> Config:
    c = Config("nl1", ADE1D, nx=nx, ny=1, nt=nt, T=1.0, scheme=scheme, alpha=1e-2, nu=1e-2, ax=1.0,
               solver="newton", tol=1e-10, maxit=40, seed=1, init="sin_noise")
    return c.scaled(**kw) if kw else c
