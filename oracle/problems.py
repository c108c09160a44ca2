"""All-at-once systems of the paper, built from their plain definitions (oracle; test infrastructure).

A = B1 (x) M + B2 (x) K            (P:l.80-84, eq 1.1), M = I for finite differences (P:l.74-76)
P_alpha = C1 (x) M + C2 (x) K      (P:l.114-116, eq 1.2)
C_j = alpha-circulant built from the first column of B_j:
      C[i, j] = c[i-j] for i >= j, alpha * c[i-j+Nt] for i < j
      which reproduces the corner entries printed in eq 2.11b (P:l.789-801) and eq 3.4 (P:l.1262-1275).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp

from workloads import ADE1D, ADE2D, BE, CN, LF, WAVE1D, WAVE2D


def theta_of(scheme: str) -> float:
    """theta-method weight: BE theta=1, CN/TR theta=1/2 (P:l.296-302, eq 2.4)."""
    return {BE: 1.0, CN: 0.5}[scheme]


# ----------------------------------------------------------------------------------------
# spatial operator K (M = I)
# ----------------------------------------------------------------------------------------
def _periodic_1d(n: int, h: float):
    """Periodic 1D negative second difference and centred first difference (eq 2.2b, P:l.259-272)."""
    e = np.ones(n)
    lap = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1], shape=(n, n), format="lil")
    lap[0, n - 1] = -1.0
    lap[n - 1, 0] = -1.0
    d1 = sp.diags([-e[:-1], e[:-1]], [-1, 1], shape=(n, n), format="lil")
    d1[0, n - 1] = -1.0
    d1[n - 1, 0] = 1.0
    return lap.tocsr() / h ** 2, d1.tocsr() / (2.0 * h)


def K_matrix(cfg) -> sp.csr_matrix:
    """Spatial operator K of M U' + K U = f (P:l.70-76).

    ADE1D : K = -nu D2 + a D1 (centred, homogeneous Dirichlet, interior nodes, reading c13)
    WAVE1D: K = A = -D2 (negative Laplacian, P:l.1208-1211)
    ADE2D : K = -nu Lap_h + ax Dx + ay Dy, 5-point Laplacian, periodic (P:l.908-918, reading c14);
            unknown index s = y*N + x (x fastest).
    WAVE2D: K = -Lap_h, 5-point, homogeneous Dirichlet on (0,1)^2, interior nodes (Table T4A, P:l.1309-1313).
    """
    if cfg.op in (ADE1D, WAVE1D):
        n, h = cfg.nx, cfg.h
        if cfg.op == ADE1D:
            nu, a = cfg.nu, cfg.ax
        else:
            nu, a = 1.0, 0.0
        sub = -nu / h ** 2 - a / (2 * h)
        dia = 2 * nu / h ** 2
        sup = -nu / h ** 2 + a / (2 * h)
        e = np.ones(n)
        return sp.diags([sub * e[:-1], dia * e, sup * e[:-1]], [-1, 0, 1], shape=(n, n), format="csr")
    if cfg.op == ADE2D:
        n = cfg.nx
        assert cfg.ny == n
        h = cfg.h  # domain length / N: [0, 2pi) for configs 3-4, (0, 1) for Table ctp-01 (P:l.908-912)
        lap, d1 = _periodic_1d(n, h)
        eye = sp.identity(n, format="csr")
        return (cfg.nu * (sp.kron(eye, lap) + sp.kron(lap, eye))
                + cfg.ax * sp.kron(eye, d1) + cfg.ay * sp.kron(d1, eye)).tocsr()
    if cfg.op == WAVE2D:
        n, h = cfg.nx, cfg.h
        assert cfg.ny == n
        e = np.ones(n)
        d2 = sp.diags([-e[:-1], 2.0 * e, -e[:-1]], [-1, 0, 1], shape=(n, n), format="csr") / h ** 2
        eye = sp.identity(n, format="csr")
        return (sp.kron(eye, d2) + sp.kron(d2, eye)).tocsr()
    raise ValueError(cfg.op)


def apply_K(cfg, U: np.ndarray) -> np.ndarray:
    """K applied to every time block of U [Nt][S] (or a single block [S]).

    Extended-precision U (np.longdouble; scipy.sparse has no such dtype) takes the row sums of the same CSR
    entries in U's precision: (K U)_i = sum_j K_ij U_j."""
    K = K_matrix(cfg)
    if U.dtype == np.longdouble:
        Ut = U.reshape(-1, K.shape[0]).T                                   # [S][blocks]
        prod = K.data.astype(np.longdouble)[:, None] * Ut[K.indices]      # one row per stored entry
        out = np.add.reduceat(prod, K.indptr[:-1], axis=0).T              # every row of K has entries
        return np.ascontiguousarray(out).reshape(U.shape)
    if U.ndim == 1:
        return K @ U
    return np.ascontiguousarray((K @ U.T).T)


# ----------------------------------------------------------------------------------------
# time matrices
# ----------------------------------------------------------------------------------------
def time_first_columns(cfg, nt: int | None = None):
    """First columns of the lower-triangular Toeplitz B1, B2 (length Nt).

    theta-method (eq 2.5b with uniform dt, P:l.309-319):  B1 = (1/dt) [1; -1, 1],  B2 = [theta; 1-theta, theta]
    implicit leapfrog (eq 3.2b, P:l.1214-1227):           B1 = (1/dt^2) [1; -2, 1; 1, -2, 1],  B2 = (1/2) [1; 0, 1; 1, 0, 1]
    """
    nt = cfg.nt if nt is None else nt
    dt = cfg.dt
    c1 = np.zeros(nt)
    c2 = np.zeros(nt)
    if cfg.scheme in (BE, CN):
        th = theta_of(cfg.scheme)
        c1[0] = 1.0 / dt
        c2[0] = th
        if nt > 1:
            c1[1] = -1.0 / dt
            c2[1] = 1.0 - th
    elif cfg.scheme == LF:
        c1[0] = 1.0 / dt ** 2
        c2[0] = 0.5
        if nt > 1:
            c1[1] = -2.0 / dt ** 2
        if nt > 2:
            c1[2] = 1.0 / dt ** 2
            c2[2] = 0.5
    else:
        raise ValueError(cfg.scheme)
    return c1, c2


def toeplitz_lower(c: np.ndarray) -> np.ndarray:
    """Dense lower-triangular Toeplitz matrix with first column c."""
    n = len(c)
    B = np.zeros((n, n))
    for i in range(n):
        for j in range(i + 1):
            B[i, j] = c[i - j]
    return B


def alpha_circulant(c: np.ndarray, alpha: float) -> np.ndarray:
    """Dense Strang-type alpha-circulant with first column c (P:l.112-119; corners of eq 2.11b / 3.4)."""
    n = len(c)
    C = np.zeros((n, n))
    for i in range(n):
        for j in range(n):
            C[i, j] = c[i - j] if i >= j else alpha * c[i - j + n]
    return C


def apply_time(c: np.ndarray, U: np.ndarray, alpha: float | None) -> np.ndarray:
    """(C (x) I) U for the Toeplitz (alpha=None) or alpha-circulant matrix with first column c.

    Plain definition: (C U)_n = sum_k c_k U_{n-k}, where U_{n-k} with n-k<0 is
    dropped (Toeplitz) or replaced by alpha*U_{n-k+Nt} (alpha-circulant).
    """
    nt = U.shape[0]
    out = np.zeros_like(U)
    for k in np.nonzero(c)[0]:
        out[k:] += c[k] * U[: nt - k]
        if alpha is not None and k > 0:
            out[:k] += alpha * c[k] * U[nt - k:]
    return out


def matvec_A(cfg, u: np.ndarray) -> np.ndarray:
    """A u with A = B1 (x) I + B2 (x) K (eq 1.1), u as [Nt][S]."""
    c1, c2 = time_first_columns(cfg, u.shape[0])
    return apply_time(c1, u, None) + apply_K(cfg, apply_time(c2, u, None))


def matvec_P(cfg, u: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """P_alpha u with P_alpha = C1 (x) I + C2 (x) K (eq 1.2), u as [Nt][S]."""
    alpha = cfg.alpha if alpha is None else alpha
    c1, c2 = time_first_columns(cfg, u.shape[0])
    return apply_time(c1, u, alpha) + apply_K(cfg, apply_time(c2, u, alpha))


# ----------------------------------------------------------------------------------------
# right-hand side b of A u = b
# ----------------------------------------------------------------------------------------
def rhs(cfg, u0: np.ndarray, v0: np.ndarray | None = None, f: np.ndarray | None = None) -> np.ndarray:
    """All-at-once right-hand side b ([Nt][S]).

    theta-method (P:l.321-323; reading c5 for the source):
        b_1 = theta f_1 + (1-theta) f_0 + (I/dt - (1-theta) K) U_0,  b_n = theta f_n + (1-theta) f_{n-1}
    implicit leapfrog (reading c4: central-difference initial velocity, halved first row):
        b_1 = f_0/2 + U_0/dt^2 + V_0/dt + (dt/2) K V_0
        b_2 = f_1 - U_0/dt^2 - K U_0 / 2
        b_n = f_{n-1}, n >= 3
    f is sampled at t_n = n dt, n = 0..Nt ([Nt+1][S]) or None for f = 0.
    """
    nt, S, dt = cfg.nt, cfg.S, cfg.dt
    b = np.zeros((nt, S))
    if cfg.scheme in (BE, CN):
        th = theta_of(cfg.scheme)
        if f is not None:
            b += th * f[1:] + (1.0 - th) * f[:-1]
        b[0] += u0 / dt - (1.0 - th) * apply_K(cfg, u0)
    elif cfg.scheme == LF:
        v0 = np.zeros(S) if v0 is None else v0
        if f is not None:
            b[0] += 0.5 * f[0]
            b[1:] += f[1:nt]
        b[0] += u0 / dt ** 2 + v0 / dt + 0.5 * dt * apply_K(cfg, v0)
        if nt > 1:
            b[1] += -u0 / dt ** 2 - 0.5 * apply_K(cfg, u0)
    else:
        raise ValueError(cfg.scheme)
    return b
