"""Residual, stationary ParaDiag-II iteration and right-preconditioned GMRES(m) (oracle; test infrastructure).

Stopping rule (reading c6): both solvers stop when ||b - A u^k||_2 <= tol ||b||_2.
Iteration count = number of P_alpha^{-1} applications inside the loop (the GMRES final-assembly
apply is not counted).
"""
from __future__ import annotations

import dataclasses

import numpy as np

from . import problems, spectral


@dataclasses.dataclass
class Report:
    iterations: int
    converged: bool
    rel_residual: float                 # true ||b - A u|| / ||b|| at exit
    history: list                       # per-iteration relative residual (true for stationary; Arnoldi estimate for GMRES)


def residual(cfg, b: np.ndarray, u: np.ndarray) -> np.ndarray:
    """r = b - A u (eq 5.1, P:l.1563-1565), A of eq 1.1."""
    return b - problems.matvec_A(cfg, u)


def solve_stationary(cfg, b, u0=None, tol=None, maxit=None, apply=None):
    """Stationary iteration in residual-correction form, eq 5.1 (P:l.1563-1565):
         r^k = b - A u^k;  P_alpha du^k = r^k;  u^{k+1} = u^k + du^k
    equivalent to P_alpha u^k = (P_alpha - A) u^{k-1} + b (P:l.120-124).
    """
    tol = cfg.tol if tol is None else tol
    maxit = cfg.maxit if maxit is None else maxit
    apply = apply or (lambda r: spectral.apply_precond(cfg, r))
    u = np.zeros_like(b) if u0 is None else u0.copy()
    bnorm = np.linalg.norm(b)
    hist = []
    k = 0
    while True:
        r = residual(cfg, b, u)
        rel = np.linalg.norm(r) / bnorm
        if k > 0:
            hist.append(rel)
        if rel <= tol:
            return u, Report(k, True, rel, hist)
        if k >= maxit:
            return u, Report(k, False, rel, hist)
        u = u + apply(r)
        k += 1


def solve_gmres(cfg, b, u0=None, tol=None, m=None, maxit=None, apply=None):
    """Right-preconditioned restarted GMRES(m) on A P_alpha^{-1} y = b, u = u0 + P_alpha^{-1} y
    (Krylov use of P_alpha, P:l.125-132; right preconditioning per north_star, reading c7).

    Arnoldi with modified Gram-Schmidt, Givens rotations, stop on the Arnoldi residual estimate
    |g_{j+1}| <= tol ||b||; at convergence or restart the true residual is recomputed and the
    iteration continues (restart) if it is still above tol.
    """
    tol = cfg.tol if tol is None else tol
    m = cfg.m if m is None else m
    maxit = cfg.maxit if maxit is None else maxit
    apply = apply or (lambda r: spectral.apply_precond(cfg, r))
    shape = b.shape
    u = np.zeros_like(b) if u0 is None else u0.copy()
    bnorm = np.linalg.norm(b)
    hist = []
    its = 0
    r = residual(cfg, b, u)
    beta = np.linalg.norm(r)
    if beta <= tol * bnorm:
        return u, Report(0, True, beta / bnorm, hist)
    while True:
        V = [r.reshape(-1) / beta]
        H = np.zeros((m + 1, m), dtype=b.dtype)   # b.dtype: float64, or np.longdouble for reading x4's reference
        cs, sn = np.zeros(m, dtype=b.dtype), np.zeros(m, dtype=b.dtype)
        g = np.zeros(m + 1, dtype=b.dtype)
        g[0] = beta
        k = 0
        breakdown = False
        for j in range(m):
            z = apply(V[j].reshape(shape))
            its += 1
            w = problems.matvec_A(cfg, z).reshape(-1)
            for i in range(j + 1):
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            hnext = np.linalg.norm(w)
            if abs(g[j + 1]) <= tol * bnorm or its >= maxit:
                break
            if hnext == 0.0:
                breakdown = True
                break
            V.append(w / hnext)
        y = np.zeros(k, dtype=b.dtype)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        comb = sum(y[i] * V[i] for i in range(k))
        u = u + apply(comb.reshape(shape))
        r = residual(cfg, b, u)
        beta = np.linalg.norm(r)
        if beta <= tol * bnorm:
            return u, Report(its, True, beta / bnorm, hist)
        if its >= maxit or breakdown:
            return u, Report(its, False, beta / bnorm, hist)
