"""O4: ParaDiag-II for a nonlinear problem by simplified Newton (eq 1.4-1.5, P:l.196-227).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Problem (1D, homogeneous Dirichlet, reading x5):  u_t + K u + g(u) = 0,  K = -nu D2 + a D1 (as ADE1D),
g(u) = c3 u^3 + c1 u pointwise (Allen-Cahn type for c3 = 1, c1 = -1), i.e. M U' + f(U) = 0 with f(U) = K U + g(U).
theta-method all-at-once system (eq 1.4):
    (B1 (x) I) u + (B2 (x) I) F(u) = b,   F(u) = (f(U_1), ..., f(U_Nt)),
with the U_0 terms of the first block row moved to b:  b_1 = U_0/dt - (1 - theta) f(U_0) (reading c5 with the
nonlinear f).  Simplified Newton (eq 1.5):
    P_alpha(u^{k-1}) du = -((B1 (x) I) u^{k-1} + (B2 (x) I) F(u^{k-1}) - b),   u^k = u^{k-1} + du,
    P_alpha(u) = C1^(alpha) (x) I + C2^(alpha) (x) J(u),   J(u) = K + diag( (1/Nt) sum_n g'(U_n) )
(the first averaging named at P:l.214-216).  Every P_alpha^{-1} is the three steps of eq 1.3 with the shifted
systems lambda_1n I + lambda_2n J (tridiagonal, no longer Toeplitz: pivoted banded LU per frequency here).
Stop when ||b - (B1 u + B2 F(u))|| <= tol ||b||; iteration count = Newton corrections applied.
"""
from __future__ import annotations

import dataclasses

import numpy as np
import scipy.linalg
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import problems, spectral
from .solvers import Report


@dataclasses.dataclass(frozen=True)
class Reaction:
    c3: float = 1.0
    c1: float = -1.0

    def g(self, u):
        return self.c3 * u ** 3 + self.c1 * u

    def dg(self, u):
        return 3.0 * self.c3 * u ** 2 + self.c1


def _theta(cfg):
    return problems.theta_of(cfg.scheme)


def F(cfg, rx: Reaction, U: np.ndarray) -> np.ndarray:
    """f(U) = K U + g(U) for every block of U ([Nt][S] or [S])."""
    return problems.apply_K(cfg, U) + rx.g(U)


def rhs(cfg, rx: Reaction, u0: np.ndarray) -> np.ndarray:
    """b of eq 1.4 for f = 0 source: block 1 = U_0/dt - (1 - theta) f(U_0), others 0."""
    th = _theta(cfg)
    b = np.zeros((cfg.nt, cfg.S))
    b[0] = u0 / cfg.dt - (1.0 - th) * F(cfg, rx, u0)
    return b


def residual(cfg, rx: Reaction, b: np.ndarray, u: np.ndarray) -> np.ndarray:
    """r = b - ((B1 (x) I) u + (B2 (x) I) F(u)) with the lower-bidiagonal B1, B2 of eq 2.5b."""
    c1, c2 = problems.time_first_columns(cfg)
    return b - problems.apply_time(c1, u, None) - problems.apply_time(c2, F(cfg, rx, u), None)


def jac_avg(cfg, rx: Reaction, u: np.ndarray) -> np.ndarray:
    """diag of J(u) - K: the time average (1/Nt) sum_n g'(U_n) ([S])."""
    return rx.dg(u).mean(axis=0)


def apply_precond(cfg, r: np.ndarray, dbar: np.ndarray) -> np.ndarray:
    """z = P_alpha^{-1} r with J = K + diag(dbar): Steps (a), (b) (banded LU of lambda_1 I + lambda_2 J), (c)."""
    lam1, lam2 = spectral.spectra(cfg)
    S1 = spectral.step_a(cfg, r)
    K = problems.K_matrix(cfg)
    sub, dia, sup = K.diagonal(-1), K.diagonal(0) + dbar, K.diagonal(1)
    n = cfg.nx
    S2 = np.empty_like(S1)
    for k in range(cfg.nt):
        ab = np.zeros((3, n), dtype=np.complex128)
        ab[0, 1:] = lam2[k] * sup
        ab[1, :] = lam1[k] + lam2[k] * dia
        ab[2, :-1] = lam2[k] * sub
        S2[k] = scipy.linalg.solve_banded((1, 1), ab, S1[k])
    return spectral.step_c(cfg, S2)


def solve_newton(cfg, rx: Reaction, b, u0=None, tol=None, maxit=None):
    """Simplified Newton eq 1.5 with the ParaDiag-II preconditioner rebuilt from the current iterate."""
    tol = cfg.tol if tol is None else tol
    maxit = cfg.maxit if maxit is None else maxit
    u = np.zeros_like(b) if u0 is None else u0.copy()
    bn = np.linalg.norm(b)
    hist = []
    k = 0
    while True:
        r = residual(cfg, rx, b, u)
        rel = np.linalg.norm(r) / bn
        if k > 0:
            hist.append(rel)
        if rel <= tol or k >= maxit:
            return u, Report(k, rel <= tol, rel, hist)
        u = u + apply_precond(cfg, r, jac_avg(cfg, rx, u))
        k += 1


def march(cfg, rx: Reaction, u0: np.ndarray, newton_tol: float = 1e-14) -> np.ndarray:
    """Sequential theta-method: (U_n - U_{n-1})/dt + theta f(U_n) + (1-theta) f(U_{n-1}) = 0, each step solved by
    full Newton with a sparse LU of its exact Jacobian (the non-parallel reference, P:l.76-78)."""
    th, dt = _theta(cfg), cfg.dt
    K = problems.K_matrix(cfg)
    I = sp.identity(cfg.S, format="csr")
    out = np.zeros((cfg.nt, cfg.S))
    prev = u0.copy()
    for n in range(cfg.nt):
        rhs_n = prev / dt - (1.0 - th) * F(cfg, rx, prev)
        x = prev.copy()
        for _ in range(50):
            res = x / dt + th * F(cfg, rx, x) - rhs_n
            if np.linalg.norm(res) <= newton_tol * max(np.linalg.norm(rhs_n), 1.0):
                break
            Jn = (I / dt + th * (K + sp.diags(rx.dg(x)))).tocsc()
            x = x - spla.spsolve(Jn, res)
        out[n] = x
        prev = x
    return out
