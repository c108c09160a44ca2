"""Sequential time stepping — the classical non-parallel route (P:l.76-78) (oracle; test infrastructure).

The unique solution of A u = b (eq 1.1) is obtained by block forward substitution, one implicit
spatial solve per step (sparse LU factorised once):
  theta-method (eq 2.4 / 2.10 with alpha = 0): (I/dt + theta K) U_n = (I/dt - (1-theta) K) U_{n-1} + b_n
  leapfrog (eq 3.2b rows): (I/dt^2 + K/2) U_n = b_n + (2 U_{n-1} - U_{n-2})/dt^2 - K U_{n-2}/2
with U_0 = U_{-1} = 0 inside the all-at-once matrix (the initial data live in b).
``march`` is the physical stepping from (U_0, V_0, f), independent of ``problems.rhs``.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import problems
from workloads import BE, CN, LF


def _lu(M):
    return spla.splu(sp.csc_matrix(M))


def solve_all_at_once(cfg, b: np.ndarray) -> np.ndarray:
    """u = A^{-1} b by forward substitution over the time blocks."""
    K = problems.K_matrix(cfg)
    S, nt, dt = cfg.S, b.shape[0], cfg.dt
    I = sp.identity(S, format="csr")
    u = np.zeros_like(b)
    if cfg.scheme in (BE, CN):
        th = problems.theta_of(cfg.scheme)
        lu = _lu(I / dt + th * K)
        Rm = (I / dt - (1.0 - th) * K).tocsr()
        prev = np.zeros(S)
        for n in range(nt):
            prev = lu.solve(b[n] + Rm @ prev)
            u[n] = prev
        return u
    lu = _lu(I / dt ** 2 + 0.5 * K)
    a = np.zeros(S)   # U_{n-2}
    c = np.zeros(S)   # U_{n-1}
    for n in range(nt):
        new = lu.solve(b[n] + (2.0 * c - a) / dt ** 2 - 0.5 * (K @ a))
        u[n] = new
        a, c = c, new
    return u


def march(cfg, u0: np.ndarray, v0: np.ndarray | None = None, f: np.ndarray | None = None) -> np.ndarray:
    """Physical time stepping U_1..U_Nt from the initial data ([Nt][S]).

    theta-method: (U_n - U_{n-1})/dt + K(theta U_n + (1-theta) U_{n-1}) = theta f_n + (1-theta) f_{n-1}  (eq 2.4)
    leapfrog: (U_{n+1} - 2U_n + U_{n-1})/dt^2 + K (U_{n+1} + U_{n-1})/2 = f_n  (P:l.1199-1230),
              U_{-1} = U_1 - 2 dt V_0 (central-difference initial velocity, reading c4).
    """
    K = problems.K_matrix(cfg)
    S, nt, dt = cfg.S, cfg.nt, cfg.dt
    I = sp.identity(S, format="csr")
    fz = (lambda n: np.zeros(S)) if f is None else (lambda n: f[n])
    u = np.zeros((nt, S))
    if cfg.scheme in (BE, CN):
        th = problems.theta_of(cfg.scheme)
        lu = _lu(I / dt + th * K)
        Rm = (I / dt - (1.0 - th) * K).tocsr()
        prev = u0.copy()
        for n in range(1, nt + 1):
            prev = lu.solve(Rm @ prev + th * fz(n) + (1.0 - th) * fz(n - 1))
            u[n - 1] = prev
        return u
    v0 = np.zeros(S) if v0 is None else v0
    L = I / dt ** 2 + 0.5 * K
    lu = _lu(L)
    # scheme at n = 0 with U_{-1} = U_1 - 2 dt V_0, solved for U_1
    # (2U_1 - 2U_0 - 2dt V_0)/dt^2 + K(2U_1 - 2 dt V_0)/2 = f_0
    U1 = lu.solve(0.5 * fz(0) + u0 / dt ** 2 + v0 / dt + 0.5 * dt * (K @ v0))
    u[0] = U1
    a, c = u0.copy(), U1
    for n in range(1, nt):
        new = lu.solve(fz(n) + (2.0 * c - a) / dt ** 2 - 0.5 * (K @ a))
        u[n] = new
        a, c = c, new
    return u


def march_fourier(cfg, u0: np.ndarray, f: np.ndarray | None = None) -> np.ndarray:
    """The theta-method ``march`` for the 2D periodic operator (ADE2D), written in the eigenbasis of K.

    K = F2^{-1} diag(kappa) F2 with the 2D DFT F2 and the symbol kappa of reading c14 (spectral.symbol_2d,
    pinned against the sparse stencil), so each Fourier coefficient follows the scalar form of eq 2.4:
      (1/dt + theta kappa) u^_n = (1/dt - (1-theta) kappa) u^_{n-1} + theta f^_n + (1-theta) f^_{n-1}
    and U_n = F2^{-1} u^_n.  The same time stepping as ``march`` (pinned equal to it in
    tests/test_oracle_pins.py), with numpy.fft as the library primitive for F2 instead of a sparse LU solve per
    step, so it reaches config 4 (512^2 x 2048) in seconds.
    """
    from workloads import ADE2D
    from .spectral import symbol_2d
    if cfg.op != ADE2D or cfg.scheme not in (BE, CN):
        raise ValueError("march_fourier: 2D periodic theta-method only")
    n, nt, dt = cfg.nx, cfg.nt, cfg.dt
    th = problems.theta_of(cfg.scheme)
    kap = symbol_2d(cfg)                                   # [ky][kx], the layout of fft2 on [y][x]
    lhs = 1.0 / dt + th * kap
    rmul = (1.0 / dt - (1.0 - th) * kap) / lhs
    fh = (lambda k: 0.0) if f is None else (lambda k: np.fft.fft2(f[k].reshape(n, n)))
    prev = np.fft.fft2(u0.reshape(n, n))
    fprev = fh(0)
    u = np.empty((nt, n * n))
    for k in range(1, nt + 1):
        fk = fh(k)
        prev = rmul * prev + (th * fk + (1.0 - th) * fprev) / lhs
        fprev = fk
        u[k - 1] = np.fft.ifft2(prev).real.reshape(-1)
    return u
