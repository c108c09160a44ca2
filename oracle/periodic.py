"""O2: P_alpha^{-1} r by alpha-periodic time stepping — no time DFT at all (oracle; test infrastructure).

P_alpha z = r is the all-at-once form of the WR iteration's head-tail condition (eq 2.9-2.11a,
P:l.757-801): time stepping of the same scheme with the initial data replaced by alpha times the
final data,
  theta-method: z_0 := alpha z_Nt                      (corner entries of eq 2.11b)
  leapfrog    : (z_{-1}, z_0) := alpha (z_{Nt-1}, z_Nt) (corner entries of eq 3.4)
Linear in the head-tail state w: step from zero data to get y, solve (I - alpha G^Nt) w = y_Nt with
the one-step propagator G (dense, repeated squaring), then re-step from alpha w.  This pins Gamma,
the DFT sign and the normalisation used by O1 independently of any Fourier matrix in time.
Two variants: dense propagator in the nodal basis (any operator, Nx up to ~1e3), and a modal version
for operators with a known orthogonal/unitary eigenbasis (WAVE1D: DST-I; ADE2D: 2D DFT).
"""
from __future__ import annotations

import math

import numpy as np

from . import problems
from workloads import ADE1D, ADE2D, BE, CN, LF, WAVE1D, WAVE2D


def _matpow(G: np.ndarray, n: int) -> np.ndarray:
    R = np.eye(G.shape[0], dtype=G.dtype)
    P = G.copy()
    while n:
        if n & 1:
            R = R @ P
        n >>= 1
        if n:
            P = P @ P
    return R


def _theta_dense(cfg, r, alpha, K):
    dt, nt = cfg.dt, r.shape[0]
    th = problems.theta_of(cfg.scheme)
    n = K.shape[0]
    I = np.eye(n, dtype=K.dtype)
    L = I / dt + th * K
    Rm = I / dt - (1.0 - th) * K
    Linv = np.linalg.inv(L)
    G = Linv @ Rm

    def sweep(z0):
        z = np.empty((nt, n), dtype=np.result_type(r, K))
        prev = z0
        for k in range(nt):
            prev = Linv @ (Rm @ prev + r[k])
            z[k] = prev
        return z

    y = sweep(np.zeros(n, dtype=np.result_type(r, K)))
    w = np.linalg.solve(I - alpha * _matpow(G, nt), y[-1])
    return sweep(alpha * w)


def _lf_dense(cfg, r, alpha, K):
    dt, nt = cfg.dt, r.shape[0]
    n = K.shape[0]
    I = np.eye(n, dtype=K.dtype)
    Linv = np.linalg.inv(I / dt ** 2 + 0.5 * K)
    # state (z_{k-1}, z_k) -> (z_k, z_{k+1}):  z_{k+1} = Linv (r + (2 z_k - z_{k-1})/dt^2 - K z_{k-1}/2)
    G = np.zeros((2 * n, 2 * n), dtype=K.dtype)
    G[:n, n:] = I
    G[n:, :n] = Linv @ (-I / dt ** 2 - 0.5 * K)
    G[n:, n:] = Linv @ (2.0 * I / dt ** 2)

    def sweep(zm1, z0):
        z = np.empty((nt, n), dtype=np.result_type(r, K))
        a, b = zm1, z0
        for k in range(nt):
            c = Linv @ (r[k] + (2.0 * b - a) / dt ** 2 - 0.5 * (K @ a))
            z[k] = c
            a, b = b, c
        return z

    zero = np.zeros(n, dtype=np.result_type(r, K))
    y = sweep(zero, zero)
    w = np.linalg.solve(np.eye(2 * n) - alpha * _matpow(G, nt), np.concatenate([y[-2], y[-1]]))
    return sweep(alpha * w[:n], alpha * w[n:])


def apply_precond_dense(cfg, r: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """z = P_alpha^{-1} r by alpha-periodic stepping with the dense nodal propagator."""
    alpha = cfg.alpha if alpha is None else alpha
    K = problems.K_matrix(cfg).toarray()
    if cfg.scheme in (BE, CN):
        return _theta_dense(cfg, r, alpha, K)
    return _lf_dense(cfg, r, alpha, K)


def apply_precond_modal(cfg, r: np.ndarray, alpha: float | None = None, precision=np.float64) -> np.ndarray:
    """Same as apply_precond_dense, in the eigenbasis of K (scalar recurrences per mode).

    WAVE1D: K = Q diag(mu) Q^T with the DST-I basis Q_{jk} = sqrt(2/(N+1)) sin(pi j k/(N+1)),
            mu_k = (4/h^2) sin^2(pi k / (2(N+1)))  (textbook eigenpairs of the Dirichlet -D2).
    ADE2D : K = F^{-1} diag(kappa) F with the 2D DFT (symbol: reading c14).
    precision: np.float64, or np.longdouble (WAVE1D / WAVE2D only) for the extended-precision references of
    readings t1 and x4 (the same steps in x87 80-bit arithmetic; the 2x2 head-tail systems by Cramer's rule).
    """
    alpha = cfg.alpha if alpha is None else alpha
    nt, dt = r.shape[0], cfg.dt
    ext = np.dtype(precision) != np.float64
    cdt = np.result_type(precision, np.complex64)
    if ext and cfg.op not in (WAVE1D, WAVE2D):
        raise ValueError("extended precision: WAVE1D / WAVE2D only")
    pi = 4 * np.arctan(np.asarray(1, dtype=precision)) if ext else math.pi
    if ext:
        r = np.asarray(r, dtype=precision)
        dt = precision(1) * cfg.T / nt
    if cfg.op == WAVE1D:
        n, h = cfg.nx, cfg.h
        j = np.arange(1, n + 1, dtype=precision)
        Q = np.sqrt(precision(2) / (n + 1)) * np.sin(pi * np.outer(j, j) / (n + 1))
        mu = (4 / precision(h) ** 2) * np.sin(pi * j / (2 * (n + 1))) ** 2
        rh = r @ Q                      # modal coefficients (Q symmetric orthogonal)
        to_nodal = lambda zh: zh @ Q
    elif cfg.op == ADE2D:
        from .spectral import dft_matrix, symbol_2d
        n = cfg.nx
        Fn, Fi = dft_matrix(n, -1), dft_matrix(n, +1)
        mu = symbol_2d(cfg).reshape(-1)
        rh = (Fn @ r.reshape(nt, n, n) @ Fn.T).reshape(nt, n * n)
        to_nodal = lambda zh: ((Fi @ zh.reshape(nt, n, n) @ Fi.T) / (n * n)).real.reshape(nt, n * n)
    elif cfg.op == WAVE2D:  # tensor DST-I basis, mu_{kl} = mu_k + mu_l
        n, h = cfg.nx, cfg.h
        j = np.arange(1, n + 1, dtype=precision)
        Q = np.sqrt(precision(2) / (n + 1)) * np.sin(pi * np.outer(j, j) / (n + 1))
        m1 = (4 / precision(h) ** 2) * np.sin(pi * j / (2 * (n + 1))) ** 2
        mu = (m1[:, None] + m1[None, :]).reshape(-1)
        rh = (Q @ r.reshape(nt, n, n) @ Q).reshape(nt, n * n)
        to_nodal = lambda zh: (Q @ zh.reshape(nt, n, n) @ Q).reshape(nt, n * n)
    else:
        raise ValueError("modal O2 needs a known eigenbasis (WAVE1D, ADE2D or WAVE2D)")

    if cfg.scheme in (BE, CN):
        th = problems.theta_of(cfg.scheme)
        l = 1.0 / dt + th * mu
        g = (1.0 / dt - (1.0 - th) * mu) / l

        def sweep(z0):
            z = np.empty((nt, mu.size), dtype=cdt)
            prev = z0
            for k in range(nt):
                prev = g * prev + rh[k] / l
                z[k] = prev
            return z

        y = sweep(np.zeros(mu.size, dtype=cdt))
        w = y[-1] / (1.0 - alpha * g ** nt)
        zh = sweep(alpha * w)
    else:
        l = 1.0 / dt ** 2 + 0.5 * mu
        c_a = (-1.0 / dt ** 2 - 0.5 * mu) / l   # coefficient of z_{k-1}
        c_b = (2.0 / dt ** 2) / l                # coefficient of z_k

        def sweep(zm1, z0):
            z = np.empty((nt, mu.size), dtype=cdt)
            a, b = zm1, z0
            for k in range(nt):
                c = c_a * a + c_b * b + rh[k] / l
                z[k] = c
                a, b = b, c
            return z

        zero = np.zeros(mu.size, dtype=cdt)
        y = sweep(zero, zero)
        # per-mode 2x2 propagator G = [[0, 1], [c_a, c_b]] raised to Nt
        G = np.zeros((mu.size, 2, 2), dtype=cdt)
        G[:, 0, 1] = 1.0
        G[:, 1, 0] = c_a
        G[:, 1, 1] = c_b
        Gn = np.broadcast_to(np.eye(2, dtype=cdt), G.shape).copy()
        P, e = G.copy(), nt
        while e:
            if e & 1:
                Gn = Gn @ P
            e >>= 1
            if e:
                P = P @ P
        Mtx = np.broadcast_to(np.eye(2), G.shape) - alpha * Gn
        rhs = np.stack([y[-2], y[-1]], axis=-1)[..., None]
        if ext:  # LAPACK has no extended precision: Cramer's rule on the 2x2 systems
            det = Mtx[:, 0, 0] * Mtx[:, 1, 1] - Mtx[:, 0, 1] * Mtx[:, 1, 0]
            w = np.stack([(Mtx[:, 1, 1] * y[-2] - Mtx[:, 0, 1] * y[-1]) / det,
                          (Mtx[:, 0, 0] * y[-1] - Mtx[:, 1, 0] * y[-2]) / det], axis=-1)
        else:
            w = np.linalg.solve(Mtx, rhs)[..., 0]
        zh = sweep(alpha * w[:, 0], alpha * w[:, 1])
    z = to_nodal(zh)
    return np.real(z) if np.iscomplexobj(z) else z
