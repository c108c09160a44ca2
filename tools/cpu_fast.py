"""Fast CPU reference of the ParaDiag-II solve (the fair CPU comparison for bench.py).

Not the oracle: the same method written for speed on the host cores -- Step (a) / (c) as real FFTs along time
(scipy.fft.rfft / irfft, workers = all cores) with Gamma fused, Step (b) as a Thomas sweep vectorised over the
frequencies (1D; no pivoting: the configs' shifted systems are diagonally dominant or, for the wave family,
stable without pivoting, SURVEY [V3]) or a 2D FFT -> divide by lambda1 + lambda2 kappa -> inverse 2D FFT per
frequency slab (2D periodic), the residual by array slicing, and the same solvers and stopping rule as the GPU
(stationary eq 5.1; right-preconditioned GMRES(m), MGS).  Also the sequential time stepping of the classical route
(P:l.76-78; item 3): one banded solve (1D) or one 2D FFT solve (2D periodic) per step.

Everything is fp64 / complex128 numpy + scipy; used only by bench.py's CPU legs.
"""
from __future__ import annotations

import math
import os
import time

import numpy as np
import scipy.fft as sfft
import scipy.linalg as sla

import workloads as W

NPROC = os.cpu_count() or 1


def _theta(cfg):
    return 1.0 if cfg.scheme == W.BE else 0.5


def _taps(cfg):
    """(sub, dia, sup) of the 1D K (ADE / wave), or the 2D periodic stencil weights."""
    if cfg.op in (W.ADE1D, W.WAVE1D):
        h = cfg.h
        nu, a = (cfg.nu, cfg.ax) if cfg.op == W.ADE1D else (1.0, 0.0)
        return -nu / h ** 2 - a / (2 * h), 2 * nu / h ** 2, -nu / h ** 2 + a / (2 * h)
    h = cfg.h
    return (-cfg.nu / h ** 2 - cfg.ax / (2 * h), -cfg.nu / h ** 2 + cfg.ax / (2 * h),
            -cfg.nu / h ** 2 - cfg.ay / (2 * h), -cfg.nu / h ** 2 + cfg.ay / (2 * h), 4 * cfg.nu / h ** 2)


def apply_K(cfg, U):
    """K U for U [..., S] (last axis spatial)."""
    if cfg.op in (W.ADE1D, W.WAVE1D):
        sub, dia, sup = _taps(cfg)
        out = dia * U
        out[..., 1:] += sub * U[..., :-1]
        out[..., :-1] += sup * U[..., 1:]
        return out
    xm, xp, ym, yp, c = _taps(cfg)
    n = cfg.nx
    V = U.reshape(U.shape[:-1] + (n, n))
    out = c * V + xm * np.roll(V, 1, -1) + xp * np.roll(V, -1, -1) + ym * np.roll(V, 1, -2) + yp * np.roll(V, -1, -2)
    return out.reshape(U.shape)


def spectra(cfg):
    nt, dt, a = cfg.nt, cfg.dt, cfg.alpha
    z = a ** (1.0 / nt) * np.exp(-2j * math.pi * np.arange(nt // 2 + 1) / nt)
    if cfg.scheme == W.LF:
        return (1 - z) ** 2 / dt ** 2, (1 + z * z) / 2
    return (1 - z) / dt, (np.ones_like(z) if cfg.scheme == W.BE else (1 + z) / 2)


class FastParaDiag:
    def __init__(self, cfg):
        self.cfg = cfg
        nt = cfg.nt
        self.g = cfg.alpha ** (np.arange(nt) / nt)
        self.l1, self.l2 = spectra(cfg)
        if cfg.op == W.ADE2D:
            n, h = cfg.nx, cfg.h
            th = 2 * math.pi * np.arange(n) / n
            sx = np.sin(th / 2) ** 2
            self.kap = (4 * cfg.nu / h ** 2) * (sx[None, :] + sx[:, None]) \
                + 1j / h * (cfg.ax * np.sin(th)[None, :] + cfg.ay * np.sin(th)[:, None])

    def apply(self, r):
        cfg = self.cfg
        S1 = sfft.rfft(self.g[:, None] * r, axis=0, workers=NPROC)            # Step (a)
        if cfg.op == W.ADE2D:                                                  # Step (b), 2D periodic
            n = cfg.nx
            X = sfft.fft2(S1.reshape(-1, n, n), axes=(1, 2), workers=NPROC, overwrite_x=True)
            X /= self.l1[:, None, None] + self.l2[:, None, None] * self.kap[None]
            S2 = sfft.ifft2(X, axes=(1, 2), workers=NPROC, overwrite_x=True).reshape(S1.shape)
        else:                                                                  # Step (b), 1D Thomas over frequencies
            sub, dia, sup = _taps(cfg)
            a, b, c = self.l2 * sub, self.l1 + self.l2 * dia, self.l2 * sup
            n = cfg.nx
            cp = np.empty((n, S1.shape[0]), dtype=np.complex128)
            d = np.empty_like(cp)
            den = b.copy()
            cp[0] = c / den
            d[0] = S1[:, 0] / den
            for i in range(1, n):
                den = b - a * cp[i - 1]
                cp[i] = c / den
                d[i] = (S1[:, i] - a * d[i - 1]) / den
            for i in range(n - 2, -1, -1):
                d[i] -= cp[i] * d[i + 1]
            S2 = d.T
        z = sfft.irfft(S2, n=cfg.nt, axis=0, workers=NPROC)                   # Step (c)
        return z / self.g[:, None]

    def matvec(self, u):
        cfg = self.cfg
        dt = cfg.dt
        if cfg.scheme == W.LF:
            Bu = u / dt ** 2
            Bu[1:] -= 2 * u[:-1] / dt ** 2
            Bu[2:] += u[:-2] / dt ** 2
            v = 0.5 * u
            v[2:] += 0.5 * u[:-2]
        else:
            th = _theta(cfg)
            Bu = u / dt
            Bu[1:] -= u[:-1] / dt
            v = th * u
            v[1:] += (1 - th) * u[:-1]
        return Bu + apply_K(cfg, v)

    def solve(self, b):
        cfg = self.cfg
        if cfg.solver == "stationary":
            return self._stationary(b)
        return self._gmres(b)

    def _stationary(self, b):
        u = np.zeros_like(b)
        bn = np.linalg.norm(b)
        k = 0
        while True:
            r = b - self.matvec(u)
            if np.linalg.norm(r) <= self.cfg.tol * bn or k >= self.cfg.maxit:
                return u, k
            u += self.apply(r)
            k += 1

    def _gmres(self, b):
        cfg = self.cfg
        m, tol = cfg.m, cfg.tol
        u = np.zeros_like(b)
        bn = np.linalg.norm(b)
        r = b.copy()
        beta = bn
        its = 0
        while True:
            V = [r / beta]
            H = np.zeros((m + 1, m))
            cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
            g[0] = beta
            k = 0
            for j in range(m):
                w = self.matvec(self.apply(V[j]))
                its += 1
                for i in range(j + 1):
                    H[i, j] = np.vdot(V[i], w)
                    w -= H[i, j] * V[i]
                H[j + 1, j] = np.linalg.norm(w)
                for i in range(j):
                    t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                    H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                    H[i, j] = t
                den = math.hypot(H[j, j], H[j + 1, j])
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
                H[j, j], H[j + 1, j] = den, 0.0
                g[j + 1], g[j] = -sn[j] * g[j], cs[j] * g[j]
                k = j + 1
                if abs(g[j + 1]) <= tol * bn or its >= cfg.maxit:
                    break
                V.append(w / np.linalg.norm(w))
            y = sla.solve_triangular(H[:k, :k], g[:k])
            comb = sum(y[i] * V[i] for i in range(k))
            del V
            u += self.apply(comb)
            r = b - self.matvec(u)
            beta = np.linalg.norm(r)
            if beta <= tol * bn or its >= cfg.maxit:
                return u, its


def sequential(cfg, u0, v0=None, f=None):
    """Sequential time stepping from the initial data (the classical route, P:l.76-78): per step one banded solve
    (1D, LAPACK gbsv) or one 2D FFT diagonal solve (2D periodic).  Returns U_1..U_Nt [Nt][S]."""
    nt, dt, S = cfg.nt, cfg.dt, cfg.S
    u = np.empty((nt, S))
    fz = (lambda n: 0.0) if f is None else (lambda n: f[n])
    if cfg.op == W.ADE2D:
        n = cfg.nx
        kap = FastParaDiag(cfg).kap
        th = _theta(cfg)
        lhs = 1 / dt + th * kap
        rm = (1 / dt - (1 - th) * kap) / lhs
        p = sfft.fft2(u0.reshape(n, n), workers=NPROC)
        for k in range(nt):
            p = rm * p
            if f is not None:
                p += sfft.fft2((th * f[k + 1] + (1 - th) * f[k]).reshape(n, n), workers=NPROC) / lhs
            u[k] = sfft.ifft2(p, workers=NPROC).real.reshape(-1)
        return u
    sub, dia, sup = _taps(cfg)
    if cfg.scheme == W.LF:
        ab = np.zeros((3, S))
        ab[0, 1:], ab[1], ab[2, :-1] = 0.5 * sup, 1 / dt ** 2 + 0.5 * dia, 0.5 * sub
        v0 = np.zeros(S) if v0 is None else v0
        u[0] = sla.solve_banded((1, 1), ab, 0.5 * fz(0) + u0 / dt ** 2 + v0 / dt + 0.5 * dt * apply_K(cfg, v0))
        a, c = u0, u[0]
        for k in range(1, nt):
            u[k] = sla.solve_banded((1, 1), ab, fz(k) + (2 * c - a) / dt ** 2 - 0.5 * apply_K(cfg, a))
            a, c = c, u[k]
        return u
    th = _theta(cfg)
    ab = np.zeros((3, S))
    ab[0, 1:], ab[1], ab[2, :-1] = th * sup, 1 / dt + th * dia, th * sub
    prev = u0
    for k in range(nt):
        rhs = prev / dt - (1 - th) * apply_K(cfg, prev) + th * fz(k + 1) + (1 - th) * fz(k)
        prev = sla.solve_banded((1, 1), ab, rhs)
        u[k] = prev
    return u


def rhs(cfg, u0, v0=None, f=None):
    """b of A u = b (readings c4, c5), as the library's pd_build_rhs."""
    nt, S, dt = cfg.nt, cfg.S, cfg.dt
    b = np.zeros((nt, S))
    if cfg.scheme == W.LF:
        v0 = np.zeros(S) if v0 is None else v0
        if f is not None:
            b[0] += 0.5 * f[0]
            b[1:] += f[1:nt]
        b[0] += u0 / dt ** 2 + v0 / dt + 0.5 * dt * apply_K(cfg, v0)
        b[1] += -u0 / dt ** 2 - 0.5 * apply_K(cfg, u0)
        return b
    th = _theta(cfg)
    if f is not None:
        b += th * f[1:] + (1 - th) * f[:-1]
    b[0] += u0 / dt - (1 - th) * apply_K(cfg, u0)
    return b


def timed_solve(cfg):
    """(seconds, iterations) of one fast-CPU ParaDiag-II solve of the workload, and (seconds) of sequential stepping."""
    u0, v0, f = W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg)
    b = rhs(cfg, u0, v0, f)
    pd = FastParaDiag(cfg)
    t0 = time.perf_counter()
    u, its = pd.solve(b)
    t_pd = time.perf_counter() - t0
    t0 = time.perf_counter()
    seq = sequential(cfg, u0, v0, f)
    t_seq = time.perf_counter() - t0
    err = float(np.linalg.norm(u - seq) / np.linalg.norm(seq))
    return t_pd, its, t_seq, err
