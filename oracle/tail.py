"""O3: the waveform-relaxation "tail" form of the stationary iteration and of GMRES.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference arm may import this module.

Why it exists (P:l.120-124, 762-773, 928-931).  P_alpha - A = (C1 - B1) (x) I + (C2 - B2) (x) K is non-zero
only in the alpha-corner of the alpha-circulants: entry (i, j), i < j, equals alpha c_{i-j+Nt} (eq 2.9-2.10 for
the theta-method, eq 3.4 for leapfrog).  With H taps beyond the diagonal (H = 1 theta-method, H = 2 leapfrog)
the corner couples the first H time blocks (the "head") to the last H blocks (the "tail") only:
    (P - A) u = E_H G U_tail,   (G U_tail)_i = sum_j alpha (c1_{i-j+Nt} U_j + c2_{i-j+Nt} K U_j),
so the stationary iteration  P u^{k+1} = (P - A) u^k + b  (P:l.120-124) is
    u^{k+1} = P^{-1} b + P^{-1}(E_H G U^k_tail)
and only the tail has to be carried between iterations (the head-tail coupling of waveform relaxation,
P:l.762-773).  Step (a) of a head-supported vector is the H-term sum S1_n = sum_{t<H} gamma_t w^{nt} g_t (the
"economical" Step (a) of P:l.928-931), and only the last H rows of Step (c) are needed.
Residual: r^k = b - A u^k = (P - A)(u^k - u^{k-1}) = E_H G (U^k_tail - U^{k-1}_tail).

GMRES (right-preconditioned, as solvers.solve_gmres): with r0 = b - A u0, every Krylov vector has the form
a r0 + E_H h, because A P^{-1} v = v - E_H G tail(P^{-1} v) and tail(P^{-1}(a r0 + E_H h)) =
a tail(P^{-1} r0) + T(h) with T the tail map below.  The basis is carried as (a_j, h_j); inner products
expand into a_i a_j ||r0||^2 + a_i <r0_head, h_j> + a_j <h_i, r0_head> + <h_i, h_j>.  Arnoldi, Givens and the
stopping rule are those of solvers.solve_gmres (same iterates in exact arithmetic).
"""
from __future__ import annotations

import numpy as np

from . import problems, solvers, spectral
from .solvers import Report


def head_blocks(cfg) -> int:
    """H = number of non-zero taps of the time first columns beyond the diagonal (1 theta, 2 leapfrog)."""
    c1, c2 = problems.time_first_columns(cfg)
    nz = [k for k in range(1, len(c1)) if c1[k] != 0.0 or c2[k] != 0.0]
    return max(nz) if nz else 0


def head_from_tail(cfg, tail: np.ndarray) -> np.ndarray:
    """(P - A) restricted to head rows x tail columns: head[i] = sum_j alpha (c1_{i-j+Nt} U_j + c2_{i-j+Nt} K U_j).

    tail: [H][S] = blocks Nt-H .. Nt-1 of u.  Built from the alpha-circulant definition (P:l.80-84, eq 1.2).
    """
    nt, alpha = cfg.nt, cfg.alpha
    c1, c2 = problems.time_first_columns(cfg)
    H = tail.shape[0]
    head = np.zeros_like(tail)
    for i in range(H):
        for jj in range(H):
            j = nt - H + jj
            if i >= j:
                continue                       # only the strictly upper (wrapped) corner
            k = i - j + nt
            if k >= nt:
                continue
            head[i] += alpha * c1[k] * tail[jj]
            if c2[k] != 0.0:
                head[i] += alpha * c2[k] * problems.apply_K(cfg, tail[jj][None, :])[0]
    return head


def tail_map(cfg, head: np.ndarray) -> np.ndarray:
    """T(g) = last H blocks of P^{-1}(E_H g), by the three steps restricted to the support (P:l.928-931).

    Step (a): S1_n = sum_{t<H} gamma_t exp(-2 pi i n t / Nt) g_t   (the DFT of a vector supported on t < H)
    Step (b): S2_n = (lambda_1n I + lambda_2n K)^{-1} S1_n          (spectral.step_b, every n)
    Step (c): z_t = gamma_t^{-1} / Nt sum_n exp(+2 pi i n t / Nt) S2_n  for t = Nt-H .. Nt-1 only.
    """
    nt, alpha = cfg.nt, cfg.alpha
    H = head.shape[0]
    g = spectral.gamma(nt, alpha)
    n = np.arange(nt)
    S1 = np.zeros((nt, head.shape[1]), dtype=np.complex128)
    for t in range(H):
        S1 += (g[t] * np.exp(-2j * np.pi * n * t / nt))[:, None] * head[t][None, :]
    lam1, lam2 = spectral.spectra(cfg)
    S2 = spectral.step_b(cfg, S1, lam1, lam2)
    out = np.empty((H, head.shape[1]))
    for a in range(H):
        t = nt - H + a
        z = (np.exp(2j * np.pi * n * t / nt) @ S2) / nt / g[t]
        # imaginary residue relative to the size of the summed terms (reading t1: rounding of Steps (a)-(b)
        # amplified by at most Cond_2(V) <= 1/alpha, eq 2.13); the tail itself may be far smaller
        scale = max(np.abs(S2).max() / g[t], 1e-300)
        if np.abs(z.imag).max() > max(1e-10, 1e-11 / alpha) * scale:
            raise AssertionError("tail map: imaginary residue %.3e" % (np.abs(z.imag).max() / scale))
        out[a] = z.real
    return out


def _embed_head(cfg, head: np.ndarray) -> np.ndarray:
    v = np.zeros((cfg.nt, cfg.S))
    v[: head.shape[0]] = head
    return v


def solve_stationary_tail(cfg, b, u0=None, tol=None, maxit=None):
    """Stationary ParaDiag-II (eq 5.1) carried on the tail: t^{k+1} = tail(P^{-1} b) + T(G t^k),
    ||r^k|| = ||G (t^k - t^{k-1})||, u^k = P^{-1}(b + E_H G t^{k-1}) assembled once at exit."""
    tol = cfg.tol if tol is None else tol
    maxit = cfg.maxit if maxit is None else maxit
    H = head_blocks(cfg)
    u = np.zeros_like(b) if u0 is None else u0.copy()
    bnorm = np.linalg.norm(b)
    rel = np.linalg.norm(solvers.residual(cfg, b, u)) / bnorm
    if rel <= tol or maxit <= 0:
        return u, Report(0, rel <= tol, rel, [])
    y_tail = spectral.apply_precond(cfg, b)[cfg.nt - H:]
    t_prev = u[cfg.nt - H:].copy()
    hist = []
    k = 0
    while True:
        t = y_tail + tail_map(cfg, head_from_tail(cfg, t_prev))
        k += 1
        rel = np.linalg.norm(head_from_tail(cfg, t - t_prev)) / bnorm
        hist.append(rel)
        if rel <= tol or k >= maxit:
            break
        t_prev = t
    u = spectral.apply_precond(cfg, b + _embed_head(cfg, head_from_tail(cfg, t_prev)))
    return u, Report(k, rel <= tol, rel, hist)


def solve_gmres_tail(cfg, b, u0=None, tol=None, m=None, maxit=None):
    """Right-preconditioned restarted GMRES(m) with the basis carried as (a_j, h_j): v_j = a_j r0 + E_H h_j.

    Same Arnoldi (modified Gram-Schmidt), Givens rotations and stopping rule as solvers.solve_gmres; at exit or
    restart u = u0 + P^{-1}(c r0 + E_H h) and the true residual is recomputed from u.
    """
    tol = cfg.tol if tol is None else tol
    m = cfg.m if m is None else m
    maxit = cfg.maxit if maxit is None else maxit
    H = head_blocks(cfg)
    u = np.zeros_like(b) if u0 is None else u0.copy()
    bnorm = np.linalg.norm(b)
    hist = []
    its = 0
    r0 = solvers.residual(cfg, b, u)
    beta = np.linalg.norm(r0)
    if beta <= tol * bnorm:
        return u, Report(0, True, beta / bnorm, hist)
    while True:
        r0h = r0[:H]
        rr = float(np.sum(r0 * r0))
        q0 = head_from_tail(cfg, spectral.apply_precond(cfg, r0)[cfg.nt - H:])  # G tail(P^{-1} r0)

        def dot(x, y):
            (a1, h1), (a2, h2) = x, y
            return a1 * a2 * rr + a1 * np.sum(r0h * h2) + a2 * np.sum(h1 * r0h) + np.sum(h1 * h2)

        V = [(1.0 / beta, np.zeros((H, cfg.S)))]
        Hm = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        k = 0
        breakdown = False
        for j in range(m):
            a, h = V[j]
            # A P^{-1} (a r0 + E h) = a (r0 - E q0) + E (h - G T(h))
            wa, wh = a, h - head_from_tail(cfg, tail_map(cfg, h)) - a * q0
            its += 1
            for i in range(j + 1):
                Hm[i, j] = dot((wa, wh), V[i])
                wa, wh = wa - Hm[i, j] * V[i][0], wh - Hm[i, j] * V[i][1]
            hnext = np.sqrt(max(dot((wa, wh), (wa, wh)), 0.0))
            Hm[j + 1, j] = hnext
            for i in range(j):
                t = cs[i] * Hm[i, j] + sn[i] * Hm[i + 1, j]
                Hm[i + 1, j] = -sn[i] * Hm[i, j] + cs[i] * Hm[i + 1, j]
                Hm[i, j] = t
            den = np.hypot(Hm[j, j], Hm[j + 1, j])
            cs[j], sn[j] = Hm[j, j] / den, Hm[j + 1, j] / den
            Hm[j, j] = den
            Hm[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) <= tol * bnorm or its >= maxit:
                break
            if hnext == 0.0:
                breakdown = True
                break
            V.append((wa / hnext, wh / hnext))
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - np.dot(Hm[i, i + 1:k], y[i + 1:k])) / Hm[i, i]
        ca = sum(y[i] * V[i][0] for i in range(k))
        ch = sum(y[i] * V[i][1] for i in range(k))
        u = u + spectral.apply_precond(cfg, ca * r0 + _embed_head(cfg, ch))
        r0 = solvers.residual(cfg, b, u)
        beta = np.linalg.norm(r0)
        if beta <= tol * bnorm:
            return u, Report(its, True, beta / bnorm, hist)
        if its >= maxit or breakdown:
            return u, Report(its, False, beta / bnorm, hist)
