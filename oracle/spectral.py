"""O1: the three-step P_alpha^{-1} r written out with naive DFT matrices (oracle; test infrastructure).

Lemma 1 (P:l.155-174): C_j = V D_j V^{-1}, V = Gamma^{-1} F^*, D_j = diag(sqrt(Nt) F Gamma C_j(:,1)),
Gamma = diag(alpha^{(l-1)/Nt}).  Three steps (eq 1.3, P:l.179-185; eq 2.12, P:l.813-819):
  Step (a)  S1 = (F (x) I)(Gamma (x) I) r
  Step (b)  S2_n = (lambda_{1,n} M + lambda_{2,n} K)^{-1} S1_n,  n = 1..Nt
  Step (c)  z  = (Gamma^{-1} (x) I)(F^* (x) I) S2
Implemented in the Matlab pairing of P:l.864-875 (fft in Step (a), ifft in Step (c)), i.e. numpy's
sign convention e^{-2 pi i jn/Nt}; reading c1 — Lemma 1's omega = e^{+2 pi i/Nt} gives the
same P_alpha^{-1} r with n -> -n.  Every transform here is a dense DFT matrix with exactly reduced
twiddle indices (jk mod N); no FFT, no half-spectrum shortcut.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg

from . import problems
from workloads import ADE1D, ADE2D, WAVE1D, WAVE2D


def gamma(nt: int, alpha: float) -> np.ndarray:
    """diag of Gamma_alpha = (1, alpha^{1/Nt}, ..., alpha^{(Nt-1)/Nt}) (P:l.163-165, 'Gam' at P:l.877-878)."""
    return alpha ** (np.arange(nt, dtype=np.float64) / nt)


def dft_matrix(n: int, sign: int) -> np.ndarray:
    """[exp(sign * 2 pi i (j k mod n) / n)]_{j,k}: the unnormalised DFT matrix (sign=-1: Matlab/numpy fft)."""
    j = np.arange(n)
    idx = np.outer(j, j) % n
    return np.exp(sign * 2j * math.pi * idx / n)


def spectra(cfg, nt: int | None = None, alpha: float | None = None):
    """(lambda_1, lambda_2): the DFT of the Gamma-weighted first columns of C1, C2 (P:l.860-864; Lemma 1).

    lambda_{j,n} = sum_k exp(-2 pi i k n / Nt) alpha^{k/Nt} c_{j,k}   (numpy convention, reading c1)
    """
    nt = cfg.nt if nt is None else nt
    alpha = cfg.alpha if alpha is None else alpha
    c1, c2 = problems.time_first_columns(cfg, nt)
    return column_spectrum(c1, alpha), column_spectrum(c2, alpha)


def column_spectrum(c: np.ndarray, alpha: float) -> np.ndarray:
    """Eigenvalues of the alpha-circulant with first column c: fft(Gam .* c) (P:l.860-864)."""
    return dft_matrix(len(c), -1) @ (gamma(len(c), alpha) * np.asarray(c, dtype=np.float64))


def symbol_2d(cfg) -> np.ndarray:
    """kappa(ky, kx): eigenvalue of the periodic 2D K on the DFT mode exp(i(theta_x x_j + theta_y y_l)).

    Reading c14: kappa = (4 nu / h^2)(sin^2(theta_x/2) + sin^2(theta_y/2)) + (i/h)(a_x sin theta_x + a_y sin theta_y),
    theta = 2 pi k / N.  (Pinned against the sparse stencil in tests/test_oracle_pins.py.)
    """
    n = cfg.nx
    h = cfg.h  # domain length / N
    th = 2.0 * math.pi * np.arange(n) / n
    sx = np.sin(th / 2) ** 2
    kap = (4.0 * cfg.nu / h ** 2) * (sx[None, :] + sx[:, None]) \
        + 1j / h * (cfg.ax * np.sin(th)[None, :] + cfg.ay * np.sin(th)[:, None])
    return kap  # [ky][kx]


def step_a(cfg, r: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """S1 = (F (x) I)(Gamma (x) I) r, unnormalised DFT along time (P:l.866-868: fft(Gam.*(b.')).')."""
    alpha = cfg.alpha if alpha is None else alpha
    nt = r.shape[0]
    return dft_matrix(nt, -1) @ (gamma(nt, alpha)[:, None] * r)


def _tridiag_coeffs(cfg):
    K = problems.K_matrix(cfg)
    return K.diagonal(-1), K.diagonal(0), K.diagonal(1)


def step_b(cfg, S1: np.ndarray, lam1: np.ndarray, lam2: np.ndarray) -> np.ndarray:
    """S2_n = (lambda_{1,n} I + lambda_{2,n} K)^{-1} S1_n for every n (P:l.182, 816; M = I).

    1D (ADE1D, WAVE1D): pivoted banded LU (LAPACK gbsv via scipy.linalg.solve_banded) per n.
    2D periodic: K is diagonalised by the 2D DFT, so the solve is naive 2D DFT -> divide by
    lambda_1 + lambda_2 kappa(k) -> naive inverse 2D DFT (exact, not an approximation).
    2D Dirichlet (WAVE2D): sparse direct LU of lambda_1 I + lambda_2 K per n (as the paper's Matlab code,
    "MATLAB's sparse direct solver", P:l.1315-1316).
    """
    nt = S1.shape[0]
    S2 = np.empty_like(S1, dtype=np.complex128)
    if cfg.op in (ADE1D, WAVE1D):
        sub, dia, sup = _tridiag_coeffs(cfg)
        n = cfg.nx
        for k in range(nt):
            ab = np.zeros((3, n), dtype=np.complex128)
            ab[0, 1:] = lam2[k] * sup
            ab[1, :] = lam1[k] + lam2[k] * dia
            ab[2, :-1] = lam2[k] * sub
            S2[k] = scipy.linalg.solve_banded((1, 1), ab, S1[k])
        return S2
    if cfg.op == ADE2D:
        n = cfg.nx
        Fn, Fi = dft_matrix(n, -1), dft_matrix(n, +1)
        kap = symbol_2d(cfg)
        X = S1.reshape(nt, n, n)                               # [t][y][x]
        Xh = Fn @ X @ Fn.T                                     # forward 2D DFT (y then x)
        Xh = Xh / (lam1[:, None, None] + lam2[:, None, None] * kap[None, :, :])
        Y = (Fi @ Xh @ Fi.T) / (n * n)
        return Y.reshape(nt, n * n)
    if cfg.op == WAVE2D:
        import scipy.sparse as sps
        import scipy.sparse.linalg as spla
        K = problems.K_matrix(cfg).astype(np.complex128)
        eye = sps.identity(cfg.S, format="csc", dtype=np.complex128)
        for k in range(nt):
            S2[k] = spla.splu(sps.csc_matrix(lam1[k] * eye + lam2[k] * K)).solve(S1[k])
        return S2
    raise ValueError(cfg.op)


def step_c(cfg, S2: np.ndarray, alpha: float | None = None, imag_check: bool = True) -> np.ndarray:
    """z = (Gamma^{-1} (x) I)(F^* (x) I) S2 (P:l.870-875: invGam.*ifft(...)); real by conjugate symmetry.

    The imaginary residue is checked before it is discarded (S:l.85, 111) against 1e-11/alpha relative
    to max|z|: rounding in Steps (a)-(b) is amplified by up to Cond_2(V) <= 1/alpha in Step (c)
    (eq 2.13, P:l.823-826), so a fixed 1e-10 rejects correct fp64 results at alpha = 1e-2 (config 2,
    DESIGN.md reading t1); a mis-assembled stencil still leaves an O(1) residue.
    """
    alpha = cfg.alpha if alpha is None else alpha
    nt = S2.shape[0]
    z = (dft_matrix(nt, +1) @ S2) / nt
    z = z / gamma(nt, alpha)[:, None]
    if imag_check:
        scale = max(np.abs(z.real).max(), 1e-300)
        if np.abs(z.imag).max() > max(1e-10, 1e-11 / alpha) * scale:
            raise AssertionError("imaginary residue %.3e too large" % (np.abs(z.imag).max() / scale))
    return z.real.copy()


def apply_precond(cfg, r: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """z = P_alpha^{-1} r by Steps (a), (b), (c) (eq 1.3 / eq 2.12)."""
    alpha = cfg.alpha if alpha is None else alpha
    lam1, lam2 = spectra(cfg, r.shape[0], alpha)
    return step_c(cfg, step_b(cfg, step_a(cfg, r, alpha), lam1, lam2), alpha)
