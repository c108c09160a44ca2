"""O0: brute-force dense assembly and dense LU (oracle; test infrastructure). Tiny sizes only.

A = B1 (x) M + B2 (x) K (P:l.80-84, eq 1.1);  P_alpha = C1 (x) M + C2 (x) K (P:l.114-116, eq 1.2).
z = P_alpha^{-1} r is *defined* as the unique solution of P_alpha z = r ("plain definition").
"""
from __future__ import annotations

import numpy as np

from . import problems


def assemble_A(cfg) -> np.ndarray:
    c1, c2 = problems.time_first_columns(cfg)
    K = problems.K_matrix(cfg).toarray()
    return np.kron(problems.toeplitz_lower(c1), np.eye(cfg.S)) + np.kron(problems.toeplitz_lower(c2), K)


def assemble_P(cfg, alpha: float | None = None) -> np.ndarray:
    alpha = cfg.alpha if alpha is None else alpha
    c1, c2 = problems.time_first_columns(cfg)
    K = problems.K_matrix(cfg).toarray()
    return (np.kron(problems.alpha_circulant(c1, alpha), np.eye(cfg.S))
            + np.kron(problems.alpha_circulant(c2, alpha), K))


def apply_precond(cfg, r: np.ndarray, alpha: float | None = None) -> np.ndarray:
    """z = P_alpha^{-1} r by dense LU of the assembled P_alpha."""
    P = assemble_P(cfg, alpha)
    return np.linalg.solve(P, r.reshape(-1)).reshape(r.shape)


def solve_A(cfg, b: np.ndarray) -> np.ndarray:
    """u = A^{-1} b by dense LU of the assembled all-at-once matrix."""
    return np.linalg.solve(assemble_A(cfg), b.reshape(-1)).reshape(b.shape)
