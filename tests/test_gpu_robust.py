"""Robustness of the 1D Step (b): the pivoted elimination (csrc/gtsv.cu) behind the recurrence solver.

* Forced (PD_TRIDIAG_GTSV=1) on the configs' operators, the apply and the solves match the oracle exactly as the
  recurrence path does (O1: pivoted banded LU, `oracle.spectral.step_b`).
* A shifted system outside the recurrence regime (both characteristic roots inside the unit circle; it used to be
  rejected with PD_EINVAL) now runs through the fallback.  Such finite Toeplitz sections are ill-conditioned roughly
  like |root|^-N (reading t4): the normwise backward error ||r - P z|| / (||P|| ||z||) is held to 1e-14
  and the forward error to cond * 1e-14.
* Simplified Newton (NEXT-4) on an advection-dominated operator (cell Peclet 8) whose averaged-Jacobian shifted
  systems are not diagonally dominant: row interchanges happen, and the GPU still takes the oracle's iterations.
"""
import os

import numpy as np
import pytest

import workloads as W
from oracle import nonlinear as NL
from oracle import problems, solvers, spectral
from tests.helpers import make_ctx, rel, to_dev, to_host


class forced_gtsv:
    def __enter__(self):
        os.environ["PD_TRIDIAG_GTSV"] = "1"

    def __exit__(self, *a):
        os.environ.pop("PD_TRIDIAG_GTSV", None)


# the least ill-conditioned out-of-regime case of a 4000-point random search (cond_2 = 6.4e8 at its worst frequency)
OUT_OF_REGIME = W.BY_NAME["cfg0"].scaled(name="gtsv_oor", nx=63, nt=16, nu=-0.30771295897629886, ax=-11.408057357170517,
                                         alpha=0.004818795549103244, scheme=W.CN, T=0.18823179057195527)


def shifted_systems(cfg):
    """(A, B, C) of the half-spectrum shifted systems lambda1 I + lambda2 K (test-side, from the oracle's spectra)."""
    lam1, lam2 = spectral.spectra(cfg)
    F = cfg.nt // 2 + 1
    h = 1.0 / (cfg.nx + 1)
    nu = cfg.nu if cfg.op == W.ADE1D else 1.0
    a = cfg.ax if cfg.op == W.ADE1D else 0.0
    sub, dia, sup = -nu / h ** 2 - a / (2 * h), 2 * nu / h ** 2, -nu / h ** 2 + a / (2 * h)
    return lam2[:F] * sub, lam1[:F] + lam2[:F] * dia, lam2[:F] * sup


def test_out_of_regime_case_is_out_of_regime():
    """CPU: the chosen case really leaves the recurrence regime (|r2|^N >= 1e8 or |s|^N >= 1e8 at some frequency)."""
    A, B, C = shifted_systems(OUT_OF_REGIME)
    D = np.sqrt(B * B - 4 * A * C)
    den = np.where(abs(-B - D) >= abs(-B + D), -B - D, -B + D)
    tau = 2 / den
    g = np.maximum(abs(A * tau) ** OUT_OF_REGIME.nx, abs(C * tau) ** OUT_OF_REGIME.nx)
    assert (g >= 1e8).any()


@pytest.mark.gpu
@pytest.mark.parametrize("name,nx,nt", [("cfg0", 63, 32), ("cfg1", 1023, 1024), ("cfg1", 100, 64), ("cfg2", 255, 512),
                                        ("cfg2", 4095, 64)])
def test_forced_gtsv_apply_matches_oracle(name, nx, nt):
    cfg = W.BY_NAME[name].scaled(nx=nx, nt=nt)
    with forced_gtsv():
        ctx = make_ctx(cfg)
    r = W.random_vector(cfg)
    z = to_host(ctx.apply_precond(to_dev(r)))
    ref = spectral.apply_precond(cfg, r)
    assert rel(z, ref) < 1e-10
    assert rel(problems.matvec_P(cfg, z), r) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
def test_forced_gtsv_solve_matches_oracle(name):
    cfg = W.BY_NAME[name]
    with forced_gtsv():
        ctx = make_ctx(cfg)
    b = problems.rhs(cfg, W.initial_u0(cfg), None, W.source_samples(cfg))
    if cfg.solver == "stationary":
        u, rep = ctx.solve_stationary(to_dev(b), tol=cfg.tol, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_stationary(cfg, b)
    else:
        u, rep = ctx.solve_gmres(to_dev(b), tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_gmres(cfg, b)
    assert rep.converged and rep.iterations == rep_ref.iterations
    assert rel(to_host(u), u_ref) < 1e-8


@pytest.mark.gpu
def test_out_of_regime_shift_uses_pivoted_fallback():
    cfg = OUT_OF_REGIME
    A, B, C = shifted_systems(cfg)
    cond = max(np.linalg.cond(np.diag(np.full(cfg.nx, B[n])) + np.diag(np.full(cfg.nx - 1, A[n]), -1)
                              + np.diag(np.full(cfg.nx - 1, C[n]), 1)) for n in range(len(B)))
    ctx = make_ctx(cfg)  # PD_EINVAL before the fallback existed
    r = W.random_vector(cfg)
    z = to_host(ctx.apply_precond(to_dev(r)))
    c1, c2 = problems.time_first_columns(cfg)
    P = np.kron(problems.alpha_circulant(c1, cfg.alpha), np.eye(cfg.S)) + \
        np.kron(problems.alpha_circulant(c2, cfg.alpha), problems.K_matrix(cfg).toarray())
    eta = np.linalg.norm(r.reshape(-1) - P @ z.reshape(-1)) / (np.linalg.norm(P, 2) * np.linalg.norm(z))
    assert eta < 1e-14  # backward stable
    assert rel(z, spectral.apply_precond(cfg, r)) < 1e-14 * cond
    with pytest.raises(RuntimeError, match="recurrence"):  # the 1D tail map needs the recurrence Step (b)
        ctx.tail_map(to_dev(np.zeros((1, cfg.S))))


def _interchanges(cfg, dbar):
    """Row interchanges of partial pivoting (|re| + |im|) over the half-spectrum systems (test-side emulation)."""
    A, B, C = shifted_systems(cfg)
    lam1, lam2 = spectral.spectra(cfg)
    c1 = lambda v: abs(v.real) + abs(v.imag)
    n_sw = 0
    for n in range(len(A)):
        bd = B[n] + lam2[n] * dbar
        cd, cdu = bd[0], C[n]
        for j in range(1, cfg.nx):
            ndu = C[n] if j < cfg.nx - 1 else 0
            if c1(cd) >= c1(A[n]):
                cd, cdu = bd[j] - A[n] / cd * cdu, ndu
            else:
                n_sw += 1
                l = cd / A[n]
                cd, cdu = cdu - l * bd[j], -l * ndu
    return n_sw


@pytest.mark.gpu
def test_newton_without_diagonal_dominance_matches_oracle():
    cfg = W.nl_config(nx=63, nt=64, nu=1e-3, T=0.25)
    rx = NL.Reaction(1.0, -2.0)
    u0 = W.initial_u0(cfg)
    b = NL.rhs(cfg, rx, u0)
    u_ref, rep_ref = NL.solve_newton(cfg, rx, b)
    assert rep_ref.converged
    assert _interchanges(cfg, NL.jac_avg(cfg, rx, u_ref)) > 0
    ctx = make_ctx(cfg)
    ctx.set_reaction(1.0, -2.0)
    u, rep = ctx.solve_newton(to_dev(b), tol=cfg.tol, maxit=cfg.maxit)
    assert rep.converged and rep.iterations == rep_ref.iterations, (rep.history, rep_ref.history)
    assert rel(to_host(u), u_ref) < 1e-8


@pytest.mark.gpu
def test_newton_singular_pivot_reported():
    """A diverging simplified Newton (strong anti-diffusive reaction) ends with PD_ESINGULAR or PD_NOT_CONVERGED,
    never with a silent non-finite iterate reported as converged."""
    cfg = W.nl_config(nx=63, nt=64)
    ctx = make_ctx(cfg)
    ctx.set_reaction(1.0, -60.0)
    u0 = W.initial_u0(cfg)
    b = ctx.build_rhs(to_dev(u0))
    try:
        u, rep = ctx.solve_newton(b, tol=cfg.tol, maxit=cfg.maxit)
    except RuntimeError as e:
        assert "pivot" in str(e) or "not converged" in str(e).lower()
    else:
        assert not rep.converged
