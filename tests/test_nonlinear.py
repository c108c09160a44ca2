"""Nonlinear ParaDiag-II by simplified Newton (eq 1.4-1.5, P:l.196-227): oracle O4 pins
(CPU) and GPU parity of pd_solve_newton (same iteration count, same iterates, converged = sequential stepping)."""
import numpy as np
import pytest

import workloads as W
from oracle import problems, solvers
from oracle import nonlinear as NL
from tests.helpers import make_ctx, rel, to_dev, to_host

RX = NL.Reaction(*W.NL_REACTION)


def _small(scheme=W.CN, **kw):
    return W.nl_config(nx=63, nt=64, scheme=scheme, **kw)


def test_nl_reduces_to_linear_residual():
    """g = 0: the nonlinear residual and rhs are the linear ones (eq 1.4 with F(u) = (I (x) K) u)."""
    cfg = _small()
    rng = np.random.default_rng(0)
    u, b = rng.standard_normal((cfg.nt, cfg.S)), rng.standard_normal((cfg.nt, cfg.S))
    z = NL.Reaction(0.0, 0.0)
    assert rel(NL.residual(cfg, z, b, u), solvers.residual(cfg, b, u)) < 1e-14
    u0 = rng.standard_normal(cfg.S)
    assert rel(NL.rhs(cfg, z, u0), problems.rhs(cfg, u0)) < 1e-14


@pytest.mark.parametrize("scheme", [W.BE, W.CN])
def test_nl_sequential_solution_has_zero_residual(scheme):
    """The sequential full-Newton march solves eq 1.4 with the b of NL.rhs: pins rhs, F, the time taps and g."""
    cfg = _small(scheme)
    u0 = W.initial_u0(cfg)
    seq = NL.march(cfg, RX, u0)
    b = NL.rhs(cfg, RX, u0)
    assert np.linalg.norm(NL.residual(cfg, RX, b, seq)) <= 1e-11 * np.linalg.norm(b)


def test_nl_preconditioner_is_the_averaged_jacobian_circulant():
    """P_alpha(u)^{-1} r solves (C1 (x) I + C2 (x) (K + diag(mean_n g'(U_n)))) z = r (dense assembly)."""
    cfg = _small()
    rng = np.random.default_rng(1)
    u, r = rng.standard_normal((cfg.nt, cfg.S)), rng.standard_normal((cfg.nt, cfg.S))
    dbar = NL.jac_avg(cfg, RX, u)
    assert np.allclose(dbar, (3 * u ** 2 - 1).mean(axis=0))
    z = NL.apply_precond(cfg, r, dbar)
    c1, c2 = problems.time_first_columns(cfg)
    J = problems.K_matrix(cfg).toarray() + np.diag(dbar)
    P = np.kron(problems.alpha_circulant(c1, cfg.alpha), np.eye(cfg.S)) + np.kron(problems.alpha_circulant(c2, cfg.alpha), J)
    assert rel(P @ z.reshape(-1), r.reshape(-1)) < 1e-12


@pytest.mark.parametrize("scheme", [W.BE, W.CN])
def test_nl_newton_converges_to_sequential(scheme):
    cfg = _small(scheme)
    u0 = W.initial_u0(cfg)
    u, rep = NL.solve_newton(cfg, RX, NL.rhs(cfg, RX, u0))
    assert rep.converged and 5 <= rep.iterations <= 20
    assert rel(u, NL.march(cfg, RX, u0)) < 1e-8
    h = rep.history
    for i in range(2, len(h)):  # linear convergence of the simplified Newton (rate well below 1)
        assert h[i] < 0.5 * h[i - 1]


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,nx,nt", [(W.CN, 63, 64), (W.BE, 255, 256), (W.CN, 1023, 1024), (W.CN, 100, 32),
                                          (W.BE, 4095, 16)])
def test_nl_gpu_matches_oracle(scheme, nx, nt):
    cfg = W.nl_config(nx=nx, nt=nt, scheme=scheme)
    u0 = W.initial_u0(cfg)
    b = NL.rhs(cfg, RX, u0)
    ctx = make_ctx(cfg)
    ctx.set_reaction(*W.NL_REACTION)
    bd = ctx.build_rhs(to_dev(u0))
    assert rel(to_host(bd), b) < 1e-13
    u, rep = ctx.solve_newton(bd, tol=cfg.tol, maxit=cfg.maxit)
    u_ref, rep_ref = NL.solve_newton(cfg, RX, b)
    assert rep.converged and rep.iterations == rep_ref.iterations, (rep.history, rep_ref.history)
    assert rel(to_host(u), u_ref) < 1e-8
    floor = residual_floor(cfg, b, u_ref)
    print(f"newton {nx}x{nt}: residual rounding floor {floor:.2e}")
    for a, c in zip(rep.history, rep_ref.history):
        assert abs(a - c) <= 1e-6 * c + floor


def residual_floor(cfg, b, u):
    """Rounding floor of a relative residual ||b - (B1 u + B2 F(u))|| / ||b|| computed in fp64 (DESIGN.md reading
    n1): each entry is a sum of O(10) products, so its absolute error is of order eps times the same sum taken over
    absolute values, |b| + |B1| |u| + |B2| (|K| |u| + |g(u)|) (8 eps used); the history entries near tol are
    differences of such sums and cannot agree below it (1023 x 1024: 1.8e-12; 4095 x 16, where |K| = 3.4e5: 2e-10)."""
    c1, c2 = problems.time_first_columns(cfg)
    absK = abs(problems.K_matrix(cfg))
    au = np.abs(u)
    kg = np.ascontiguousarray((absK @ au.T).T) + np.abs(RX.g(u))
    tot = np.abs(b) + problems.apply_time(np.abs(c1), au, None) + problems.apply_time(np.abs(c2), kg, None)
    return 8 * np.finfo(np.float64).eps * float(np.linalg.norm(tot) / np.linalg.norm(b))
