"""GPU parity of the waveform-relaxation tail form: pd_tail_map against the oracle's
tail map (O3, oracle/tail.py), and pd_solve_stationary_tail / pd_solve_gmres_tail against both the O3 tail-form
solvers and the residual-form oracle solvers (same iteration counts, same solution) on the full configs."""
import numpy as np
import pytest

import workloads as W
from oracle import periodic, problems, solvers, spectral, stepping, tail
from tests.helpers import make_ctx, rel, to_dev, to_host

pytestmark = pytest.mark.gpu

SOLVE_TOL = 1e-8

MAP_CASES = [
    W.CONFIGS[0],                                        # 1D ADE BE, Nx = 63
    W.CONFIGS[1].scaled(nx=1023, nt=256),                # 1D ADE CN, 64 threads x 16 rows (ragged last row)
    W.CONFIGS[2].scaled(nx=4095, nt=64),                 # leapfrog, H = 2, 256 threads
    W.CONFIGS[1].scaled(nx=17, nt=8),                    # tiny, one warp, F < grid
    W.CONFIGS[3].scaled(nx=32, ny=32, nt=64),            # 2D periodic, transfer function
    W.CONFIGS[4].scaled(nx=32, ny=32, nt=1024),          # 2D, tfx context (x-FFT folded into the time FFT)
    W.t4a_config(32),                                    # 2D Dirichlet leapfrog (H = 2): DST-I transfer tables
    W.t4a_config(64, 1.0),                               # 2D Dirichlet, alpha = 1 (resonant), 63 x 63 (ragged tiles)
    W.t4a_config(32).scaled(scheme=W.CN),                # 2D Dirichlet theta-method (H = 1)
]


@pytest.mark.parametrize("cfg", MAP_CASES, ids=lambda c: f"{c.op}-{c.scheme}-{c.nx}-{c.nt}")
def test_tail_map_matches_oracle(cfg):
    ctx = make_ctx(cfg)
    H = ctx.head_blocks
    assert H == tail.head_blocks(cfg)
    g = np.random.default_rng(cfg.nx + cfg.nt).standard_normal((H, cfg.S))
    t_gpu = to_host(ctx.tail_map(to_dev(g)))
    t_ref = tail.tail_map(cfg, g)
    # reading t1 as for the apply: error relative to the whole P^{-1}(E_H g) (the tail alone can be orders of
    # magnitude smaller than the terms summed in Step (c): wave ~1e-6), or 4 delta, delta = distance between the
    # tails of the two independent oracles O1 (DFT) and O2 (alpha-periodic stepping) = the fp64 rounding floor
    # (wave: resonance-conditioned shifted solves, SURVEY [V3])
    v = np.zeros((cfg.nt, cfg.S))
    v[:H] = g
    z1 = spectral.apply_precond(cfg, v)
    delta = 0.0
    if cfg.op != W.ADE1D:  # modal O2 needs the known eigenbasis (wave: DST, 2D: DFT), as check_apply
        delta = np.linalg.norm(z1[cfg.nt - H:] - periodic.apply_precond_modal(cfg, v)[cfg.nt - H:])
    assert np.linalg.norm(t_gpu - t_ref) <= max(max(1e-10, 1e-12 / cfg.alpha) * np.linalg.norm(z1), 4 * delta)


def _rhs(ctx, cfg):
    u0, v0, f = W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg)
    b_dev = ctx.build_rhs(to_dev(u0), to_dev(v0), None if f is None else to_dev(f))
    return b_dev, problems.rhs(cfg, u0, v0, f)


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "cfg2", "cfg3"])
def test_tail_solver_full_config_matches_oracle(name):
    """The config's own solver in tail form: same iteration count as the residual-form oracle, same u,
    residual <= tol; cfg1 has a source (full-support b, anchor path), the others a head-only b."""
    cfg = W.BY_NAME[name]
    ctx = make_ctx(cfg)
    b_dev, b = _rhs(ctx, cfg)
    if cfg.solver == "stationary":
        u, rep = ctx.solve_stationary_tail(b_dev, tol=cfg.tol, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_stationary(cfg, b)
    else:
        u, rep = ctx.solve_gmres_tail(b_dev, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_gmres(cfg, b)
    assert rep.converged and rep_ref.converged
    assert rep.iterations == rep_ref.iterations, (rep.history, rep_ref.history)
    assert rel(to_host(u), u_ref) < SOLVE_TOL
    assert rep.rel_residual <= cfg.tol
    # the reported residual is the true one
    r, n2 = ctx.residual(b_dev, u, norm=True)
    assert np.sqrt(n2) / np.linalg.norm(b) <= 1.01 * cfg.tol


@pytest.mark.parametrize("name,solver", [("cfg1", "stationary"), ("cfg3", "stationary"), ("cfg0", "gmres"),
                                         ("cfg2", "gmres")])
def test_tail_solver_variants_match_o3(name, solver):
    cfg = W.BY_NAME[name]
    if name in ("cfg2", "cfg3"):
        cfg = cfg.scaled(nt=cfg.nt // 4) if cfg.op != W.ADE2D else cfg.scaled(nx=64, ny=64, nt=64)
    cfg = cfg.scaled(solver=solver)
    ctx = make_ctx(cfg)
    b_dev, b = _rhs(ctx, cfg)
    if solver == "stationary":
        u, rep = ctx.solve_stationary_tail(b_dev, tol=cfg.tol, maxit=cfg.maxit)
        u_ref, rep_ref = tail.solve_stationary_tail(cfg, b)
    else:
        u, rep = ctx.solve_gmres_tail(b_dev, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
        u_ref, rep_ref = tail.solve_gmres_tail(cfg, b)
    assert rep.converged and rep.iterations == rep_ref.iterations
    assert rel(to_host(u), u_ref) < SOLVE_TOL


@pytest.mark.parametrize("solver", ["stationary", "gmres"])
def test_tail_full_support_rhs_initial_guess_and_restarts(solver):
    """General b (all blocks non-zero), non-zero initial guess, GMRES(3) restarts: same iterates as the
    residual-form oracle solver."""
    cfg = W.CONFIGS[1].scaled(nx=255, nt=128, alpha=0.05)
    rng = np.random.default_rng(9)
    b = rng.standard_normal((cfg.nt, cfg.S))
    u0 = rng.standard_normal((cfg.nt, cfg.S))
    ctx = make_ctx(cfg)
    if solver == "stationary":
        u, rep = ctx.solve_stationary_tail(to_dev(b), to_dev(u0), tol=1e-10, maxit=60)
        u_ref, rep_ref = solvers.solve_stationary(cfg, b, u0=u0, tol=1e-10, maxit=60)
    else:
        u, rep = ctx.solve_gmres_tail(to_dev(b), to_dev(u0), tol=1e-10, m=3, maxit=60)
        u_ref, rep_ref = solvers.solve_gmres(cfg, b, u0=u0, tol=1e-10, m=3, maxit=60)
    assert rep.converged and rep.iterations == rep_ref.iterations, (rep.history, rep_ref.history)
    assert rel(to_host(u), u_ref) < SOLVE_TOL


def test_tail_cfg4_full_gmres():
    """Full config 4 in tail form: 3 iterations (as the residual form), true residual <= tol, and the same u as
    the residual-form GPU solver."""
    cfg = W.BY_NAME["cfg4"]
    ctx = make_ctx(cfg)
    b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
    u, rep = ctx.solve_gmres_tail(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    assert rep.converged and rep.rel_residual <= cfg.tol and rep.iterations == 3
    u2, rep2 = ctx.solve_gmres(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    assert rep2.iterations == 3
    import torch
    assert float(torch.linalg.norm(u - u2) / torch.linalg.norm(u2)) < SOLVE_TOL


def test_tail_cfg2_matches_sequential():
    cfg = W.BY_NAME["cfg2"]
    ctx = make_ctx(cfg)
    b_dev, _ = _rhs(ctx, cfg)
    u, rep = ctx.solve_stationary_tail(b_dev, tol=cfg.tol, maxit=cfg.maxit)
    seq = stepping.march(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    assert rep.converged and rep.iterations == 5
    assert rel(to_host(u), seq) < SOLVE_TOL


@pytest.mark.parametrize("name,P", [("cfg1", 3), ("cfg2", 2), ("cfg3", 4), ("cfg0", 2)])
def test_tail_sharded_virtual_ranks(name, P):
    """Sharded tail form on P virtual ranks (replicated heads, per-shard frequency split of the 1D tail map summed
    over the shards, distributed applies at start and exit): same counts and solution as the oracle."""
    cfg = W.BY_NAME[name]
    if name == "cfg2":
        cfg = cfg.scaled(nt=1024)
    ctx = make_ctx(cfg, rank=-1, size=P)
    b_dev, b = _rhs(ctx, cfg)
    g = np.random.default_rng(P).standard_normal((ctx.head_blocks, cfg.S))
    t_ref = tail.tail_map(cfg, g)
    v = np.zeros((cfg.nt, cfg.S))
    v[: ctx.head_blocks] = g
    scale = np.linalg.norm(spectral.apply_precond(cfg, v))
    assert np.linalg.norm(to_host(ctx.tail_map(to_dev(g))) - t_ref) <= 1e-10 * max(scale, 1.0)
    if cfg.solver == "stationary":
        u, rep = ctx.solve_stationary_tail(b_dev, tol=cfg.tol, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_stationary(cfg, b)
    else:
        u, rep = ctx.solve_gmres_tail(b_dev, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
        u_ref, rep_ref = solvers.solve_gmres(cfg, b)
    assert rep.converged and rep.iterations == rep_ref.iterations
    assert rel(to_host(u), u_ref) < SOLVE_TOL


@pytest.mark.parametrize("label,alpha", [(32, 0.1), (64, 0.1), (128, 0.1), (32, 1.0)])
def test_tail_gmres_2d_dirichlet_matches_oracle(label, alpha):
    """Table T4A in tail form (NEXT-3 with NEXT-1): GMRES on the head/tail reduced problem takes the residual-form
    oracle's iteration count and solution (alpha = 1: the count pinned per mesh as in test_t4a, reading x4)."""
    cfg = W.t4a_config(label, alpha)
    ctx = make_ctx(cfg)
    b_dev, b = _rhs(ctx, cfg)
    u, rep = ctx.solve_gmres_tail(b_dev, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    u_ref, rep_ref = solvers.solve_gmres(cfg, b)
    assert rep.converged
    if alpha < 1.0:
        assert rep.iterations == rep_ref.iterations
        assert rel(to_host(u), u_ref) < SOLVE_TOL
    else:  # reading x4: within the range of the three references of tests/golden/t4a_alpha1_counts.json
        import json
        import os
        with open(os.path.join(os.path.dirname(__file__), "golden", "t4a_alpha1_counts.json")) as fh:
            runs = json.load(fh)["runs"]
        refs = [runs[f"{label}_{n}"]["iterations"] for n in ("O1_fp64", "O2_fp64", "O2_longdouble")]
        assert min(refs) <= rep.iterations <= max(refs), (rep.iterations, refs)
        assert np.linalg.norm(problems.matvec_A(cfg, to_host(u)) - b) <= 1.01 * cfg.tol * np.linalg.norm(b)
