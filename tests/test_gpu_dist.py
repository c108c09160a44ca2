"""GPU parity of the sharded path on one B200: `size` virtual ranks in one process execute
the same partition plan, slab time FFTs, frequency-shard spatial solves, pitched all-to-all block moves and
halo residuals as the NCCL mode, compared with the CPU oracle."""
import numpy as np
import pytest

import workloads as W
from oracle import problems, solvers, spectral
from tests.helpers import make_ctx, rel, to_dev, to_host

pytestmark = pytest.mark.gpu


def _cases():
    return [
        ("ade1d_be_P2", W.CONFIGS[0].scaled(nx=63, nt=32), 2),
        ("ade1d_cn_P3_ragged", W.CONFIGS[1].scaled(nx=301, nt=64, alpha=0.02), 3),
        ("wave_P4", W.CONFIGS[2].scaled(nx=255, nt=128, alpha=0.02), 4),
        ("ade1d_cn_tf4_P2", W.CONFIGS[1].scaled(nx=511, nt=1024), 2),
        ("ade2d_be_P2", W.CONFIGS[3].scaled(nx=32, ny=32, nt=16), 2),
        ("ade2d_cn_P3", W.CONFIGS[4].scaled(nx=64, ny=64, nt=64, alpha=1e-3), 3),
        ("ade2d_cn_tf4_P4", W.CONFIGS[4].scaled(nx=32, ny=32, nt=2048, alpha=1e-3), 4),
        ("ade2d_be_tfx_P3_ragged", W.CONFIGS[3].scaled(nx=64, ny=64, nt=1024), 3),
        ("wave2d_P3_ragged", W.t4a_config(32, 0.1), 3),
    ]


@pytest.mark.parametrize("name,cfg,P", _cases())
def test_sharded_apply_residual_rhs(name, cfg, P):
    ctx = make_ctx(cfg, rank=-1, size=P)
    rng = np.random.default_rng(P)
    r = W.random_vector(cfg, seed=11)
    z = to_host(ctx.apply_precond(to_dev(r)))
    assert rel(z, spectral.apply_precond(cfg, r)) < 1e-10
    assert rel(problems.matvec_P(cfg, z), r) < 1e-10
    u = rng.standard_normal((cfg.nt, cfg.S))
    b = rng.standard_normal((cfg.nt, cfg.S))
    res, n2 = ctx.residual(to_dev(b), to_dev(u), norm=True)
    ref = solvers.residual(cfg, b, u)
    assert rel(to_host(res), ref) < 1e-13
    assert n2 == pytest.approx(float((ref ** 2).sum()), rel=1e-12)
    assert rel(to_host(ctx.matvec(to_dev(u))), problems.matvec_A(cfg, u)) < 1e-13
    u0, v0 = rng.standard_normal(cfg.S), rng.standard_normal(cfg.S)
    f = rng.standard_normal((cfg.nt + 1, cfg.S))
    assert rel(to_host(ctx.build_rhs(to_dev(u0), to_dev(v0), to_dev(f))), problems.rhs(cfg, u0, v0, f)) < 1e-13
    assert rel(to_host(ctx.build_rhs(to_dev(u0))), problems.rhs(cfg, u0)) < 1e-13


@pytest.mark.parametrize("name,P", [("cfg0", 2), ("cfg1", 4), ("cfg3", 4)])
def test_sharded_solves_match_single_gpu_and_oracle(name, P):
    cfg = W.BY_NAME[name]
    b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    ctx1 = make_ctx(cfg)
    ctxP = make_ctx(cfg, rank=-1, size=P)
    fn = "solve_stationary" if cfg.solver == "stationary" else "solve_gmres"
    kw = dict(tol=cfg.tol, maxit=cfg.maxit) if fn == "solve_stationary" else dict(tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    u1, rep1 = getattr(ctx1, fn)(to_dev(b), **kw)
    uP, repP = getattr(ctxP, fn)(to_dev(b), **kw)
    ref = (solvers.solve_stationary if fn == "solve_stationary" else solvers.solve_gmres)(cfg, b)
    assert repP.converged and repP.iterations == rep1.iterations == ref[1].iterations
    assert rel(to_host(uP), ref[0]) < 1e-8
    assert rel(to_host(uP), to_host(u1)) < 1e-10


def test_partition_rejects_too_many_ranks():
    from paper_2005_09158_b200 import ParaDiagError
    with pytest.raises(ParaDiagError):
        make_ctx(W.CONFIGS[0].scaled(nx=3, nt=32), rank=-1, size=4)
