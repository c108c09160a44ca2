"""Table ctp-01 (P:l.954-978): iteration numbers of ParaDiag-II (B-E) and (TR) for the 2D
periodic advection-diffusion problem eq 2.14 on (0,1)^2, dx = dy = dt = 1/128, Nt = 512, alpha = 0.02,
tol = 1e-6, nu = 1 .. 1e-5.

The paper does not state which quantity it compares with tol (reading x2).  tests/golden/
ctp01_oracle.json (written by tools/ctp01_rules.py, oracle only) holds the oracle's per-iteration residuals,
successive differences and errors; under the solvers' rule ||b - A u^k|| <= tol ||b|| (reading c6) every case
takes 4 iterations, under a successive-difference rule 5.  The printed counts are 4-5; what is pinned here is the
paper's claim itself - parameter-robust counts within one iteration of the printed ones - and, on the GPU, that
the CUDA path takes exactly the oracle's iterations with the oracle's residual history."""
import json
import os

import numpy as np
import pytest

import workloads as W
from oracle import problems, solvers, spectral
from tests.helpers import make_ctx, rel, to_dev, to_host

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ctp01_oracle.json")


def _golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def test_ctp01_config_is_the_papers():
    """dx = dy = dt = 1/128, Nt = 512 (P:l.957-959), Omega = (0,1)^2, alpha = 0.02 (P:l.946), tol = 1e-6
    (P:l.982-984), u0 = exp(-20((x-1/2)^2 + (y-1/2)^2)) (P:l.910-912)."""
    for s in (W.BE, W.CN):
        cfg = W.ctp01_config(s, 1e-2)
        assert cfg.h == 1.0 / 128 and cfg.dt == 1.0 / 128 and cfg.nt == 512 and cfg.nx == cfg.ny == 128
        assert cfg.alpha == 0.02 and cfg.tol == 1e-6 and cfg.length == 1.0
    u0 = W.initial_u0(W.ctp01_config(W.BE, 1.0)).reshape(128, 128)
    assert u0[64, 64] == 1.0 and abs(u0[0, 0] - np.exp(-10.0)) < 1e-15


def test_ctp01_golden_counts_within_one_of_paper():
    g = _golden()
    assert g["paper_counts"] == {"be": [4, 4, 5, 5, 5, 5], "cn": [4, 5, 5, 5, 5, 5]}
    for s in ("be", "cn"):
        paper = np.array(g["paper_counts"][s])
        res = np.array(g["counts"]["res_rel2"][s])
        dif = np.array(g["counts"]["dif_inf"][s])
        assert np.all(res <= paper) and np.all(res >= paper - 1)       # residual rule: 4 vs 4-5
        assert np.all(dif >= paper) and np.all(dif <= paper + 1)       # successive differences: 5 vs 4-5
        for c in (res, dif):
            assert c.max() - c.min() <= 1                               # robust in nu (the table's claim)


@pytest.mark.slow
def test_ctp01_golden_reproduced_by_oracle():
    """Re-run one case of the generator (B-E, nu = 1e-2) with the oracle as it stands."""
    g = _golden()
    cfg = W.ctp01_config(W.BE, 1e-2)
    b = problems.rhs(cfg, W.initial_u0(cfg))
    u = np.zeros_like(b)
    rows = g["runs"]["be_0.01"]
    for k in range(3):
        u = u + spectral.apply_precond(cfg, solvers.residual(cfg, b, u))
        rr = np.linalg.norm(solvers.residual(cfg, b, u)) / np.linalg.norm(b)
        assert abs(rr - rows[k]["res_rel2"]) <= 1e-8 * rows[k]["res_rel2"]


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", [W.BE, W.CN])
@pytest.mark.parametrize("nu", list(W.CTP01_NUS))
def test_ctp01_gpu_matches_oracle(scheme, nu):
    g = _golden()
    cfg = W.ctp01_config(scheme, nu)
    rows = g["runs"][f"{scheme}_{nu}"]
    expect = g["counts"]["res_rel2"][scheme][list(W.CTP01_NUS).index(nu)]
    ctx = make_ctx(cfg)
    b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
    u_ref = None
    if nu == 1e-2:  # one viscosity per scheme: the oracle's iterate itself, element by element
        bh = problems.rhs(cfg, W.initial_u0(cfg))
        assert rel(to_host(b), bh) < 1e-13
        u_ref, rep_ref = solvers.solve_stationary(cfg, bh)
        assert rep_ref.iterations == expect
    for solve in (ctx.solve_stationary, ctx.solve_stationary_tail):
        u, rep = solve(b, tol=cfg.tol, maxit=cfg.maxit)
        assert rep.converged and rep.iterations == expect
        for k, h in enumerate(rep.history):
            assert abs(h - rows[k]["res_rel2"]) <= 1e-6 * rows[k]["res_rel2"] + 1e-14
        if u_ref is not None:
            assert rel(to_host(u), u_ref) < 1e-9    # the same iterate u^k (not a converged limit): rounding only
    assert np.all(np.isfinite(to_host(u)))
