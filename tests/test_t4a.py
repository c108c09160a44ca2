"""Table T4A (P:l.1309-1349): 2D Dirichlet wave u_tt = Lap u + f on (0,1)^2, T = 2, exact
u = sin(pi x) sin(pi y) e^t, implicit leapfrog (eq 3.2b), right-preconditioned GMRES with P_alpha, tol 1e-10.

Oracle pins of the new operator (K = -Lap_h, Dirichlet; O1 with sparse direct Step (b), O2 in the tensor DST-I
basis, O0 dense) and the table's claims against tests/golden/t4a_oracle.json (tools/t4a_oracle.py, oracle only):
alpha = 0.1 takes 3 iterations at every mesh (printed: 3, 3, 3, 3), alpha = 1 grows with the mesh (printed 3, 7,
37, > 50; the counts are sensitive to the unstated mesh/GMRES details, readings x3/x4), second-order
errors (printed orders 1.9-2.0) within a factor two of the printed 7.17e-3 ... 1.20e-4.  GPU: the CUDA path takes
the oracle's iterations with the oracle's solution."""
import json
import math
import os

import numpy as np
import pytest

import workloads as W
from oracle import dense, periodic, problems, solvers, spectral, stepping
from tests.helpers import make_ctx, rel, to_dev, to_host

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "t4a_oracle.json")


def _golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def test_wave2d_operator_is_dirichlet_laplacian():
    """K = -Lap_h: 4/h^2 on the diagonal, -1/h^2 to the four neighbours, nothing across the boundary, and the
    tensor DST-I modes are its eigenvectors with mu_k + mu_l (textbook eigenpairs)."""
    cfg = W.t4a_config(8)
    n, h = cfg.nx, cfg.h
    assert n == 7 and h == 1.0 / 8
    K = problems.K_matrix(cfg).toarray()
    assert K[0, 0] == pytest.approx(4 / h ** 2) and K[0, 1] == pytest.approx(-1 / h ** 2)
    assert K[0, n] == pytest.approx(-1 / h ** 2) and K[n - 1, n] == 0.0  # row end: no wrap
    j = np.arange(1, n + 1)
    for k, l in ((1, 1), (2, 5), (7, 3)):
        v = np.outer(np.sin(math.pi * l * j / (n + 1)), np.sin(math.pi * k * j / (n + 1))).reshape(-1)
        mu = 4 / h ** 2 * (math.sin(math.pi * k / (2 * (n + 1))) ** 2 + math.sin(math.pi * l / (2 * (n + 1))) ** 2)
        assert np.abs(K @ v - mu * v).max() < 1e-10 * mu


@pytest.mark.parametrize("alpha", [0.1, 1.0])
def test_wave2d_oracles_agree(alpha):
    """O1 (DFT in time + sparse direct Step (b)) = O0 (dense solve) = O2 (alpha-periodic stepping in the DST basis)."""
    cfg = W.t4a_config(8, alpha)
    r = np.random.default_rng(5).standard_normal((cfg.nt, cfg.S))
    z1 = spectral.apply_precond(cfg, r)
    assert rel(z1, dense.apply_precond(cfg, r)) < 1e-12
    assert rel(periodic.apply_precond_modal(cfg, r), z1) < 1e-11
    assert rel(problems.matvec_P(cfg, z1), r) < 1e-12


def test_wave2d_converged_equals_sequential_and_exact():
    cfg = W.t4a_config(16)
    b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    u, rep = solvers.solve_gmres(cfg, b, tol=1e-12, m=20, maxit=20)
    seq = stepping.march(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    assert rep.converged and rel(u, seq) < 1e-10
    ex = W.exact_wave_solution(cfg)
    assert np.sqrt(cfg.h ** 2 * np.sum((u - ex) ** 2, axis=1)).max() < 2e-2


def test_t4a_golden_matches_table_claims():
    g = _golden()
    assert g["paper_iters"]["0.1"] == [3, 3, 3, 3] and g["paper_iters"]["1.0"][:3] == [3, 7, 37]
    assert g["paper_errors"] == [7.17e-3, 1.86e-3, 4.74e-4, 1.20e-4]
    runs = g["runs"]
    for L in W.T4A_LABELS:
        assert runs[f"{L}_0.1"]["iterations"] == 3 and runs[f"{L}_0.1"]["converged"]
    a1 = [runs[f"{L}_1.0"]["iterations"] for L in (32, 64, 128)]
    assert a1 == sorted(a1) and a1[-1] > a1[0] >= 3        # alpha = 1 grows with the mesh (not pinned to 7, 37)
    errs = [runs[f"{L}_0.1"]["error"] for L in W.T4A_LABELS]
    for e0, e1 in zip(errs, errs[1:]):
        assert 1.9 <= math.log2(e0 / e1) <= 2.1               # printed orders 1.9, 2.0, 2.0
    for e, p in zip(errs, g["paper_errors"]):
        assert p / 2 <= e <= p                                # reading x4: a constant factor ~1.6 below print


COUNTS = os.path.join(os.path.dirname(__file__), "golden", "t4a_alpha1_counts.json")


def _alpha1_counts():
    with open(COUNTS) as fh:
        return json.load(fh)


def test_t4a_alpha1_count_not_fixed_in_fp64():
    """Reading x4: at alpha = 1 the GMRES count is not determined by the method in fp64.  Three correct references
    (tools/t4a_alpha1_counts.py, oracle only) -- O1 (time DFT + sparse LU), O2 (alpha-periodic stepping in the DST
    basis) and O2 with the whole GMRES in x87 extended precision -- agree on the first two Arnoldi residuals, then
    stagnate in pairs a few times above tol (the Arnoldi residual of a plateau pair is nearly constant) and cross
    tol at different iterations: L = 64 gives 9 / 7 / 7, L = 128 gives 13 / 9 / 7 (the paper prints 7 and 37).
    The GPU count is therefore pinned to the range of these references, per mesh (test_t4a_gpu_matches_oracle)."""
    g = _alpha1_counts()
    names = ("O1_fp64", "O2_fp64", "O2_longdouble")
    for L in (32, 64, 128):
        runs = [g["runs"][f"{L}_{n}"] for n in names]
        assert all(r["converged"] and r["rel_residual"] <= 1e-10 for r in runs)
        h0 = runs[0]["history"]
        for r in runs[1:]:
            for a, c in zip(r["history"][:2], h0[:2]):        # before the plateau: the same Krylov residuals
                assert abs(a - c) <= 1e-6 * c
        for r in runs:
            h = r["history"]
            assert 1e-10 < h[2] < 1e-7 and h[3] >= 0.97 * h[2]  # iteration 3 lands on a plateau pair above tol
        counts = [r["iterations"] for r in runs]
        if L == 32:
            assert counts == [5, 5, 5]
        else:
            assert max(counts) - min(counts) >= 2, counts     # three correct references, three different counts
    # the golden is the oracle's: O1 and O2 in fp64 re-run live at L = 64 (~15 s) disagree by two iterations
    cfg = W.t4a_config(64, 1.0)
    b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    _, r1 = solvers.solve_gmres(cfg, b, tol=1e-10, m=50, maxit=50)
    _, r2 = solvers.solve_gmres(cfg, b, tol=1e-10, m=50, maxit=50, apply=lambda r: periodic.apply_precond_modal(cfg, r))
    assert (r1.iterations, r2.iterations) == (g["runs"]["64_O1_fp64"]["iterations"], g["runs"]["64_O2_fp64"]["iterations"])


@pytest.mark.gpu
@pytest.mark.parametrize("label,alpha", [(32, 0.1), (64, 0.1), (128, 0.1), (256, 0.1), (32, 1.0), (64, 1.0),
                                         (128, 1.0)])
def test_t4a_gpu_matches_oracle(label, alpha):
    g = _golden()
    run = g["runs"][f"{label}_{alpha}"]
    cfg = W.t4a_config(label, alpha)
    ctx = make_ctx(cfg)
    b = ctx.build_rhs(to_dev(W.initial_u0(cfg)), to_dev(W.initial_v0(cfg)), to_dev(W.source_samples(cfg)))
    u, rep = ctx.solve_gmres(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    assert rep.converged
    if alpha < 1.0:
        assert rep.iterations == run["iterations"]
    else:
        # alpha = 1: not fixed in fp64 (test_t4a_alpha1_count_not_fixed_in_fp64): within the references' range
        refs = [_alpha1_counts()["runs"][f"{label}_{n}"]["iterations"] for n in ("O1_fp64", "O2_fp64", "O2_longdouble")]
        print(f"T4A L={label} alpha=1: GPU {rep.iterations} its, references O1/O2/O2-longdouble {refs}")
        assert min(refs) <= rep.iterations <= max(refs), (rep.iterations, refs)
    ex = W.exact_wave_solution(cfg)
    uh = to_host(u)
    err = np.sqrt(cfg.h ** 2 * np.sum((uh - ex) ** 2, axis=1)).max()
    assert abs(err - run["error"]) <= 1e-6 * run["error"]
    if label <= 64:
        seq = stepping.march(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
        assert rel(uh, seq) < 1e-8
