"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test pins an oracle function to something other than itself: the printed Lemma 1 factorisation,
closed forms, brute-force dense assembly, theorems of the paper, textbook eigenpairs, sequential
time stepping, the SPEC worked example.  A plausible mistake in the oracle (dropped term, wrong sign
or index, transposed operand, wrong Gamma exponent, wrong DFT normalisation) fails at least one.
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import workloads as W
from oracle import dense, periodic, problems, solvers, spectral, stepping, tail

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rel(a, b):
    return np.linalg.norm(np.ravel(a - b)) / np.linalg.norm(np.ravel(b))


def tiny(op, scheme, nx=7, nt=8, alpha=0.05, **kw):
    base = {W.ADE1D: W.CONFIGS[0], W.WAVE1D: W.CONFIGS[2], W.ADE2D: W.CONFIGS[3]}[op]
    if op == W.ADE2D:
        return base.scaled(nx=nx, ny=nx, nt=nt, scheme=scheme, alpha=alpha, **kw)
    return base.scaled(nx=nx, nt=nt, scheme=scheme, alpha=alpha, **kw)


CASES = [(W.ADE1D, W.BE), (W.ADE1D, W.CN), (W.WAVE1D, W.LF), (W.ADE2D, W.BE), (W.ADE2D, W.CN)]


# ----------------------------------------------------------------------------- Lemma 1 / spectra
@pytest.mark.parametrize("nt,alpha", [(1, 0.3), (2, 0.25), (5, 0.3), (8, 1e-2), (16, 1e-3)])
def test_lemma1_factorisation_as_printed(nt, alpha):
    """C = V D V^{-1}, V = Gamma^{-1} F^*, D = diag(sqrt(Nt) F Gamma c), F_{l1,l2} = omega^{(l1-1)(l2-1)}/sqrt(Nt),
    omega = e^{2 pi i/Nt} (P:l.155-174), built literally, vs the dense alpha-circulant."""
    rng = np.random.default_rng(nt)
    c = rng.standard_normal(nt)
    C = problems.alpha_circulant(c, alpha)
    l = np.arange(nt)
    F = np.exp(2j * math.pi * np.outer(l, l) / nt) / math.sqrt(nt)
    G = np.diag(alpha ** (l / nt))
    V = np.linalg.inv(G) @ F.conj().T
    D = np.diag(math.sqrt(nt) * F @ G @ c)
    assert rel(V @ D @ np.linalg.inv(V), C) < 1e-13
    # the oracle's (numpy-convention) spectrum is the same multiset, index n -> -n (reading c1)
    lam = spectral.column_spectrum(c, alpha)
    assert np.allclose(lam[(-l) % nt], np.diag(D), rtol=1e-12, atol=1e-12 * np.abs(lam).max())


def test_spec_worked_example_golden():
    vals = {}
    with open(os.path.join(GOLDEN, "spec_alpha_circulant_2x2.txt")) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, *v = line.split()
                vals[k] = [float(x) for x in v]
    lam = spectral.column_spectrum(np.array(vals["column"]), vals["alpha"][0])
    assert np.allclose(sorted(lam.real), sorted(vals["eigenvalues"]), atol=1e-14)
    assert np.abs(lam.imag).max() < 1e-14


@pytest.mark.parametrize("scheme", [W.BE, W.CN, W.LF])
@pytest.mark.parametrize("nt", [2, 3, 8, 64])
def test_spectra_closed_forms(scheme, nt):
    """lambda from the DFT of Gamma-weighted first columns (P:l.860-864) = closed forms of SURVEY §8(c):
    z_n = alpha^{1/Nt} e^{-2 pi i n/Nt}; BE (1-z)/dt, 1; CN (1-z)/dt, (1+z)/2; LF (1-z)^2/dt^2, (1+z^2)/2."""
    if scheme == W.LF and nt < 3:
        pytest.skip("leapfrog needs Nt >= 3 for the full stencil")
    cfg = W.CONFIGS[2 if scheme == W.LF else 0].scaled(nt=nt, scheme=scheme, alpha=0.07)
    l1, l2 = spectral.spectra(cfg)
    z = cfg.alpha ** (1.0 / nt) * np.exp(-2j * math.pi * np.arange(nt) / nt)
    dt = cfg.dt
    if scheme == W.BE:
        e1, e2 = (1 - z) / dt, np.ones(nt)
    elif scheme == W.CN:
        e1, e2 = (1 - z) / dt, (1 + z) / 2
    else:
        e1, e2 = (1 - z) ** 2 / dt ** 2, (1 + z ** 2) / 2
    assert np.allclose(l1, e1, rtol=1e-12, atol=1e-12 * np.abs(e1).max())
    assert np.allclose(l2, e2, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("scheme", [W.BE, W.CN, W.LF])
def test_spectra_are_dense_eigenvalues(scheme):
    cfg = W.CONFIGS[2 if scheme == W.LF else 0].scaled(nt=12, scheme=scheme, alpha=0.2)
    c1, c2 = problems.time_first_columns(cfg)
    for c, lam in zip((c1, c2), spectral.spectra(cfg)):
        ev = np.linalg.eigvals(problems.alpha_circulant(c, cfg.alpha))
        for x in lam:
            assert np.abs(ev - x).min() < 1e-9 * max(1.0, abs(x))


def test_corner_entries_as_printed():
    """eq 2.11b (P:l.789-801) and eq 3.4 (P:l.1262-1275) corner entries."""
    a = 0.37
    cfg = W.CONFIGS[1].scaled(nt=6, alpha=a)                      # CN, theta = 1/2
    c1, c2 = problems.time_first_columns(cfg)
    C1, C2 = problems.alpha_circulant(c1, a), problems.alpha_circulant(c2, a)
    dt = cfg.dt
    assert C1[0, -1] == pytest.approx(-a / dt) and C2[0, -1] == pytest.approx(0.5 * a)
    assert np.count_nonzero(np.triu(C1, 1)) == 1 and np.count_nonzero(np.triu(C2, 1)) == 1
    cfg = W.CONFIGS[2].scaled(nt=7, alpha=a)                      # leapfrog
    c1, c2 = problems.time_first_columns(cfg)
    C1, C2 = problems.alpha_circulant(c1, a), problems.alpha_circulant(c2, a)
    dt2 = cfg.dt ** 2
    assert C1[0, -2] * dt2 == pytest.approx(a) and C1[0, -1] * dt2 == pytest.approx(-2 * a)
    assert C1[1, -1] * dt2 == pytest.approx(a)
    assert C2[0, -2] == pytest.approx(a / 2) and C2[0, -1] == 0 and C2[1, -1] == pytest.approx(a / 2)
    assert np.count_nonzero(np.triu(C1, 1)) == 3 and np.count_nonzero(np.triu(C2, 1)) == 2


@pytest.mark.parametrize("alpha", [1.0, 0.1, 1e-2, 1e-4])
def test_cond_V_bound(alpha):
    """Cond_2(V) <= 1/alpha (eq 2.13, P:l.823-826)."""
    nt = 32
    l = np.arange(nt)
    F = np.exp(2j * math.pi * np.outer(l, l) / nt) / math.sqrt(nt)
    V = np.diag(alpha ** (-l / nt)) @ F.conj().T
    assert np.linalg.cond(V) <= 1.0 / alpha * (1 + 1e-12)
    assert np.linalg.cond(V) == pytest.approx(alpha ** (-(nt - 1) / nt), rel=1e-10)


def test_alpha_one_identity_column():
    assert np.allclose(spectral.column_spectrum(np.eye(8)[0], 1.0), 1.0)


# ----------------------------------------------------------------------------- spatial operator
@pytest.mark.parametrize("domain", [0.0, 1.0])
def test_symbol_2d_matches_stencil(domain):
    """kappa (reading c14) reproduces the sparse periodic stencil K on random data (ax != ay catches a transpose),
    on [0, 2pi) (configs 3-4) and (0, 1) (Table ctp-01)."""
    cfg = W.CONFIGS[3].scaled(nx=8, ny=8, nu=0.3, ax=1.0, ay=-0.4, domain=domain)
    n = cfg.nx
    u = np.random.default_rng(1).standard_normal(n * n)
    Ku = problems.K_matrix(cfg) @ u
    Fn, Fi = spectral.dft_matrix(n, -1), spectral.dft_matrix(n, +1)
    uh = Fn @ u.reshape(n, n) @ Fn.T
    Ku2 = (Fi @ (spectral.symbol_2d(cfg) * uh) @ Fi.T).real.reshape(-1) / n ** 2
    assert rel(Ku2, Ku) < 1e-13
    # the centred stencil itself on the domain's spacing h = length / N
    h = cfg.h
    K = problems.K_matrix(cfg).toarray()
    assert K[1, 0] == pytest.approx(-0.3 / h ** 2 - 1.0 / (2 * h)) and K[1, 1] == pytest.approx(4 * 0.3 / h ** 2)


def test_1d_operators_stencil():
    cfg = W.CONFIGS[0]
    K = problems.K_matrix(cfg).toarray()
    h = 1 / 64
    assert K[5, 4] == pytest.approx(-0.01 / h ** 2 - 1 / (2 * h))
    assert K[5, 5] == pytest.approx(0.02 / h ** 2)
    assert K[5, 6] == pytest.approx(-0.01 / h ** 2 + 1 / (2 * h))
    # wave: textbook DST-I eigenpairs of the Dirichlet -D2
    cfg = W.CONFIGS[2].scaled(nx=15)
    K = problems.K_matrix(cfg).toarray()
    j = np.arange(1, 16)
    mu = (4 / cfg.h ** 2) * np.sin(math.pi * j / 32) ** 2
    assert np.allclose(np.sort(np.linalg.eigvalsh(K)), np.sort(mu), rtol=1e-12)


# ----------------------------------------------------------------------------- the apply
@pytest.mark.parametrize("op,scheme", CASES)
@pytest.mark.parametrize("nx,nt", [(7, 8), (5, 1), (6, 16), (9, 2)])
def test_apply_O1_equals_dense_O0(op, scheme, nx, nt):
    if scheme == W.LF and nt < 3:
        pytest.skip("leapfrog needs Nt >= 3")
    if op == W.ADE2D:
        nx = min(nx, 6)
    cfg = tiny(op, scheme, nx=nx, nt=nt, alpha=0.03)
    r = np.random.default_rng(nx * 100 + nt).standard_normal((nt, cfg.S))
    z0 = dense.apply_precond(cfg, r)
    assert rel(spectral.apply_precond(cfg, r), z0) < 1e-12
    if nt == 1:
        return  # alpha-periodic stepping needs the wrap entry, absent from a 1x1 alpha-circulant (S:l.89)
    assert rel(periodic.apply_precond_dense(cfg, r), z0) < 1e-12
    if op != W.ADE1D:
        assert rel(periodic.apply_precond_modal(cfg, r), z0) < 1e-12


@pytest.mark.parametrize("name", ["cfg0", "cfg1s", "cfg2s", "cfg3s"])
def test_apply_O1_equals_O2_medium(name):
    """O1 (DFT in time) vs O2 (alpha-periodic stepping, no time DFT) at config-like sizes."""
    cfg = {"cfg0": W.CONFIGS[0],
           "cfg1s": W.CONFIGS[1].scaled(nx=255, nt=256),
           "cfg2s": W.CONFIGS[2].scaled(nx=511, nt=512),
           "cfg3s": W.CONFIGS[3].scaled(nx=32, ny=32, nt=64)}[name]
    r = W.random_vector(cfg, seed=7)
    z1 = spectral.apply_precond(cfg, r)
    z2 = periodic.apply_precond_modal(cfg, r) if cfg.op != W.ADE1D else periodic.apply_precond_dense(cfg, r)
    assert rel(z1, z2) < 1e-10
    assert rel(problems.matvec_P(cfg, z1), r) < 1e-10


@pytest.mark.slow
def test_wave_rounding_floor_reading_t1():
    """Reading t1: on the config-2 recipe (leapfrog, alpha = 1e-2, T = 2, resonant systems) the two
    fp64 oracles' forward errors against an extended-precision reference (O2 modal in np.longdouble, whose backward
    error ||P_alpha z - r|| / ||r|| in longdouble is 6e-16) are of the size of their mutual distance delta and grow
    with the size, O1 (dense DFT-matrix sums) the most: the fp64 floor, amplified by Cond_2(V) <= 1/alpha (eq 2.13),
    not a defect of either oracle.  Measured: 1023 x 1024 delta 2.0e-11, O1 2.0e-11, O2 4.1e-12; 2047 x 2048 delta
    8.7e-11, O1 1.0e-10, O2 3.0e-11; full config 2 delta 4.8e-10."""
    cfg = W.CONFIGS[2].scaled(nx=1023, nt=1024)
    r = W.random_vector(cfg, seed=7)
    z1 = spectral.apply_precond(cfg, r)
    z2 = periodic.apply_precond_modal(cfg, r)
    zl = periodic.apply_precond_modal(cfg, r, precision=np.longdouble)
    c1, c2 = problems.time_first_columns(cfg)
    pz = problems.apply_time(c1, zl, cfg.alpha) + problems.apply_K(cfg, problems.apply_time(c2, zl, cfg.alpha))
    assert float(np.linalg.norm(pz - r) / np.linalg.norm(r)) < 1e-14    # measured 6.4e-16 (|K| ~ 4/h^2 = 4e6)
    delta = rel(z1, z2)
    e1, e2 = float(rel(z1, zl)), float(rel(z2, zl))
    assert 1e-12 < delta < 1e-10
    assert e2 < e1 <= 2 * delta and delta <= e1 + e2


def test_apply_special_cases():
    cfg = tiny(W.ADE1D, W.BE, nx=9, nt=1)
    r = np.random.default_rng(3).standard_normal((1, 9))
    K = problems.K_matrix(cfg)
    direct = spla.spsolve(sp.csc_matrix(sp.identity(9) / cfg.dt + K), r[0])
    assert rel(spectral.apply_precond(cfg, r)[0], direct) < 1e-13      # Nt=1: one plain solve (S:l.89)
    assert np.all(spectral.apply_precond(cfg.scaled(nt=8), np.zeros((8, 9))) == 0)


def test_step_b_banded_vs_dense():
    cfg = W.CONFIGS[2].scaled(nx=31, nt=16)
    lam1, lam2 = spectral.spectra(cfg)
    S1 = np.random.default_rng(5).standard_normal((16, 31)) + 1j
    S2 = spectral.step_b(cfg, S1, lam1, lam2)
    K = problems.K_matrix(cfg).toarray()
    for n in range(16):
        assert rel(S2[n], np.linalg.solve(lam1[n] * np.eye(31) + lam2[n] * K, S1[n])) < 1e-12


@pytest.mark.parametrize("op,scheme", CASES)
def test_matvecs_equal_dense(op, scheme):
    cfg = tiny(op, scheme, nx=5, nt=7)
    u = np.random.default_rng(11).standard_normal((7, cfg.S))
    assert rel(problems.matvec_A(cfg, u), (dense.assemble_A(cfg) @ u.reshape(-1)).reshape(u.shape)) < 1e-14
    assert rel(problems.matvec_P(cfg, u), (dense.assemble_P(cfg) @ u.reshape(-1)).reshape(u.shape)) < 1e-14


# ----------------------------------------------------------------------------- right-hand side / stepping
@pytest.mark.parametrize("op,scheme", CASES)
def test_rhs_consistent_with_physical_stepping(op, scheme):
    """A (march from U0, V0, f) = b: the all-at-once b reproduces the sequential scheme (eq 2.4, 2.5b; reading c4, c5)."""
    cfg = tiny(op, scheme, nx=9 if op != W.ADE2D else 6, nt=10)
    rng = np.random.default_rng(2)
    u0, v0 = rng.standard_normal(cfg.S), rng.standard_normal(cfg.S)
    f = rng.standard_normal((cfg.nt + 1, cfg.S))
    b = problems.rhs(cfg, u0, v0, f)
    um = stepping.march(cfg, u0, v0, f)
    assert rel(problems.matvec_A(cfg, um), b) < 1e-12
    assert rel(stepping.solve_all_at_once(cfg, b), um) < 1e-12
    assert rel(dense.solve_A(cfg, b), um) < 1e-12


def test_leapfrog_rhs_second_order():
    """Reading c4 pinned by second-order convergence to u = sin(pi x) e^t (1D analogue of P:l.1311-1314)."""
    errs = []
    for nx in (15, 31, 63):
        cfg = W.Config("lfx", W.WAVE1D, nx=nx, ny=1, nt=nx + 1, T=2.0, scheme=W.LF, alpha=0.1,
                       init="exact_wave", source="exact_wave")
        b = problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
        u = stepping.solve_all_at_once(cfg, b)
        ex = W.exact_wave_solution(cfg)
        errs.append(max(math.sqrt(cfg.h) * np.linalg.norm(u[n] - ex[n]) for n in range(cfg.nt)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(1.85 < o < 2.15 for o in orders), (errs, orders)


# ----------------------------------------------------------------------------- theorems
@pytest.mark.parametrize("scheme", [W.BE, W.CN])
def test_error_propagation_eigenvalues_theta(scheme):
    """Non-zero eigenvalues of I - P^{-1}A are -alpha R^Nt/(1 - alpha R^Nt), R the stability function at dt*mu
    (mode-wise form of Thm 1.2 / Thm 5.1, P:l.830-846, 1598-1617); |.| <= alpha/(1-alpha)."""
    cfg = tiny(W.ADE1D, scheme, nx=8, nt=10, alpha=0.05)
    E = np.eye(80) - np.linalg.solve(dense.assemble_P(cfg), dense.assemble_A(cfg))
    ev = np.linalg.eigvals(E)
    mu = np.linalg.eigvals(problems.K_matrix(cfg).toarray())
    th = problems.theta_of(scheme)
    R = (1 - (1 - th) * cfg.dt * mu) / (1 + th * cfg.dt * mu)
    pred = -cfg.alpha * R ** cfg.nt / (1 - cfg.alpha * R ** cfg.nt)
    big = ev[np.abs(ev) > 1e-10]
    assert len(big) == len(pred)
    for p in pred:
        assert np.abs(big - p).min() < 1e-9 * max(abs(p), 1e-3)
    assert np.abs(ev).max() <= cfg.alpha / (1 - cfg.alpha) + 1e-12


def test_theorem_3_1_leapfrog_spectrum():
    """sigma(P^{-1}A) = (Nt-2)Nx ones U {1/(1 - alpha e^{+-i Nt theta_j})}, theta_j = arctan sqrt(lambda_j^2-1),
    lambda_j eig of D = I + dt^2 A/2 (Thm 3.1, P:l.1282-1308); annulus alpha/(1+alpha) <= |z-1| <= alpha/(1-alpha)."""
    cfg = tiny(W.WAVE1D, W.LF, nx=8, nt=8, alpha=0.3)
    M = np.linalg.solve(dense.assemble_P(cfg), dense.assemble_A(cfg))
    ev = np.linalg.eigvals(M)
    lamD = np.linalg.eigvalsh(np.eye(8) + cfg.dt ** 2 * problems.K_matrix(cfg).toarray() / 2)
    thj = np.arctan(np.sqrt(lamD ** 2 - 1))
    pred = np.concatenate([1 / (1 - cfg.alpha * np.exp(1j * cfg.nt * thj)),
                           1 / (1 - cfg.alpha * np.exp(-1j * cfg.nt * thj))])
    ones = np.abs(ev - 1) < 1e-6
    assert ones.sum() == (cfg.nt - 2) * cfg.nx
    rest = ev[~ones]
    for p in pred:
        assert np.abs(rest - p).min() < 1e-8
    d = np.abs(rest - 1)
    a = cfg.alpha
    assert d.min() >= a / (1 + a) - 1e-12 and d.max() <= a / (1 - a) + 1e-12


def test_gmres_finite_termination():
    """rank(P_alpha - A) <= Nx (theta-method) => right-preconditioned GMRES terminates in <= Nx+1 steps."""
    cfg = tiny(W.ADE1D, W.CN, nx=5, nt=12, alpha=0.5)
    P, A = dense.assemble_P(cfg), dense.assemble_A(cfg)
    assert np.linalg.matrix_rank(P - A) <= cfg.nx
    b = np.random.default_rng(0).standard_normal((12, 5))
    u, rep = solvers.solve_gmres(cfg, b, tol=1e-13, m=100, maxit=100)
    assert rep.converged and rep.iterations <= cfg.nx + 1
    assert rel(u, dense.solve_A(cfg, b)) < 1e-11


# ----------------------------------------------------------------------------- solvers
def _problem(cfg):
    return problems.rhs(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))


@pytest.mark.parametrize("name,solver,expect", [
    ("cfg0", "stationary", 3), ("cfg0", "gmres", 3),
    ("cfg1s", "gmres", None), ("cfg2s", "stationary", None), ("cfg3s", "gmres", None)])
def test_converged_solution_equals_sequential(name, solver, expect):
    """The converged all-at-once solution equals step-by-step time stepping (P:l.76-80)."""
    cfg = {"cfg0": W.CONFIGS[0],
           "cfg1s": W.CONFIGS[1].scaled(nx=255, nt=256),
           "cfg2s": W.CONFIGS[2].scaled(nx=255, nt=256),
           "cfg3s": W.CONFIGS[3].scaled(nx=16, ny=16, nt=32)}[name]
    b = _problem(cfg)
    fn = solvers.solve_stationary if solver == "stationary" else solvers.solve_gmres
    u, rep = fn(cfg, b)
    assert rep.converged
    if expect is not None:
        assert rep.iterations == expect
    seq = stepping.march(cfg, W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg))
    assert rel(u, seq) < 1e-8
    # contraction per stationary iteration bounded by alpha/(1-alpha) (Thm 5.1 / eq 5.2)
    if solver == "stationary":
        h = rep.history
        for i in range(1, len(h)):
            if h[i - 1] > 1e-13:
                assert h[i] / h[i - 1] <= 1.5 * cfg.alpha / (1 - cfg.alpha) + 1e-3


@pytest.mark.parametrize("cfg", [W.CONFIGS[4].scaled(nx=32, ny=32, nt=64), W.CONFIGS[3].scaled(nx=16, ny=16, nt=32),
                                 W.ctp01_config(W.CN, 1e-2, nx=32, ny=32, nt=16)], ids=["cfg4s", "cfg3s", "ctp01s"])
def test_march_fourier_equals_sparse_march(cfg):
    """stepping.march_fourier (eq 2.4 per 2D Fourier mode, used at config-4 size) = stepping.march (sparse LU per
    step), with and without a source; and a single mode e_k decays by the scalar amplification factor."""
    u0 = W.initial_u0(cfg)
    f = np.random.default_rng(1).standard_normal((cfg.nt + 1, cfg.S))
    assert rel(stepping.march_fourier(cfg, u0), stepping.march(cfg, u0)) < 1e-13
    assert rel(stepping.march_fourier(cfg, u0, f), stepping.march(cfg, u0, None, f)) < 1e-13
    X, Y = W.grid(cfg)
    n, kx, ky = cfg.nx, 3, 1
    th = problems.theta_of(cfg.scheme)
    kap = spectral.symbol_2d(cfg)[ky, kx]
    g = (1 / cfg.dt - (1 - th) * kap) / (1 / cfg.dt + th * kap)
    mode = np.exp(2j * math.pi / cfg.length * (kx * X + ky * Y)).reshape(-1)
    u = stepping.march_fourier(cfg, mode.real)  # Re e_k = (e_k + e_-k)/2, kappa(-k) = conj kappa(k)
    ex = np.real(g ** np.arange(1, cfg.nt + 1)[:, None] * mode[None, :])
    assert rel(u, ex) < 1e-12


def test_residual_definitions():
    cfg = tiny(W.ADE1D, W.CN, nx=9, nt=6)
    b = np.random.default_rng(4).standard_normal((6, 9))
    assert np.array_equal(solvers.residual(cfg, b, np.zeros_like(b)), b)
    u = dense.solve_A(cfg, b)
    assert np.linalg.norm(solvers.residual(cfg, b, u)) < 1e-12 * np.linalg.norm(b)


# ------------------------------------------------------------------------------------------ O3 tail form (NEXT-1)
TAIL_CASES = [W.CONFIGS[0], W.CONFIGS[1].scaled(nx=63, nt=64), W.CONFIGS[2].scaled(nx=31, nt=32),
              W.CONFIGS[3].scaled(nx=16, ny=16, nt=16)]


@pytest.mark.parametrize("cfg", TAIL_CASES, ids=lambda c: f"{c.op}-{c.scheme}")
def test_tail_corner_is_P_minus_A(cfg):
    """head_from_tail reproduces P_alpha - A from the plain matvecs (eq 1.1 vs eq 1.2): non-zero only in the first
    H block rows, and there a function of the last H blocks only (H = 1 theta, 2 leapfrog)."""
    H = tail.head_blocks(cfg)
    assert H == (2 if cfg.scheme == W.LF else 1)
    u = np.random.default_rng(1).standard_normal((cfg.nt, cfg.S))
    d = problems.matvec_P(cfg, u) - problems.matvec_A(cfg, u)
    assert np.abs(d[H:]).max() == 0.0
    assert rel(tail.head_from_tail(cfg, u[cfg.nt - H:]), d[:H]) < 1e-12


@pytest.mark.parametrize("cfg", TAIL_CASES, ids=lambda c: f"{c.op}-{c.scheme}")
def test_tail_map_equals_last_blocks_of_full_apply(cfg):
    """Economical Step (a) + truncated Step (c) (P:l.928-931) == last H blocks of O1 on the embedded vector."""
    H = tail.head_blocks(cfg)
    g = np.random.default_rng(2).standard_normal((H, cfg.S))
    v = np.zeros((cfg.nt, cfg.S))
    v[:H] = g
    # both sides carry fp64 rounding amplified by up to Cond_2(V) <= 1/alpha (eq 2.13, reading t1)
    assert rel(tail.tail_map(cfg, g), spectral.apply_precond(cfg, v)[cfg.nt - H:]) < max(1e-10, 1e-12 / cfg.alpha)


@pytest.mark.parametrize("cfg", TAIL_CASES, ids=lambda c: f"{c.op}-{c.scheme}")
def test_tail_solvers_same_iterates(cfg):
    """[V6]: the tail-form stationary iteration and GMRES take the same number of iterations and return the same
    u as the residual-form oracle solvers, for a head-supported b, a full-support b, a non-zero u0 and restarts."""
    rng = np.random.default_rng(3)
    b = problems.rhs(cfg, rng.standard_normal(cfg.S), rng.standard_normal(cfg.S) if cfg.scheme == W.LF else None)
    u1, r1 = solvers.solve_stationary(cfg, b, tol=1e-10, maxit=30)
    u2, r2 = tail.solve_stationary_tail(cfg, b, tol=1e-10, maxit=30)
    assert (r1.iterations, r1.converged) == (r2.iterations, r2.converged)
    assert rel(u2, u1) < 1e-11
    bb = rng.standard_normal((cfg.nt, cfg.S))
    u0 = rng.standard_normal((cfg.nt, cfg.S))
    u1, r1 = solvers.solve_stationary(cfg, bb, u0=u0, tol=1e-10, maxit=40)
    u2, r2 = tail.solve_stationary_tail(cfg, bb, u0=u0, tol=1e-10, maxit=40)
    assert r1.iterations == r2.iterations and rel(u2, u1) < 1e-11
    for rhs_, m in ((b, 5), (bb, 3)):
        u1, r1 = solvers.solve_gmres(cfg, rhs_, tol=1e-10, m=m, maxit=40)
        u2, r2 = tail.solve_gmres_tail(cfg, rhs_, tol=1e-10, m=m, maxit=40)
        assert (r1.iterations, r1.converged) == (r2.iterations, r2.converged)
        assert rel(u2, u1) < 1e-11
