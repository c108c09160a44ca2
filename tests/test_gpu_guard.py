"""Red-zone checks of every C-ABI entry point that writes caller memory (a stand-in for compute-sanitizer memcheck,
which is closed on this GPU pool: profiles/r02_sanitizer_closed.log).

Each device vector handed to the library is a view into a larger allocation whose leading and trailing red zones
hold a canary bit pattern; after the call the red zones must be bit-identical and the outputs finite.  The sizes are
ragged (odd Nx, non-multiples of the tile widths) so that every kernel's tail handling is exercised, and the vector
starts are offset by one double (8-byte aligned, not 16) in a second pass, which routes the kernels with 16-byte
vector paths through their scalar fallbacks."""
import numpy as np
import pytest

import workloads as W
from tests.helpers import make_ctx

GUARD = 4096  # doubles of red zone on each side
CANARY = np.int64(0x7FF4DEADBEEF0123)  # a signalling-NaN bit pattern no kernel produces


def _guarded(n, misalign, torch):
    buf = torch.full((GUARD + n + GUARD + 1,), 0, dtype=torch.int64, device="cuda")
    buf.fill_(int(CANARY))
    raw = buf.view(torch.float64)
    start = GUARD + (1 if misalign else 0)
    return raw, raw[start:start + n], start


def _check(raw, start, n, torch):
    iv = raw.view(torch.int64)
    lo = iv[:start]
    hi = iv[start + n:]
    assert bool((lo == int(CANARY)).all()), "write below the vector"
    assert bool((hi == int(CANARY)).all()), "write past the vector"
    assert bool(torch.isfinite(raw[start:start + n]).all()), "non-finite output"


CASES = [
    W.BY_NAME["cfg0"],
    W.BY_NAME["cfg1"].scaled(nx=133, nt=1024),           # 1D four-step, odd Nx
    W.BY_NAME["cfg2"].scaled(nx=77, nt=64),              # leapfrog (H = 2)
    W.BY_NAME["cfg0"].scaled(nt=1),                      # Nt = 1
    W.BY_NAME["cfg3"].scaled(nx=32, ny=32, nt=256),      # 2D fused time/x FFT at Nt = 256
    W.BY_NAME["cfg4"].scaled(nx=64, ny=64, nt=1024),     # 2D four-step
    W.BY_NAME["cfg3"].scaled(nx=16, ny=16, nt=8),        # 2D single-tile + slab row passes
    W.t4a_config(32),                                    # 2D Dirichlet DST path
]


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", CASES, ids=lambda c: f"{c.name}-{c.nx}x{c.ny}x{c.nt}")
@pytest.mark.parametrize("misalign", [False, True])
def test_entry_points_stay_inside_caller_vectors(cfg, misalign):
    import torch
    ctx = make_ctx(cfg)
    n = cfg.nt * cfg.S
    rng = np.random.default_rng(7)
    rr, r, rs = _guarded(n, misalign, torch)
    rz, z, zs = _guarded(n, misalign, torch)
    r.copy_(torch.from_numpy(rng.standard_normal(n)))
    R, Z = r.view(cfg.nt, cfg.S), z.view(cfg.nt, cfg.S)
    ctx.apply_precond(R, Z)
    _check(rz, zs, n, torch)
    _check(rr, rs, n, torch)
    ctx.residual(R, Z, Z.clone())  # b - A z into a fresh tensor; then in place into the guarded one
    ctx.matvec(R, Z)
    _check(rz, zs, n, torch)
    if cfg.nt >= 2:
        rb, b, bs = _guarded(n, misalign, torch)
        ru, u, us = _guarded(n, misalign, torch)
        u0 = torch.from_numpy(W.initial_u0(cfg)).cuda()
        v0 = torch.from_numpy(W.initial_v0(cfg)).cuda() if cfg.op in (W.WAVE1D, W.WAVE2D) else None
        f = W.source_samples(cfg)
        ctx.build_rhs(u0, v0, None if f is None else torch.from_numpy(f).cuda(), b.view(cfg.nt, cfg.S))
        _check(rb, bs, n, torch)
        B, U = b.view(cfg.nt, cfg.S), u.view(cfg.nt, cfg.S)
        U.zero_()
        ctx.solve_stationary(B, U, tol=1e-10, maxit=3, raise_on_fail=False)
        _check(ru, us, n, torch)
        ctx.solve_gmres(B, U, tol=1e-10, m=3, maxit=4, raise_on_fail=False)
        _check(ru, us, n, torch)
        ctx.solve_gmres(B, U, tol=1e-10, m=3, maxit=4, raise_on_fail=False, zero_guess=True)
        _check(ru, us, n, torch)
        if cfg.op != W.WAVE2D:
            U.zero_()
            ctx.solve_gmres_tail(B, U, tol=1e-10, m=3, maxit=4, raise_on_fail=False)
            _check(ru, us, n, torch)
        _check(rb, bs, n, torch)
