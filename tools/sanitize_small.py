"""Small end-to-end run of every kernel family for compute-sanitizer: configs 0-1 (recurrence Step (b),
single-tile and four-step time FFTs, stationary and GMRES, tail form), a small 2D periodic four-step with the x-FFT
fold and the y-pass, the 2D Dirichlet DST path, the pivoted 1D Step (b) and a Newton solve; one tool per process."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from tests.helpers import make_ctx, to_dev  # noqa: E402

torch.cuda.set_device(0)


def run(cfg, solve=True, tail=True):
    ctx = make_ctx(cfg)
    r = to_dev(W.random_vector(cfg))
    z = ctx.apply_precond(r)
    ctx.residual(r, z)
    b = ctx.build_rhs(to_dev(W.initial_u0(cfg)), to_dev(W.initial_v0(cfg)) if cfg.op in (W.WAVE1D, W.WAVE2D) else None,
                      None if W.source_samples(cfg) is None else to_dev(W.source_samples(cfg)))
    if solve:
        if cfg.solver == "stationary":
            ctx.solve_stationary(b, tol=cfg.tol, maxit=6, raise_on_fail=False)
            if tail:
                ctx.solve_stationary_tail(b, tol=cfg.tol, maxit=6, raise_on_fail=False)
        else:
            ctx.solve_gmres(b, tol=cfg.tol, m=4, maxit=6, raise_on_fail=False)
            ctx.solve_gmres(b, tol=cfg.tol, m=4, maxit=6, raise_on_fail=False, zero_guess=True)
            if tail:
                ctx.solve_gmres_tail(b, tol=cfg.tol, m=4, maxit=6, raise_on_fail=False)
    torch.cuda.synchronize()
    print("ok", cfg.name, cfg.nx, cfg.ny, cfg.nt, flush=True)


run(W.BY_NAME["cfg0"])
run(W.BY_NAME["cfg1"].scaled(nx=255, nt=1024))
run(W.BY_NAME["cfg2"].scaled(nx=127, nt=256))
run(W.BY_NAME["cfg3"].scaled(nx=64, ny=64, nt=64))
run(W.BY_NAME["cfg4"].scaled(nx=32, ny=32, nt=1024))
run(W.t4a_config(32), tail=False)
os.environ["PD_TRIDIAG_GTSV"] = "1"
run(W.BY_NAME["cfg0"], tail=False)
os.environ.pop("PD_TRIDIAG_GTSV")
cfg = W.nl_config(nx=63, nt=64)
ctx = make_ctx(cfg)
ctx.set_reaction(*W.NL_REACTION)
b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
ctx.solve_newton(b, tol=cfg.tol, maxit=4, raise_on_fail=False)
torch.cuda.synchronize()
print("ok newton", flush=True)
