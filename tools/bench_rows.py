"""Measurement of the SURVEY 8(f) rows on one B200 (CUDA events on the context stream, after warm-up):
NEXT-1 tail form vs residual form on configs 0-4, NEXT-2 Table ctp-01, NEXT-3 Table T4A, NEXT-4 simplified Newton.
Writes one JSON document (argv[1], default profiles/r01_next_rows.json).  Inputs are resident in HBM."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from tests.helpers import make_ctx, to_dev  # noqa: E402

PH = ["tfft_fwd", "spatial_solve", "tfft_inv", "residual", "tfft_inv_update", "matvec", "krylov_blas1", "residual_norm"]


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        out = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def apply_phases(ctx, reps=10):
    r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda")
    z = torch.empty_like(r)
    for _ in range(2):
        ctx.apply_precond(r, z)
    ctx.enable_phase_timing(True)
    for _ in range(reps):
        ctx.apply_precond(r, z)
    torch.cuda.synchronize()
    ms, n = ctx.phase_times()
    ctx.enable_phase_timing(False)
    ams, _ = timed(lambda: ctx.apply_precond(r, z), reps=reps)
    return {"apply_ms": round(ams, 4), **{PH[i]: round(ms[i] / n[i], 4) for i in range(3) if n[i]}}


def rhs_of(ctx, cfg):
    f = W.source_samples(cfg)
    return ctx.build_rhs(to_dev(W.initial_u0(cfg)), to_dev(W.initial_v0(cfg)), None if f is None else to_dev(f))


out = {"device": torch.cuda.get_device_name(0), "tail_form": {}, "ctp01": {}, "t4a": {}, "newton": {}}

# NEXT-1: both forms of each config's own solver
for cfg in W.CONFIGS:
    ctx = make_ctx(cfg)
    b = rhs_of(ctx, cfg)
    rows = {}
    for form in ("residual", "tail"):
        if cfg.solver == "stationary":
            fn = ctx.solve_stationary if form == "residual" else ctx.solve_stationary_tail
            call = lambda fn=fn: fn(b, tol=cfg.tol, maxit=cfg.maxit)
        else:
            fn = ctx.solve_gmres if form == "residual" else ctx.solve_gmres_tail
            call = lambda fn=fn: fn(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
        ms, (u, rep) = timed(call, reps=3 if cfg.name == "cfg4" else 5)
        rows[form] = {"ms": round(ms, 4), "iterations": rep.iterations, "rel_residual": rep.rel_residual,
                      "dofs_per_s": cfg.D / (ms / 1e3)}
    rows["speedup"] = round(rows["residual"]["ms"] / rows["tail"]["ms"], 3)
    out["tail_form"][cfg.name] = rows
    print(cfg.name, rows, flush=True)
    del ctx, b
    torch.cuda.empty_cache()

# NEXT-2: Table ctp-01 (stationary, both forms)
for s in (W.BE, W.CN):
    for nu in W.CTP01_NUS:
        cfg = W.ctp01_config(s, nu)
        ctx = make_ctx(cfg)
        b = rhs_of(ctx, cfg)
        ms, (u, rep) = timed(lambda: ctx.solve_stationary(b, tol=cfg.tol, maxit=cfg.maxit))
        mst, (u, rept) = timed(lambda: ctx.solve_stationary_tail(b, tol=cfg.tol, maxit=cfg.maxit))
        out["ctp01"][f"{s}_{nu}"] = {"iterations": rep.iterations, "ms": round(ms, 4), "tail_ms": round(mst, 4),
                                     "paper_iterations": W.CTP01_COUNTS[s][list(W.CTP01_NUS).index(nu)]}
    out["ctp01"][f"{s}_phases"] = apply_phases(ctx)
    print("ctp01", s, {k: v for k, v in out["ctp01"].items() if k.startswith(s)}, flush=True)

# NEXT-3: Table T4A (GMRES, alpha = 0.1 and 1)
for L in W.T4A_LABELS:
    for alpha in (0.1, 1.0):
        cfg = W.t4a_config(L, alpha)
        ctx = make_ctx(cfg)
        b = rhs_of(ctx, cfg)
        ms, (u, rep) = timed(lambda: ctx.solve_gmres(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit))
        rec = {"iterations": rep.iterations, "converged": rep.converged, "ms": round(ms, 4), "dofs": cfg.D}
        if alpha == 0.1:
            rec["phases"] = apply_phases(ctx)
            # Step (b) moves the half spectrum once in and once out, 2 F S 16 B (the DST kernels' own
            # row / column / row passes are implementation traffic, not algorithmic bytes)
            rec["spatial_GBps"] = round(2 * (cfg.nt // 2 + 1) * cfg.S * 16 / (rec["phases"]["spatial_solve"] / 1e3) / 1e9, 1)
        out["t4a"][f"{L}_{alpha}"] = rec
        print("t4a", L, alpha, rec, flush=True)
        del ctx, b
        torch.cuda.empty_cache()

# NEXT-4: simplified Newton
for nx, nt in ((1023, 1024), (4095, 1024)):
    cfg = W.nl_config(nx=nx, nt=nt)
    ctx = make_ctx(cfg)
    ctx.set_reaction(*W.NL_REACTION)
    b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
    ms, (u, rep) = timed(lambda: ctx.solve_newton(b, tol=cfg.tol, maxit=cfg.maxit), reps=3)
    out["newton"][f"{nx}x{nt}"] = {"iterations": rep.iterations, "ms": round(ms, 4), "dofs": cfg.D,
                                   "ms_per_iteration": round(ms / max(rep.iterations, 1), 4)}
    print("newton", nx, nt, out["newton"][f"{nx}x{nt}"], flush=True)

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                          "profiles", "r02_next_rows.json")
with open(path, "w") as fh:
    json.dump(out, fh, indent=1)
