timeout 1800 python -m pytest tests/test_gpu_tail.py -q -x -k "rejects" > gpurun_out/pytest34.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest34.log
cat > /tmp/tb.py <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import workloads as W
from tests.helpers import make_ctx, to_dev
for name in ["cfg4", "cfg3", "cfg2", "cfg1", "cfg0"]:
    cfg = W.BY_NAME[name]
    ctx = make_ctx(cfg)
    u0, v0, f = W.initial_u0(cfg), W.initial_v0(cfg), W.source_samples(cfg)
    b = ctx.build_rhs(to_dev(u0), to_dev(v0), None if f is None else to_dev(f))
    for form in ["residual", "tail"]:
        ts = []
        for rep_i in range(4):
            u = torch.zeros_like(b)
            torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
            if cfg.solver == "stationary":
                fn = ctx.solve_stationary if form == "residual" else ctx.solve_stationary_tail
                u, rep = fn(b, u, tol=cfg.tol, maxit=cfg.maxit)
            else:
                fn = ctx.solve_gmres if form == "residual" else ctx.solve_gmres_tail
                u, rep = fn(b, u, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(name, form, "its", rep.iterations, "res %.2e" % rep.rel_residual, "ms", ["%.3f" % t for t in ts])
    del ctx, b, u
    torch.cuda.empty_cache()
PY
python /tmp/tb.py
