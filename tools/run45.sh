source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest45.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest45.log
for L in 256 128; do python - <<PY
import sys, time, torch; sys.path.insert(0, ".")
import workloads as W
from tests.helpers import make_ctx, to_dev
cfg = W.t4a_config($L, 0.1)
ctx = make_ctx(cfg)
b = ctx.build_rhs(to_dev(W.initial_u0(cfg)), to_dev(W.initial_v0(cfg)), to_dev(W.source_samples(cfg)))
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u, rep = ctx.solve_gmres(b, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
print("t4a", $L, "its", rep.iterations, "solve ms %.3f" % (dt * 1e3), "dofs", cfg.D)
ctx.enable_phase_timing(True); r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for i in range(5): ctx.apply_precond(r, z)
torch.cuda.synchronize(); ms, n = ctx.phase_times(); print("phases", [round(ms[i] / max(n[i], 1), 4) for i in range(3)])
PY
done
