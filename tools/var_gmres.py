import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx, to_dev
cfg = W.BY_NAME["cfg4"]
ctx = make_ctx(cfg)
b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
u = torch.zeros_like(b)
for _ in range(2): u.zero_(); ctx.solve_gmres(b, u, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
torch.cuda.synchronize(); ctx.enable_phase_timing(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True); e0.record()
for _ in range(4): u.zero_(); u, rep = ctx.solve_gmres(b, u, tol=cfg.tol, m=cfg.m, maxit=cfg.maxit)
e1.record(); torch.cuda.synchronize(); ms, n = ctx.phase_times()
print(os.path.basename(sys.argv[1]), "step %.3f" % (e0.elapsed_time(e1) / 4), "blas ms/call %.4f calls %d" % (ms[6] / n[6], n[6]),
      "inv_update ms/call %.4f" % (ms[4] / max(n[4], 1)), "its", rep.iterations, "res %.3e" % rep.rel_residual)
