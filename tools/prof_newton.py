import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from tests.helpers import make_ctx, to_dev
cfg = W.nl_config()
ctx = make_ctx(cfg)
ctx.set_reaction(*W.NL_REACTION)
b = ctx.build_rhs(to_dev(W.initial_u0(cfg)))
u, rep = ctx.solve_newton(b, tol=cfg.tol, maxit=cfg.maxit)
torch.cuda.synchronize()
print("its", rep.iterations)
