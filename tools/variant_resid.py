"""Tuning helper: time the all-at-once residual of a config with an alternative libparadiag build (argv: lib config)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx
cfg = W.BY_NAME[sys.argv[2]]
ctx = make_ctx(cfg)
u = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); b = torch.randn_like(u); r = torch.empty_like(u)
for _ in range(3): ctx.residual(b, u, r)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.residual(b, u, r)
e1.record(); torch.cuda.synchronize()
print(os.path.basename(sys.argv[1]), sys.argv[2], "residual ms %.3f" % (e0.elapsed_time(e1) / 10))
