import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx
cfg = W.BY_NAME["cfg2"]
ctx = make_ctx(cfg)
u = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); b = torch.randn_like(u); r = torch.empty_like(u)
for _ in range(3): ctx.residual(b, u, r)
torch.cuda.synchronize()
l0 = ctx.kernel_launches()
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 5): ctx.residual(b, u, r)
torch.cuda.synchronize()
print(os.path.basename(sys.argv[1]), "launches", ctx.kernel_launches() - l0)
