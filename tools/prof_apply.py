"""Small driver for ncu: one warm-up and `reps` applies + residual + matvec of a config."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from tests.helpers import make_ctx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
cfg = W.BY_NAME[a.config]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
b = torch.randn_like(r)
for _ in range(a.reps + 1):
    ctx.apply_precond(r, z)
    ctx.residual(b, z, r)
    ctx.matvec(z, b)
torch.cuda.synchronize()
print("done", ctx.kernel_launches())
