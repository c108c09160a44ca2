import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads as W
from tests.helpers import make_ctx
cfg = W.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "cfg4"]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda")
z = torch.empty_like(r)
for _ in range(3): ctx.apply_precond(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); n = 10
for _ in range(n): ctx.apply_precond(r, z)
e1.record(); torch.cuda.synchronize()
print(cfg.name, "env", {k: os.environ.get(k) for k in ("PD_GRAPH", "PD_TF4_CHUNK_MB", "PD_SLAB_CHUNK_MB")}, "apply ms", e0.elapsed_time(e1) / n)
