import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2005_09158_b200 import _lib
_lib._LIB_PATH = sys.argv[1]
import workloads as W
from tests.helpers import make_ctx
for name in ["cfg4", "cfg2"]:
    cfg = W.BY_NAME[name]
    ctx = make_ctx(cfg)
    u = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); b = torch.randn_like(u); r = torch.empty_like(u)
    for _ in range(3): ctx.residual(b, u, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ctx.residual(b, u, r)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(os.path.basename(sys.argv[1]), name, "residual ms %.3f  GB/s %.0f" % (ms, 24 * cfg.D / ms / 1e6))
    del ctx, u, b, r
    torch.cuda.empty_cache()
