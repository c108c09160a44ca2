"""A/B of the persistent fused time FFT (PD_TFX_PERSIST=1) against the default chunk pipeline: same tiles, so the
outputs agree to rounding; phase times per call (0 = forward, 1 = Step (b), 2 = inverse).  argv: config [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["PD_GRAPH"] = "0"  # the same (r, z) pair runs both modes: no replay of the first one captured
import torch
import workloads as W
from tests.helpers import make_ctx
name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
cfg = W.BY_NAME[name]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda")
out = {}
for mode in ("0", "1", "0", "1"):
    os.environ["PD_TFX_PERSIST"] = mode
    z = torch.empty_like(r)
    for _ in range(2): ctx.apply_precond(r, z)
    torch.cuda.synchronize()
    ctx.enable_phase_timing(True)
    for _ in range(reps): ctx.apply_precond(r, z)
    torch.cuda.synchronize()
    ms, cnt = ctx.phase_times()
    ctx.enable_phase_timing(False)
    print(name, "persist=" + mode, " ".join("%d:%.3f" % (i, ms[i] / max(cnt[i], 1)) for i in range(3)), flush=True)
    out[mode] = z
d = (out["0"] - out["1"]).abs().max().item()
print(name, "max |z_default - z_persist| =", d, "max|z| =", out["0"].abs().max().item())
assert d <= 1e-11 * out["0"].abs().max().item()  # same tiles, separately compiled: rounding-level differences only
