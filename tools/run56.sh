source tools/gpu_preflight.sh
for mb in 1024 256 64 32; do for g in 0 1; do echo "chunk ${mb}MB graph=$g"; PD_TF4_CHUNK_MB=$mb PD_GRAPH=$g python - <<'PY'
import sys, os, torch
sys.path.insert(0, ".")
import workloads as W
from tests.helpers import make_ctx
cfg = W.BY_NAME["cfg4"]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(3): ctx.apply_precond(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.apply_precond(r, z)
e1.record(); torch.cuda.synchronize()
print("  apply ms %.3f  launches/apply %d" % (e0.elapsed_time(e1) / 10, ctx.kernel_launches() // 13))
PY
done; done
