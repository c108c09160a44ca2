# r02ah: CUDA-graph replay of the apply (PD_GRAPH=1) on the launch-bound configs, apply wall time per call
source tools/gpu_preflight.sh
mkdir -p gpurun_out
cat > /tmp/graph_ab.py <<'P'
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from tests.helpers import make_ctx
name = sys.argv[1]
cfg = W.t4a_config(int(name[4:])) if name.startswith("t4a_") else W.BY_NAME[name]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(5): ctx.apply_precond(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 200 if cfg.nt * cfg.S < 5e7 else 20
e0.record()
for _ in range(reps): ctx.apply_precond(r, z)
e1.record(); torch.cuda.synchronize()
print(name, "PD_GRAPH=" + os.environ.get("PD_GRAPH", "0"), "apply ms %.4f" % (e0.elapsed_time(e1) / reps))
P
for c in cfg0 cfg1 cfg2 cfg3 t4a_256 cfg4; do for g in 0 1; do PD_GRAPH=$g python /tmp/graph_ab.py $c 2>&1 | tail -1; done; done | tee gpurun_out/r02ah_graph.txt
