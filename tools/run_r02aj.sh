# r02aj: auto graphs limited to Nt S <= 2^21; single-tile time FFT vs four-step on cfg1 (PD_NO_TF4=1); bench cfg0-3
source tools/gpu_preflight.sh
mkdir -p gpurun_out
cat > /tmp/graph_ab.py <<'P'
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import workloads as W
from tests.helpers import make_ctx
name = sys.argv[1]
cfg = W.BY_NAME[name]
ctx = make_ctx(cfg)
r = torch.randn(ctx.shape, dtype=torch.float64, device="cuda"); z = torch.empty_like(r)
for _ in range(5): ctx.apply_precond(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 200
e0.record()
for _ in range(reps): ctx.apply_precond(r, z)
e1.record(); torch.cuda.synchronize()
print(name, "PD_NO_TF4=" + os.environ.get("PD_NO_TF4", "-"), "PD_GRAPH=" + os.environ.get("PD_GRAPH", "-"), "apply ms %.4f" % (e0.elapsed_time(e1) / reps))
P
for c in cfg1 cfg2; do for t in "" "PD_NO_TF4=1"; do for g in "PD_GRAPH=0" "PD_GRAPH=1"; do env $t $g python /tmp/graph_ab.py $c 2>&1 | tail -1; done; done; done | tee gpurun_out/r02aj_tf4_vs_tile.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "graph or full_config" 2>&1 | tail -2
for c in cfg0 cfg1 cfg2 cfg3; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02aj_bench_$c.json 2> gpurun_out/r02aj_bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02aj_bench_$c.json')); print('$c', d['ms_per_step'], d['config'].get('iterations'), '%.4g' % d['value'], 'apply', d['apply']['ms'], d['apply']['hbm_frac'], 'e2e', d['e2e']['ms_per_step'], 'tail', d.get('tail_form',{}).get('ms_per_step'))"; done | tee gpurun_out/r02aj_bench_summary.txt
