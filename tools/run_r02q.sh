# r02q: ||b|| fused into the first GMRES apply: parity + cfg4 bench
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gmres or cfg4 or zero" > gpurun_out/r02q_tests.log 2>&1; tail -n 3 gpurun_out/r02q_tests.log
python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_r02q_cfg4.json 2> gpurun_out/bench_r02q_cfg4.err
python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02q_cfg3.json 2> gpurun_out/bench_r02q_cfg3.err
for f in cfg4 cfg3; do python - <<PY
import json
d=json.loads(open('gpurun_out/bench_r02q_$f.json').read().strip().splitlines()[-1])
print('$f', d['ms_per_step'], d['config']['iterations'], d['apply']['ms'], d['roofline']['kernel'], d['roofline']['frac'], d.get('e2e') and d['e2e']['ms_per_step'], {k:(v['ms_per_call'],v['calls']) for k,v in d['phases'].items()})
PY
done
