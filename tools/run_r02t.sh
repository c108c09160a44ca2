# r02t: GMRES u streamed to the host behind its final assembly (pd_solve_ivp_host): parity + cfg4 e2e
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -m gpu -x -q -k "host or ivp or guard" > gpurun_out/r02t_tests.log 2>&1; tail -n 3 gpurun_out/r02t_tests.log
python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_r02t_cfg4.json 2> gpurun_out/bench_r02t_cfg4.err
python - <<PY
import json
d=json.loads(open('gpurun_out/bench_r02t_cfg4.json').read().strip().splitlines()[-1])
print('cfg4', d['ms_per_step'], d['config']['iterations'], d['apply']['ms'], d['roofline']['frac'], d['e2e'])
PY
