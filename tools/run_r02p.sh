# r02p: GMRES final assembly from the stored Z_j (parity + bench cfg1/3/4)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_guard.py -m gpu -x -q -k "gmres or cfg4 or cfg3 or cfg1 or solve or guard or dist" > gpurun_out/r02p_tests.log 2>&1; tail -n 3 gpurun_out/r02p_tests.log
for c in cfg1 cfg3; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02p_$c.json 2> gpurun_out/bench_r02p_$c.err; done
python bench.py --config cfg4 --no-cpu-baseline > gpurun_out/bench_r02p_cfg4.json 2> gpurun_out/bench_r02p_cfg4.err
PD_GMRES_NO_Z=1 python bench.py --config cfg4 --no-cpu-baseline --no-e2e > gpurun_out/bench_r02p_cfg4_noz.json 2> gpurun_out/bench_r02p_cfg4_noz.err
for f in cfg1 cfg3 cfg4 cfg4_noz; do python - <<PY
import json
d=json.loads(open('gpurun_out/bench_r02p_$f.json').read().strip().splitlines()[-1])
print('$f', d['ms_per_step'], d['config']['iterations'], d['apply']['ms'], d['roofline']['kernel'], d['roofline']['frac'], d.get('e2e') and d['e2e']['ms_per_step'], {k:(v['ms_per_call'],v['calls']) for k,v in d['phases'].items()})
PY
done
