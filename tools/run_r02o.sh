# r02o: bench lines for every config with the current build (cfg4 with the CPU legs)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=${1:-r02o}
for c in cfg0 cfg1 cfg2 cfg3; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${V}_$c.json 2> gpurun_out/bench_${V}_$c.err
done
python bench.py --config cfg4 > gpurun_out/bench_${V}_cfg4.json 2> gpurun_out/bench_${V}_cfg4.err
for c in cfg0 cfg1 cfg2 cfg3 cfg4; do python - <<PY
import json
d=json.loads(open('gpurun_out/bench_${V}_$c.json').read().strip().splitlines()[-1])
print('$c', d['ms_per_step'], d['config']['iterations'], d['apply']['ms'], d['apply']['hbm_frac'], d['roofline']['kernel'], d['roofline']['frac'], d.get('e2e',{}) and d['e2e']['ms_per_step'], d['tail_form'] and d['tail_form']['ms_per_step'], d.get('clocks'))
PY
done
