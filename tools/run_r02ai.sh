# r02ai: CUDA graphs from a triple's second use at launch-bound sizes (default): tests that reuse contexts / buffers, then
# bench lines cfg0-cfg3
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02ai_gpu_tests.log 2>&1; tail -n 3 gpurun_out/r02ai_gpu_tests.log
for c in cfg0 cfg1 cfg2 cfg3; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02ai_bench_$c.json 2> gpurun_out/r02ai_bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/r02ai_bench_$c.json')); print('$c', d['ms_per_step'], d['config'].get('iterations'), '%.4g' % d['value'], 'apply', d['apply']['ms'], d['apply']['hbm_frac'], 'e2e', d['e2e']['ms_per_step'], 'tail', d.get('tail_form',{}).get('ms_per_step'))"; done | tee gpurun_out/r02ai_bench_summary.txt
