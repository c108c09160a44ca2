# r02ae: GMRES head fix fused into the mode-4 sweep: GMRES parity subset, bench lines cfg1 / cfg3 / cfg4
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "gmres or solve_full or dist" > gpurun_out/r02ae_tests.log 2>&1; tail -3 gpurun_out/r02ae_tests.log
for c in cfg1 cfg3 cfg4; do python bench.py --config $c > gpurun_out/r02ae_bench_$c.json 2> gpurun_out/r02ae_bench_$c.err; python -c "
import json,sys; d=json.load(open('gpurun_out/r02ae_bench_$c.json')); print('$c', d['ms_per_step'], d['config'].get('iterations'), d['value'], d['e2e']['ms_per_step'], d['gpu_launches'], {k:(v['ms_per_call'],v['calls']) for k,v in d['phases'].items()})"; done
