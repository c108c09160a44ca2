# r02ad: GMRES without the last basis vector of a cycle: parity of the GMRES tests, then bench lines cfg1 / cfg3 / cfg4
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_t4a.py tests/test_gpu_dist.py tests/test_gpu_robust.py -m gpu -x -q -k "gmres or solve or cfg4 or t4a or dist or newton" > gpurun_out/r02ad_tests.log 2>&1; tail -5 gpurun_out/r02ad_tests.log
for c in cfg4 cfg3 cfg1; do python bench.py --config $c > gpurun_out/r02ad_bench_$c.json 2> gpurun_out/r02ad_bench_$c.err; python -c "
import json,sys; d=json.load(open('gpurun_out/r02ad_bench_$c.json')); print('$c', d['ms_per_step'], d['config'].get('iterations'), d['value'], d['e2e']['ms_per_step'], {k:(v['ms_per_call'],v['calls']) for k,v in d['phases'].items()})"; done
PD_GMRES_NO_LAZY=1 python bench.py --config cfg4 --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('cfg4 NO_LAZY', d['ms_per_step'])"
