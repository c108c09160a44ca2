# r02ak: the driver's round-end commands on the final tree: build check, smoke, the GPU suite, both bench arms
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=r02ak
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('build + smoke ok')" > gpurun_out/${V}_smoke.log 2>&1; tail -n 1 gpurun_out/${V}_smoke.log
timeout 3000 python -m pytest tests/ -x -q -m gpu > gpurun_out/${V}_gpu_tests.log 2>&1; tail -n 2 gpurun_out/${V}_gpu_tests.log
python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/${V}_bench_reference.json 2> gpurun_out/${V}_bench_reference.err; cut -c1-400 gpurun_out/${V}_bench_reference.json
python bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/${V}_bench_cfg4.json 2> gpurun_out/${V}_bench_cfg4.err
python -c "
import json; d=json.load(open('gpurun_out/${V}_bench_cfg4.json')); print('cfg4', d['ms_per_step'], '%.4g' % d['value'], 'apply', d['apply']['ms'], d['apply']['hbm_frac'], 'e2e', d['e2e']['ms_per_step'], 'roofline', d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
for c in cfg0 cfg1; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${V}_bench_$c.json 2> gpurun_out/${V}_bench_$c.err; python -c "
import json; d=json.load(open('gpurun_out/${V}_bench_$c.json')); print('$c', d['ms_per_step'], '%.4g' % d['value'], 'apply', d['apply']['ms'], 'e2e', d['e2e']['ms_per_step'])"; done
