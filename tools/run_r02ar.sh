# r02ar: ld.lu loaders adopted: time-FFT parity tests, cfg4 / cfg3 / cfg2 phases and bench lines
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dist.py -m gpu -x -q -k "apply or dist" > gpurun_out/r02ar_tests.log 2>&1; tail -2 gpurun_out/r02ar_tests.log
for c in cfg4 cfg3 cfg2; do python tools/variant_apply.py paper_2005_09158_b200/libparadiag.so $c 20 2>&1 | tail -1; done | tee gpurun_out/r02ar_phases.txt
python bench.py > gpurun_out/r02ar_bench_cfg4.json 2> gpurun_out/r02ar_bench_cfg4.err
python -c "
import json; d=json.load(open('gpurun_out/r02ar_bench_cfg4.json')); print('cfg4', d['ms_per_step'], '%.4g' % d['value'], 'apply', d['apply']['ms'], d['apply']['hbm_frac'], 'e2e', d['e2e']['ms_per_step'], 'roofline', d['roofline']['kernel'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
