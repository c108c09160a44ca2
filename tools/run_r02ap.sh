# r02ap: round-end evidence (refresh of r02af after the graph default and the y-pass load policy) on one B200 for the final tree: full GPU suite + smoke, one bench line per config, the SURVEY
# 8(f) rows, the ncu launch list of the cfg4 bench command (first 12000 launches)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=r02ap
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${V}_smi.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${V}_gpu_tests.log 2>&1; tail -n 3 gpurun_out/${V}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${V}_smoke.log 2>&1; tail -n 1 gpurun_out/${V}_smoke.log
python bench.py > gpurun_out/${V}_bench_cfg4.json 2> gpurun_out/${V}_bench_cfg4.err
for c in cfg0 cfg1 cfg2 cfg3; do python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${V}_bench_$c.json 2> gpurun_out/${V}_bench_$c.err; done
for c in cfg0 cfg1 cfg2 cfg3 cfg4; do python -c "
import json; d=json.load(open('gpurun_out/${V}_bench_$c.json')); print('$c', d['ms_per_step'], d['config'].get('iterations'), '%.4g' % d['value'], 'apply', d['apply']['ms'], d['apply']['hbm_frac'], 'e2e', d['e2e']['ms_per_step'], 'roofline', d['roofline']['kernel'], d['roofline']['frac'])"; done | tee gpurun_out/${V}_bench_summary.txt
timeout 1500 python tools/bench_rows.py gpurun_out/${V}_next_rows.json > gpurun_out/${V}_next_rows.log 2>&1; tail -n 2 gpurun_out/${V}_next_rows.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/${V}_launches_cfg4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${V}_ncu_launch.log 2>&1
python tools/launch_summary.py gpurun_out/${V}_launches_cfg4.csv > gpurun_out/${V}_launches_cfg4_summary.txt; head -12 gpurun_out/${V}_launches_cfg4_summary.txt
gzip -f gpurun_out/${V}_launches_cfg4.csv
du -sh gpurun_out
