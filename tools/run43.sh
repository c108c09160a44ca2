source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q -x -k "ade2d or cfg3 or cfg4 or dist or tail or ctp01 or column" > gpurun_out/pytest43.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest43.log
for c in cfg4 cfg3; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b43_$c.json 2>gpurun_out/b43_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b43_$c.json')); print('$c step', d['ms_per_step'], 'apply', d['apply']['ms'], 'tail', d['tail_form']['ms_per_step']); print({k:(v['ms_per_call'],v['GBps']) for k,v in d['phases'].items()})"; done
