timeout 600 python -m pytest tests -m gpu -q -x -k "small or full_config_vs" > gpurun_out/pytest12.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest12.log
for mode in 0 1 2; do for c in cfg2 cfg4; do PD_TF4_MODE=$mode timeout 900 python bench.py --config $c --steps 2 --warmup 1 --apply-reps 10 --no-cpu-baseline --no-e2e > gpurun_out/b12_$c.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b12_$c.json')); p=d['phases']; print('mode $mode $c apply', d['apply']['ms'], {k:(v['ms_per_launch'],v['GBps']) for k,v in p.items() if 'tfft' in k})"; done; done
