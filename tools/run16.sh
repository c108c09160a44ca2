timeout 900 python -m pytest tests -m gpu -q -x -k "solve or host or smoke" > gpurun_out/pytest16.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest16.log
for c in cfg4 cfg3 cfg1; do timeout 600 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b16_$c.json 2>gpurun_out/b16_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b16_$c.json')); print('$c step', d['ms_per_step'], 'apply', d['apply']['ms']); print(json.dumps(d['phases']))"; tail -2 gpurun_out/b16_$c.err; done
