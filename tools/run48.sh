source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q -x -k "gmres or solve or cfg4 or t4a or dist or tail or corner" > gpurun_out/pytest48.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest48.log
timeout 600 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b48.json 2>gpurun_out/b48.err; python -c "
import json; d=json.load(open('gpurun_out/b48.json')); print('cfg4 step', d['ms_per_step'], 'apply', d['apply']['ms'], 'tail', d['tail_form']['ms_per_step']); print({k:(v['ms_per_call'],v['calls']) for k,v in d['phases'].items()})"
