source tools/gpu_preflight.sh
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "ivp or host" > gpurun_out/pytest61.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest61.log
timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b61.json 2> gpurun_out/b61.err; python -c "
import json; d=json.load(open('gpurun_out/b61.json')); print(d['ms_per_step'], d['e2e'])"
