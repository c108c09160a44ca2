source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest49.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest49.log
timeout 900 python bench.py > gpurun_out/b49.json 2> gpurun_out/b49.err; echo bench rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches49.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu49.log 2>&1; echo ncu-list rc=$?
