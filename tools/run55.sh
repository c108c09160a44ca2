source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest55.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest55.log
timeout 900 python bench.py > gpurun_out/b55.json 2> gpurun_out/b55.err; echo bench rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches55.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu55.log 2>&1; echo ncu-list rc=$?
timeout 1500 python tools/bench_rows.py gpurun_out/next_rows55.json > gpurun_out/rows55.log 2>&1; echo rows rc=$?
