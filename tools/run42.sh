source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest41.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest41.log
source tools/gpu_preflight.sh
timeout 900 python bench.py > gpurun_out/b40.json 2> gpurun_out/b40.err; echo bench rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches40.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu40.log 2>&1; echo ncu-list rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:tfx_inv_s1" -c 1 -o gpurun_out/ncu40_inv python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu40f.log 2>&1; echo ncu-full rc=$?
