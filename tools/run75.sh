source tools/gpu_preflight.sh
timeout 900 python bench.py > gpurun_out/b75.json 2> gpurun_out/b75.err; echo bench rc=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches75.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu75.log 2>&1; echo ncu-list rc=$?
