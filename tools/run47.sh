source tools/gpu_preflight.sh
timeout 1500 python tools/bench_rows.py gpurun_out/next_rows.json > gpurun_out/rows47.log 2>&1; echo rc=$?; tail -30 gpurun_out/rows47.log | cut -c1-400
