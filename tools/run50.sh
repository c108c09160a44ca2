source tools/gpu_preflight.sh
timeout 900 python -m pytest tests -m gpu -q -k "host or gmres or solve_full" > gpurun_out/pytest50.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest50.log
timeout 900 python bench.py > gpurun_out/b50.json 2> gpurun_out/b50.err; echo bench rc=$?
