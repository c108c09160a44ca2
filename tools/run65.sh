source tools/gpu_preflight.sh
timeout 1500 python -m pytest tests -m gpu -q -x -k "ade2d or cfg4 or tfx or 1024 or 2048 or 4096 or dist or tail" > gpurun_out/pytest65.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest65.log
