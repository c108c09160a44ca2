source tools/gpu_preflight.sh
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest73.log 2>&1; echo rc=$?; tail -2 gpurun_out/pytest73.log
