source tools/gpu_preflight.sh
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "error_paths" > gpurun_out/pytest66.log 2>&1; echo rc=$?; tail -3 gpurun_out/pytest66.log
