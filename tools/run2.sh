timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -40 gpurun_out/pytest_gpu.log
