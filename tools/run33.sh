timeout 1800 python -m pytest tests/test_gpu_tail.py -q -x > gpurun_out/pytest33.log 2>&1; echo rc=$?; tail -15 gpurun_out/pytest33.log
