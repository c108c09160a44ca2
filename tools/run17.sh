timeout 900 python -m pytest tests/test_gpu_dist.py -q -x > gpurun_out/pytest17.log 2>&1; echo dist rc=$?; tail -25 gpurun_out/pytest17.log
timeout 900 python -m pytest tests -m gpu -q -x -k "not dist" > gpurun_out/pytest17b.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest17b.log
