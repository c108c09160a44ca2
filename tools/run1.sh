set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "small or alpha or zero or residual or spectra" > gpurun_out/pytest_small.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_small.log
cat gpurun_out/smoke.log | tail -20
