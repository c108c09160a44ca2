# full GPU test suite + smoke (the round-end driver's checks)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=${1:-full}
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${V}_gpu_tests.log 2>&1; tail -n 5 gpurun_out/${V}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${V}_smoke.log 2>&1; tail -n 2 gpurun_out/${V}_smoke.log
