OMP_NUM_THREADS=16 timeout 1500 python tools/ctp01_rules.py gpurun_out/ctp01_oracle.json > gpurun_out/ctp01.log 2>&1; echo rc=$?; tail -8 gpurun_out/ctp01.log
