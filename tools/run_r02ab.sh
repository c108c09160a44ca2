# r02ab: lag sweep of the persistent fused time FFT on cfg4 (PD_TFX_LAG x-rows between the stages; ring = lag + 5 rows of 8 MB)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
for lag in 2 3 4 6; do echo "PD_TFX_LAG=$lag"; PD_TFX_LAG=$lag timeout 600 python tools/check_persist.py cfg4 10 2>&1 | grep "persist=1" | tail -1; done | tee gpurun_out/r02ab_lag.txt
