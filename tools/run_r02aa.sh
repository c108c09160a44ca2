# r02aa: persistent fused time FFT (PD_TFX_PERSIST=1) vs the default 3-stream chunk pipeline: bit-identical outputs,
# phase times on cfg3 / cfg4, oracle parity of the full cfg3 apply through the persistent path
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 300 python tools/check_persist.py cfg3 20 2>&1 | tail -8 | tee gpurun_out/r02aa_persist.txt
timeout 600 python tools/check_persist.py cfg4 10 2>&1 | tail -8 | tee -a gpurun_out/r02aa_persist.txt
PD_TFX_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "full_config or cfg3" 2>&1 | tail -3 | tee -a gpurun_out/r02aa_persist.txt
