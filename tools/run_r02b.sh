set -x
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_robust.py tests/test_nonlinear.py -m gpu -x -q > gpurun_out/r02b_robust.log 2>&1
tail -3 gpurun_out/r02b_robust.log
for v in 0 1; do
  PD_TFX_SMALL=$v python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r02b_cfg3_tfx$v.json 2> gpurun_out/r02b_cfg3_tfx$v.err
done
PD_TFX_SMALL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cfg3 or 2d or slab" > gpurun_out/r02b_tfxsmall_parity.log 2>&1
tail -3 gpurun_out/r02b_tfxsmall_parity.log
