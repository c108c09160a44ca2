# r02c: gtsv robustness tests, TMA stage-1 parity and cfg4 A/B (PD_TMA), cfg3 with the Nt=256 fold by default
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_robust.py -m gpu -q > gpurun_out/r02c_robust.log 2>&1; tail -2 gpurun_out/r02c_robust.log
PD_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "2d or cfg4 or tfx or four" > gpurun_out/r02c_tma_parity.log 2>&1; tail -2 gpurun_out/r02c_tma_parity.log
for v in "PD_TMA=0" "PD_TMA=1" "PD_TMA=1 PD_TF4_CHUNK_MB=32" "PD_TMA=1 PD_TF4_CHUNK_MB=64 PD_TF4_OVERLAP=2" "PD_TMA=0 PD_TF4_CHUNK_MB=32"; do
  tag=$(echo $v | tr ' =' '_-')
  env $v python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_cfg4_$tag.json 2> gpurun_out/r02c_cfg4_$tag.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/r02c_cfg4_$tag.json').read().strip().splitlines()[-1])
print('$tag', d['ms_per_step'], d['apply']['ms'], {k:v['ms_per_call'] for k,v in d['phases'].items()})"
done
python bench.py --config cfg3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02c_cfg3.json 2> gpurun_out/r02c_cfg3.err
