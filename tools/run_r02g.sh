# r02g: parity after the pd_spec refactor (fused all-to-all for the sharded path), tfx tuning variants on cfg3
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_parity.py tests/test_gpu_tail.py -m gpu -x -q > gpurun_out/r02g_parity.log 2>&1; tail -3 gpurun_out/r02g_parity.log
L=paper_2005_09158_b200
for v in libparadiag libparadiag_kpt2048 libparadiag_kpt8192 libparadiag_rm8 libparadiag_minb3; do
  python tools/variant_apply.py $L/$v.so cfg3 20 2>&1 | tail -1
  python tools/variant_apply.py $L/$v.so cfg4 5 2>&1 | tail -1
done | tee gpurun_out/r02g_variants.txt
