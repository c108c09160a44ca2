# r02i: single-GPU spectrum rows without owner lookup (SH=false) A/B vs the pre-refactor library; sharded parity
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200
for i in 1 2; do for v in libparadiag_prev libparadiag; do for c in cfg4 cfg3 cfg2; do python tools/variant_apply.py $L/$v.so $c 10 2>&1 | tail -1; done; done; done | tee gpurun_out/r02i_ab.txt
timeout 1500 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guard.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02i_tests.log 2>&1; tail -3 gpurun_out/r02i_tests.log
