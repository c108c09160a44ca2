# r02v: odd-S rows with 16-byte alignment use vector loads/stores in the four-step stage kernels: parity + A/B
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_gpu_tail.py tests/test_nonlinear.py tests/test_gpu_robust.py -m gpu -x -q -k "ADE1D or WAVE1D or cfg0 or cfg1 or cfg2 or guard or nl or newton or forced or pipeline or tail_map" > gpurun_out/r02v_tests.log 2>&1; tail -n 3 gpurun_out/r02v_tests.log
L=paper_2005_09158_b200
for i in 1 2; do for v in libparadiag_base libparadiag; do for c in cfg2 cfg1; do python tools/variant_apply.py $L/$v.so $c 20 2>&1 | tail -1; done; done; done | tee gpurun_out/r02v_ab.txt
