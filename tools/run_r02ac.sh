# r02ac: closed-form rank-1 boundary correction in the Toeplitz solvers (1D tridiag_kernel / tail1d_kernel, 2D Dirichlet
# dtri_kernel) and Stockham twiddles in the half-length DST rows: phase times, then the full GPU suite
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200
for c in cfg1 cfg2 t4a_256 t4a_512; do python tools/variant_apply.py $L/libparadiag.so $c 20 2>&1 | tail -1; done | tee gpurun_out/r02ac_phases.txt
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02ac_gpu_tests.log 2>&1; tail -5 gpurun_out/r02ac_gpu_tests.log
