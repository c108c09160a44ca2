# r02s: 1D stencil with warp shuffles (parity + A/B on cfg2 / cfg1), y-pass occupancy variants on cfg4, smoke
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_nonlinear.py tests/test_gpu_guard.py tests/test_gpu_dist.py tests/test_gpu_robust.py -m gpu -x -q -k "resid or matvec or rhs or stationary or cfg0 or cfg2 or cfg1 or nl or guard or dist or newton or forced" > gpurun_out/r02s_tests.log 2>&1; tail -n 3 gpurun_out/r02s_tests.log
L=paper_2005_09158_b200
for c in cfg2 cfg1; do for v in "PD_STENCIL_V1=1" "PD_X=0"; do echo "$v $(env $v python tools/variant_resid.py $L/libparadiag.so $c 2>&1 | tail -1)"; done; done | tee gpurun_out/r02s_resid.txt
for v in libparadiag libparadiag_ytri3 libparadiag_ytri3ns; do python tools/variant_apply.py $L/$v.so cfg4 5 2>&1 | tail -1; done | tee gpurun_out/r02s_ytri.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1; tail -n 2 gpurun_out/r02s_smoke.log
