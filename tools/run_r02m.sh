# r02m: vectorised 2D stencil (2 x-points per lane) A/B on the residual + residual/matvec parity
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200/libparadiag.so
for c in cfg4 cfg3; do for v in "PD_STENCIL_V1=1" "PD_X=0"; do echo "$v $(env $v python tools/variant_resid.py $L $c 2>&1 | tail -1)"; done; done | tee gpurun_out/r02m_resid.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py tests/test_ctp01.py -m gpu -x -q -k "resid or matvec or rhs or stencil or guard or ctp01 or cfg3 or cfg4" > gpurun_out/r02m_tests.log 2>&1; tail -n 3 gpurun_out/r02m_tests.log
