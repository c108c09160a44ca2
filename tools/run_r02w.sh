# r02w: odd-S aligned-row vector stores in the inverse stage 2 only (forward loads reverted) + NVTX ranges: A/B, smoke
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200
for i in 1 2; do for v in libparadiag_base libparadiag; do python tools/variant_apply.py $L/$v.so cfg2 20 2>&1 | tail -1; done; done | tee gpurun_out/r02w_ab.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "WAVE1D or ADE1D or cfg2" > gpurun_out/r02w_tests.log 2>&1; tail -n 2 gpurun_out/r02w_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
