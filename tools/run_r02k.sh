# r02k: 2D Dirichlet tail form (tail map vs O3, tail GMRES vs the residual-form oracle), full tail suite
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_tail.py -m gpu -q > gpurun_out/r02k_tail.log 2>&1; tail -n 15 gpurun_out/r02k_tail.log
