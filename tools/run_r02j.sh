# r02j: 2D Dirichlet y-pass by recurrences (dtri) parity + T4A phases before/after
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dirichlet or WAVE2D or wave2d or apply_matches_oracle_small" > gpurun_out/r02j_parity.log 2>&1; tail -3 gpurun_out/r02j_parity.log
timeout 900 python -m pytest tests/test_t4a.py -m gpu -x -q > gpurun_out/r02j_t4a.log 2>&1; tail -3 gpurun_out/r02j_t4a.log
L=paper_2005_09158_b200
for v in "PD_NO_DTRI=1" "PD_X=0"; do for c in t4a_256 t4a_512; do echo "$v $(env $v python tools/variant_apply.py $L/libparadiag.so $c 10 2>&1 | tail -1)"; done; done | tee gpurun_out/r02j_t4a_phases.txt
