# r02h: sharded corner-identity GMRES (virtual ranks), red-zone tests, refactor A/B on cfg4, cfg2 kernel profile
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dist.py tests/test_gpu_guard.py -m gpu -q > gpurun_out/r02h_tests.log 2>&1; tail -3 gpurun_out/r02h_tests.log
L=paper_2005_09158_b200
for i in 1 2; do for v in libparadiag_prev libparadiag; do python tools/variant_apply.py $L/$v.so cfg4 10 2>&1 | tail -1; done; done | tee gpurun_out/r02h_ab.txt
python tools/prof_apply.py --config cfg2 --reps 0 > gpurun_out/r02h_plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:"tridiag|tf4_inv|tf4_fwd" -c 5 -o /tmp/r02h_cfg2 python tools/prof_apply.py --config cfg2 --reps 0 > gpurun_out/r02h_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02h_cfg2.ncu-rep > gpurun_out/r02h_ncu_cfg2.txt 2>&1
ncu -i /tmp/r02h_cfg2.ncu-rep --page source --csv > gpurun_out/r02h_cfg2_source.csv 2>/dev/null
