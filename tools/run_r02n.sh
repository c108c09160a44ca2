# r02n: source-level ncu of the cfg2 Step (b) (tridiag_kernel) and the 1D inverse stage 1
source tools/gpu_preflight.sh
mkdir -p gpurun_out
python tools/prof_apply.py --config cfg2 --reps 0 > gpurun_out/r02n_plain.log 2>&1 &&
ncu -f --set full --clock-control none --import-source on -k regex:"tridiag_kernel|tf4_inv_s1" -c 2 -o /tmp/r02n python tools/prof_apply.py --config cfg2 --reps 0 > gpurun_out/r02n_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02n.ncu-rep > gpurun_out/r02n_summary.txt 2>&1
ncu -i /tmp/r02n.ncu-rep --page source --csv > gpurun_out/r02n_source.csv 2>/dev/null
