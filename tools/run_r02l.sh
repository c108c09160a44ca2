# r02l: source-level ncu of the cfg4 inverse time FFT kernels (one 1 GB chunk each) + the y-pass
source tools/gpu_preflight.sh
mkdir -p gpurun_out
export PD_TF4_OVERLAP=1 PD_TF4_CHUNK_MB=1024
python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/r02l_plain.log 2>&1 &&
ncu -f --set full --clock-control none --import-source on -k regex:"tfx_inv_s1x|tf4_inv_s2" -c 2 -o /tmp/r02l python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/r02l_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02l.ncu-rep > gpurun_out/r02l_summary.txt 2>&1
ncu -i /tmp/r02l.ncu-rep --page source --csv > gpurun_out/r02l_source.csv 2>/dev/null
ls -la /tmp/r02l.ncu-rep
