# r02d: TMA stage-1 variants (ring depth NB / consumer groups NG) vs the register-staged tf4_fwd_s1 on cfg4
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200
for mode in "" "PD_TF4_OVERLAP=1 PD_TF4_CHUNK_MB=1024"; do
  echo "== mode: ${mode:-default 3 streams x 16 MB}"
  env $mode PD_TMA=0 python tools/variant_apply.py $L/libparadiag.so cfg4 5
  for v in libparadiag libparadiag_tma74 libparadiag_tma31 libparadiag_tma73; do
    env $mode PD_TMA=1 python tools/variant_apply.py $L/$v.so cfg4 5
  done
done 2>&1 | grep -v Warning | tee gpurun_out/r02d_variants.txt
export PD_TF4_OVERLAP=1 PD_TF4_CHUNK_MB=1024
PD_TMA=1 python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/r02d_plain.log 2>&1 &&
PD_TMA=1 ncu --set full --clock-control none --import-source on -k regex:tf4_fwd_s1 -c 2 -o /tmp/r02d_tma python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/r02d_ncu.log 2>&1
PD_TMA=0 ncu --set full --clock-control none --import-source on -k regex:tf4_fwd_s1 -c 1 -o /tmp/r02d_plain python tools/prof_apply.py --config cfg4 --reps 0 >> gpurun_out/r02d_ncu.log 2>&1
python tools/ncu_summary.py /tmp/r02d_tma.ncu-rep > gpurun_out/r02d_ncu_tma.txt 2>&1
python tools/ncu_summary.py /tmp/r02d_plain.ncu-rep > gpurun_out/r02d_ncu_plain.txt 2>&1
ncu -i /tmp/r02d_tma.ncu-rep --page source --csv > gpurun_out/r02d_tma_source.csv 2>/dev/null
ls -la /tmp/r02d_*.ncu-rep
cp /tmp/r02d_tma.ncu-rep gpurun_out/ 2>/dev/null
