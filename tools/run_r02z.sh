# r02z: A/B of three CTAs per SM for the 256-thread four-step tiles (forward stage 1 / inverse stage 2,
# -DPD_TF4_S1_MINB=3: 80 registers, twiddle tables through L1) against the default; ncu of the T4A row / y kernels
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200
python tools/check_tfx.py $L/libparadiag_s1m3.so 2>&1 | tail -5 | tee gpurun_out/r02z_check.txt
for rep in 1 2; do for lib in libparadiag.so libparadiag_s1m3.so; do
  python tools/variant_apply.py $L/$lib cfg4 10 2>&1 | tail -1
  PD_TF4_OVERLAP=1 PD_TF4_CHUNK_MB=1024 python tools/variant_apply.py $L/$lib cfg4 10 2>&1 | tail -1 | sed 's/^/1x1GB /'
  python tools/variant_apply.py $L/$lib cfg3 20 2>&1 | tail -1
done; done | tee gpurun_out/r02z_s1m3_ab.txt
for k in dsth_rows dtri_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -f -o /tmp/ncu_full_r02z_$k python tools/variant_apply.py $L/libparadiag.so t4a_512 1 > gpurun_out/ncu_full_r02z_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_full_r02z_$k.ncu-rep > gpurun_out/ncu_full_r02z_$k.txt 2>&1
  ncu -i /tmp/ncu_full_r02z_$k.ncu-rep --page details --csv 2>/dev/null | grep -iE "stall|Bank|Excessive|Theoretical Occ|Achieved Occ|L2 Hit|L1/TEX Hit|uncoalesced" | cut -c1-400 >> gpurun_out/ncu_full_r02z_$k.txt
done
for k in tf4_fwd_s1 tf4_inv_s2; do
  timeout 600 ncu --set full --clock-control none -k "regex:$k" -s 300 -c 1 -f -o /tmp/ncu_m3_$k python tools/variant_apply.py $L/libparadiag_s1m3.so cfg4 1 > gpurun_out/ncu_m3_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_m3_$k.ncu-rep > gpurun_out/ncu_m3_r02z_$k.txt 2>&1
done
ls gpurun_out | tail -20
