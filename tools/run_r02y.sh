# r02y: (1) parity of the half-length DST rows (2D Dirichlet Step (b)), (2) T4A phase times old / new / chunk sizes,
# (3) ncu --set full summaries of the five cfg4 apply kernels in the default 3-stream 16 MB pipeline (one launch each,
# from the second apply; the reports stay on the box, the text summaries come back), (4) T4A launch lists
source tools/gpu_preflight.sh
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "dirichlet or WAVE2D or wave2d or apply_matches_oracle_small" > gpurun_out/r02y_parity.log 2>&1; tail -3 gpurun_out/r02y_parity.log
timeout 900 python -m pytest tests/test_t4a.py tests/test_gpu_tail.py tests/test_gpu_dist.py -m gpu -x -q > gpurun_out/r02y_t4a.log 2>&1; tail -3 gpurun_out/r02y_t4a.log
L=paper_2005_09158_b200
for v in "PD_DST_FULL=1" "PD_DST_CHUNK_MB=0" "PD_DST_CHUNK_MB=16" "PD_DST_CHUNK_MB=32" "PD_DST_CHUNK_MB=64" "PD_DST_CHUNK_MB=128"; do for c in t4a_256 t4a_512; do echo "$v $(env $v python tools/variant_apply.py $L/libparadiag.so $c 10 2>&1 | tail -1)"; done; done | tee gpurun_out/r02y_t4a_phases.txt
for c in t4a_256 t4a_512; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02y_$c.csv python tools/variant_apply.py $L/libparadiag.so $c 2 > gpurun_out/launches_r02y_$c.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_r02y_$c.csv | tee gpurun_out/launches_r02y_${c}_summary.txt
done
for k in tf4_fwd_s1 tfx_fwd_s2x slab_ytri tfx_inv_s1x tf4_inv_s2; do
  SK=300; [ $k = slab_ytri ] && SK=6
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s $SK -c 1 -f -o /tmp/ncu_full_r02y_$k python tools/prof_apply.py --config cfg4 > gpurun_out/ncu_full_r02y_$k.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_full_r02y_$k.ncu-rep > gpurun_out/ncu_full_r02y_$k.txt 2>&1
  ncu -i /tmp/ncu_full_r02y_$k.ncu-rep --page details --csv 2>/dev/null | grep -iE "stall|Bank|Excessive|Theoretical Occ|Achieved Occ|L2 Hit|L1/TEX Hit" | cut -c1-300 >> gpurun_out/ncu_full_r02y_$k.txt
done
rm -f gpurun_out/*.ncu-rep
ls -la gpurun_out | tail -30
