# r02aw: ncu --set full of the y-pass after the ld.cg tile loads (compare profiles/r02y_ncu_full_cfg4.txt: 487 us, DRAM 53 %)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
k=slab_ytri
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 6 -c 1 -f -o /tmp/ncu_full_r02aw_$k python tools/prof_apply.py --config cfg4 > gpurun_out/ncu_full_r02aw_$k.log 2>&1
python tools/ncu_summary.py /tmp/ncu_full_r02aw_$k.ncu-rep > gpurun_out/ncu_full_r02aw_$k.txt 2>&1
ncu -i /tmp/ncu_full_r02aw_$k.ncu-rep --page details --csv 2>/dev/null | grep -E '"(L1/TEX Hit Rate|L2 Hit Rate|Achieved Occupancy|DRAM Throughput|Memory Throughput)"' | awk -F'","' '{print "  " $(NF-3) ": " $(NF-1) " " $(NF-2)}' | tr -d '"' >> gpurun_out/ncu_full_r02aw_$k.txt
cat gpurun_out/ncu_full_r02aw_$k.txt
