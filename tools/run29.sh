python tools/prof_apply.py --config cfg4 --reps 0 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:tf4_fwd_s1|tfx_|tf4_inv_s2" -c 4 -o gpurun_out/ncu29_cfg4 python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu29.log 2>&1; echo ncu rc=$?
