python tools/prof_apply.py --config cfg4 --reps 0 > /dev/null || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:tfx_inv|tf4_inv_s2|slab_cols|stencil2d" -c 11 -o gpurun_out/ncu36_full python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu36f.log 2>&1; echo ncu-full rc=$?
