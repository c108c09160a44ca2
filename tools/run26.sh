python tools/prof_apply.py --config cfg4 --reps 0 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:slab|stencil2d" -c 4 -o gpurun_out/ncu27_cfg4 python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu27.log 2>&1; echo ncu rc=$?
