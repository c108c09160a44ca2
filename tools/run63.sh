source tools/gpu_preflight.sh
python tools/prof_apply.py --config cfg4 --reps 0 > /dev/null || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:tfx_" -c 2 -o gpurun_out/ncu63 python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu63.log 2>&1; echo ncu rc=$?
