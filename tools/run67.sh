source tools/gpu_preflight.sh
python tools/prof_apply.py --config cfg4 --reps 0 > /dev/null || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:tfx_inv_s1|tf4_inv_s2|stencil2d" -c 5 -o gpurun_out/ncu68 python tools/prof_apply.py --config cfg4 --reps 1 > gpurun_out/ncu67.log 2>&1; echo ncu rc=$?
