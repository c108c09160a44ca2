python tools/prof_apply.py --config cfg4 > gpurun_out/plain11.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tf4|slab" -s 60 -c 6 -o gpurun_out/prof_v3 python tools/prof_apply.py --config cfg4 > gpurun_out/ncu11.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu11.log
