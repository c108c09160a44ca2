python tools/prof_apply.py --config cfg4 > gpurun_out/plain9.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"tf4" -s 40 -c 4 -o gpurun_out/prof_tf4 python tools/prof_apply.py --config cfg4 > gpurun_out/ncu9.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu9.log
