python tools/prof_apply.py --config cfg4 > gpurun_out/plain4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -s 5 -c 5 -o gpurun_out/prof_cfg4_v1 python tools/prof_apply.py --config cfg4 > gpurun_out/ncu4.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/ncu4.log
