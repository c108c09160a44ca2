python tools/prof_apply.py --config cfg4 > gpurun_out/plain6.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"slab|tfft" -s 8 -c 4 -o gpurun_out/prof_cfg4_v2 python tools/prof_apply.py --config cfg4 > gpurun_out/ncu6.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu6.log
