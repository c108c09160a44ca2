timeout 900 python bench.py > gpurun_out/b35.json 2> gpurun_out/b35.err; echo bench rc=$?
tail -c 3000 gpurun_out/b35.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches35.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu35.log 2>&1; echo ncu-list rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:slab_cols|stencil2d|tfx_|tf4_fwd_s1|tf4_inv_s2|krylov" -c 8 -o gpurun_out/ncu35_full python tools/prof_apply.py --config cfg4 --reps 0 > gpurun_out/ncu35f.log 2>&1; echo ncu-full rc=$?
