timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/pytest15.log 2>&1; echo pytest rc=$?; tail -8 gpurun_out/pytest15.log
timeout 900 python bench.py > gpurun_out/bench15_cfg4.json 2> gpurun_out/bench15_cfg4.err; echo bench rc=$?; cat gpurun_out/bench15_cfg4.json
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench15_$c.json 2>/dev/null; echo $c rc=$?; done
timeout 600 python bench.py --steps 1 --warmup 1 --apply-reps 2 --no-cpu-baseline --no-e2e > gpurun_out/plain15.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r01_cfg4.csv python bench.py --steps 1 --warmup 1 --apply-reps 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu15.log 2>&1; echo ncu rc=$?
