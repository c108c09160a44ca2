for c in cfg2 cfg3 cfg1; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo cfg4 rc=$?
for c in cfg2 cfg3 cfg1 cfg4; do echo == $c; cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done
