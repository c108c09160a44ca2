timeout 900 python -m pytest tests -m gpu -q -x -k "small or alpha or zero or full_config_vs or cfg4_solve_reduced or solve_full_config or host" > gpurun_out/pytest8.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest8.log
for c in cfg2 cfg4 cfg1; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench8_$c.json 2> gpurun_out/bench8_$c.err; echo $c rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench8_$c.json')); print(d['ms_per_step'], d['apply']); print(json.dumps(d['phases']))"; tail -3 gpurun_out/bench8_$c.err; done
