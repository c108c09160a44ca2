timeout 900 python -m pytest tests -m gpu -q -x -k "small or cfg3 or cfg4_solve_reduced or residual" > gpurun_out/pytest5.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest5.log
for c in cfg3 cfg4; do timeout 900 python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bench5_$c.json 2> gpurun_out/bench5_$c.err; echo $c rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench5_$c.json')); print(d['ms_per_step'], d['apply']); print(json.dumps(d['phases']))"; done
