timeout 600 python -m pytest tests -m gpu -q -x -k "small or full_config_vs or solve_full_config or host" > gpurun_out/pytest14.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest14.log
for mb in 16 32; do for k in 3; do PD_TF4_CHUNK_MB=$mb PD_TF4_SLOTS=$k timeout 300 python bench.py --config cfg4 --steps 1 --warmup 1 --apply-reps 6 --no-cpu-baseline --no-e2e > gpurun_out/b14.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b14.json')); p=d['phases']; print('chunk $mb MB K=$k apply', d['apply']['ms'], {k:(v['ms_per_launch'],v['GBps']) for k,v in p.items() if k in ('tfft_fwd','tfft_inv','spatial_solve')})"; done; done
timeout 300 python bench.py --config cfg2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b14_2.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b14_2.json')); p=d['phases']; print('cfg2 apply', d['apply']['ms'], {k:(v['ms_per_launch'],v['GBps']) for k,v in p.items()})"
