# r02 evidence on one B200: one bench line per config (cfg0..cfg4), launch lists of the cfg2/cfg3 applies,
# ncu --set full of their kernels summarised on the box (argv: tag [configs])
set -e
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=${1:-r02a}
CFGS=${2:-"cfg0 cfg1 cfg2 cfg3 cfg4"}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$V.txt
for c in $CFGS; do
  if [ "$c" = cfg4 ]; then
    python bench.py --config cfg4 > gpurun_out/bench_${V}_cfg4.json 2> gpurun_out/bench_${V}_cfg4.err
  else
    python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${V}_$c.json 2> gpurun_out/bench_${V}_$c.err
  fi
done
for c in cfg2 cfg3; do
  python tools/prof_apply.py --config $c --reps 0 > gpurun_out/plain_$c.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${V}_$c.csv python tools/prof_apply.py --config $c --reps 0 > gpurun_out/ncu_launch_${V}_$c.log 2>&1
  ncu --set full --clock-control none --import-source on -c 12 -o /tmp/ncu_full_${V}_$c python tools/prof_apply.py --config $c --reps 0 > gpurun_out/ncu_full_${V}_$c.log 2>&1
  python tools/ncu_summary.py /tmp/ncu_full_${V}_$c.ncu-rep > gpurun_out/ncu_full_${V}_$c.txt 2>&1 || true
  sz=$(stat -c %s /tmp/ncu_full_${V}_$c.ncu-rep)
  if [ "$sz" -lt 20000000 ]; then cp /tmp/ncu_full_${V}_$c.ncu-rep gpurun_out/; fi
done
du -sh gpurun_out
