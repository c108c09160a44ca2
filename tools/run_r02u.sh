# r02u: launch list of the cfg4 bench command (ncu gpu__time_duration, cold/serialised: compare shares)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --apply-reps 2 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/r02u_plain.json 2> gpurun_out/r02u_plain.err &&
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv --log-file gpurun_out/r02u_launches.csv $CMD > gpurun_out/r02u_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/r02u_launches.csv > gpurun_out/r02u_launches_summary.txt 2>&1
gzip -f gpurun_out/r02u_launches.csv
head -30 gpurun_out/r02u_launches_summary.txt
