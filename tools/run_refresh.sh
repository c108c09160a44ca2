# round-end evidence refresh on one B200: bench line, launch list of the same command (first 15000 launches: ncu
# serialises ~4150 launches per cfg4 step at ~60 ms each), ncu --set full of the cfg4 apply kernels
set -e
source tools/gpu_preflight.sh
mkdir -p gpurun_out
V=${1:-v12}
python bench.py > gpurun_out/bench_$V.json 2> gpurun_out/bench_$V.err
cat gpurun_out/bench_$V.json
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 15000 --csv --log-file gpurun_out/launches_$V.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_$V.log 2>&1
for k in tf4_fwd_s1 tfx_fwd_s2x slab_ytri tfx_inv_s1x tf4_inv_s2; do
  n=$(echo "$k" | tr -dc 'a-z0-9_' | cut -c1-20)
  ncu --set full --clock-control none --import-source on -k "regex:$k" -c 1 -o gpurun_out/ncu_full_${V}_$n python tools/prof_apply.py --config cfg4 > gpurun_out/ncu_full_${V}_$n.log 2>&1
done
ls gpurun_out
