# compute-sanitizer, ONE tool per call (B200_PROFILING.md): argv tool (memcheck | racecheck | synccheck | initcheck)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
T=${1:-memcheck}
python tools/sanitize_small.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50 python tools/sanitize_small.py > gpurun_out/sanitize_$T.log 2>&1
echo "exit $?" >> gpurun_out/sanitize_$T.log
tail -5 gpurun_out/sanitize_$T.log
