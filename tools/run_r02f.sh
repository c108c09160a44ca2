# r02f: chunk / stream sweep of the time-FFT pipeline on cfg1-cfg3 applies (phase ms per call: 0 fwd, 1 Step (b), 2 inv)
source tools/gpu_preflight.sh
mkdir -p gpurun_out
L=paper_2005_09158_b200/libparadiag.so
for c in cfg3 cfg2 cfg1; do
  for v in "PD_TF4_CHUNK_MB=16" "PD_TF4_CHUNK_MB=4" "PD_TF4_CHUNK_MB=8" "PD_TF4_CHUNK_MB=32" "PD_TF4_CHUNK_MB=64" "PD_TF4_OVERLAP=2 PD_TF4_CHUNK_MB=32" "PD_TF4_OVERLAP=4 PD_TF4_CHUNK_MB=8" "PD_TF4_OVERLAP=1 PD_TF4_CHUNK_MB=1024" "PD_GRAPH=1"; do
    echo "$c $v $(env $v python tools/variant_apply.py $L $c 20 2>&1 | tail -1)"
  done
done | tee gpurun_out/r02f_sweep.txt
