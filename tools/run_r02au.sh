# r02au A/B: ld.lu instead of ld.cs in the remaining read-once loaders of the time FFTs (scalar-path stage-1 input loads
# for odd S, 1D inverse stage-1 spectrum loads, single-tile FFT loads); libparadiag_old.so = before
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag_old.so libparadiag.so; do
  for c in cfg2 cfg1 t4a_512 t4a_256 cfg0; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02au_ldlu_1d_ab.txt
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "apply" 2>&1 | tail -2
