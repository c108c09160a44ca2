# r02ag A/B: forward stage 1 without the table prologue (twiddle tables filled behind the tile loads, Gamma as a
# geometric sequence per thread) = libparadiag_g.so, against libparadiag.so (tables -> barrier -> loads)
mkdir -p gpurun_out
L=paper_2005_09158_b200
python tools/check_tfx.py $L/libparadiag_g.so 2>&1 | tail -5 | tee gpurun_out/r02ag_check.txt
for rep in 1 2; do for lib in libparadiag.so libparadiag_g.so; do
  for c in cfg4 cfg3 cfg2 cfg1; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02ag_ab.txt
