# r02at A/B: ld.lu instead of ld.cg for the stage-1 -> stage-2 scratch reads of the time FFTs (libparadiag_slu.so)
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag.so libparadiag_slu.so; do
  for c in cfg4 cfg3; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02at_scratch_ldlu_ab.txt
