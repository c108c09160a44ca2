# r02aq A/B: ld.lu (last use) instead of ld.cg in the y-pass tile loads (libparadiag_ylu.so) and instead of ld.cs in
# the forward stage-1 input loads + inverse stage-1 spectrum loads (libparadiag_flu.so)
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag.so libparadiag_ylu.so libparadiag_flu.so; do
  for c in cfg4 cfg3; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02aq_ldlu_ab.txt
