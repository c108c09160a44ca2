# r02am A/B: L2 policy of the y-pass tile loads and stores separately (kld: loads ld.cg, kst: stores st.cg, keep: both)
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag.so libparadiag_kld.so libparadiag_kst.so libparadiag_keep.so; do
  for c in cfg4 cfg3; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02am_keep_ldst_ab.txt
