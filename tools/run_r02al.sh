# r02al A/B: y-pass (slab_ytri_kernel, dtri_kernel) tile loads / stores with the default L2 policy (ld.cg / st.cg,
# libparadiag_keep.so = -DPD_SPEC_KEEP_SLAB=1) instead of evict-first (ld.cs / st.cs); the time-FFT kernels unchanged
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag.so libparadiag_keep.so; do
  for c in cfg3 cfg4 t4a_256 t4a_512; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02al_keep_slab_ab.txt
