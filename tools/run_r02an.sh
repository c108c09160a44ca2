# r02an A/B: ld.cg instead of ld.cs (evict-first) in two more streaming loaders: the 1D Step (b) rows (tridiag_kernel,
# libparadiag_tri.so) and the forward stage-1 input rows (tf4_fwd_s1, libparadiag_s1cg.so); libparadiag.so = y-pass loads
# ld.cg (new default)
mkdir -p gpurun_out
L=paper_2005_09158_b200
for rep in 1 2; do for lib in libparadiag.so libparadiag_tri.so libparadiag_s1cg.so; do
  for c in cfg4 cfg3 cfg2 cfg1; do python tools/variant_apply.py $L/$lib $c 20 2>&1 | tail -1; done
done; done | tee gpurun_out/r02an_ldcg_ab.txt
