# r02av: final check after the last loader change (single-tile inverse spectrum loads ld.lu): T4A / small-config phases,
# the whole GPU suite, smoke
source tools/gpu_preflight.sh
mkdir -p gpurun_out
for c in t4a_512 t4a_256 cfg0; do python tools/variant_apply.py paper_2005_09158_b200/libparadiag.so $c 20 2>&1 | tail -1; done | tee gpurun_out/r02av_phases.txt
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02av_gpu_tests.log 2>&1; tail -n 2 gpurun_out/r02av_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02av_smoke.log 2>&1; tail -n 1 gpurun_out/r02av_smoke.log
