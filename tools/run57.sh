source tools/gpu_preflight.sh
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()"; echo rc=$?
