python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1500 python -m pytest tests/test_gpu_sim_mesh.py tests/test_gpu_aedit_sim.py -q -x --timeout 600 > gpurun_out/r2g_sim.log 2>&1; echo "sim rc=$?"; tail -25 gpurun_out/r2g_sim.log
