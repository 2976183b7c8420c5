set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests/test_gpu_sim_mesh.py -x -q --timeout 600 2>&1 | tail -30 > gpurun_out/r2_sim.log
cat gpurun_out/r2_sim.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5
timeout 300 python __graft_entry__.py --smoke 2>&1 | tail -3
