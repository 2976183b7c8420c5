python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
nvidia-smi topo -m | head -8
export EDIT_AEDIT_LOG=gpurun_out/r2_aedit_{mesh}.json
timeout 2400 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_aedit.py -x -q --timeout 1800 > gpurun_out/r2_multirank_core.log 2>&1; tail -5 gpurun_out/r2_multirank_core.log
for g in 2 4; do
  for t in 512 256 1024; do timeout 120 tools/peer_kbench 202383360 5 $t 148 $g 0; done
  timeout 120 tools/peer_kbench 202383360 5 512 148 $g 1
  EDIT_PEER_SMEM_KB=100 timeout 120 tools/peer_kbench 202383360 5 512 296 $g 0
done > gpurun_out/r2_peer_kbench.txt 2>&1
cat gpurun_out/r2_peer_kbench.txt
