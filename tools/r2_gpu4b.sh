for g in 2 4; do
  for v in tma ldg ldg2; do EDIT_AG=$v timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0 | head -1 | sed "s/^/$v /"; done
  for v in ldg ldg2; do EDIT_AG=$v timeout 120 tools/peer_kbench 202383360 5 512 148 $g 1 | head -1 | sed "s/^/$v local_only /"; done
done > gpurun_out/r2_peer_kbench_ag.txt 2>&1
cat gpurun_out/r2_peer_kbench_ag.txt
