# Round 2, 4-GPU verification at HEAD: multi-rank parity (default subset, every mesh <= 4 ranks),
# A-EDiT real ranks, refreshed multi-GPU bench lines, isolated peer kernels.
nvidia-smi -L; nvidia-smi topo -m | head -6
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
export EDIT_AEDIT_LOG=gpurun_out/r2v4_aedit_{mesh}.json
timeout 2000 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_aedit.py -q --timeout 1500 -rs > gpurun_out/r2v4_multirank.log 2>&1; echo "multirank rc=$?"; tail -8 gpurun_out/r2v4_multirank.log
for g in 2 4; do for v in tma ldg; do EDIT_PEER_KERNELS=$v timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0; done; done > gpurun_out/r2v4_peer_kbench.txt 2>&1
cat gpurun_out/r2v4_peer_kbench.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline"
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/r2v4_$name.json 2> gpurun_out/r2v4_$name.err; echo "$name rc=$?"; }
run 7B_1x4 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 $C --overlap-tokens 8192,65536
run 7B_2x2 $T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --mesh 2x2 $C --gather --warmup-allreduce --overlap-tokens 8192,65536
run 7B_1x2 $T --nproc-per-node 2 --master-port 29703 bench.py --gpus 2 $C --overlap-tokens 0 --no-e2e
run 350M_1x4 $T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --model 350M $C --overlap-tokens 8192 --no-e2e
run 350M_1x2 $T --nproc-per-node 2 --master-port 29705 bench.py --gpus 2 --model 350M $C --overlap-tokens 0 --no-e2e
run 1B_2x2 $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 8192 --no-e2e
run 3B_2x2_sweep $T --nproc-per-node 4 --master-port 29707 bench.py --gpus 4 --model 3B --mesh 2x2 $C --overlap-tokens 0 --no-e2e --anomaly-sweep 0,0.125,0.25,0.5,1
for m in 350M 1B; do for gr in 0 1; do
  EDIT_GRAPH=$gr run ${m}_1x4_graph$gr $T --nproc-per-node 4 --master-port 29708 bench.py --gpus 4 --model $m $C --overlap-tokens 0 --no-e2e
done; done
