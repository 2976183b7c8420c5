python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for g in 2 4; do for v in tma ldg ldgall; do EDIT_PEER_KERNELS=$v timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0 | head -1; done; done > gpurun_out/r2_peer_kbench_rs.txt 2>&1
cat gpurun_out/r2_peer_kbench_rs.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline"
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/r2b4_$name.json 2> gpurun_out/r2b4_$name.err; echo "$name rc=$?"; }
run 7B_1x2 $T --nproc-per-node 2 --master-port 29751 bench.py --gpus 2 $C --overlap-tokens 0
run 7B_1x4 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 $C
run 7B_2x2 $T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --mesh 2x2 $C --gather --warmup-allreduce
run 1B_2x2_g0 $T --nproc-per-node 4 --master-port 29720 bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 0 --no-e2e
