# Measurements queued for the next round (run with gpurun --gpus 4; ~15 min of wall time).
#   1. the opt-in CUDA-graph round replay (EDIT_GRAPH=1) vs plain launches, small and large units
#   2. multi-rank parity of every case on every <= 4-rank mesh (EDIT_TEST_FULL=1)
#   3. refreshed 4-GPU bench lines with the current defaults
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --overlap-tokens 0"
for m in 350M 1B; do
  for g in 0 1; do
    EDIT_GRAPH=$g timeout 300 $T --nproc-per-node 2 --master-port 2981$g bench.py --gpus 2 $C --model $m \
      > gpurun_out/nr_${m}_1x2_graph$g.json 2> gpurun_out/nr_${m}_1x2_graph$g.err; echo "$m 1x2 graph=$g $?"
    EDIT_GRAPH=$g timeout 300 $T --nproc-per-node 4 --master-port 2982$g bench.py --gpus 4 $C --model $m --mesh 2x2 \
      > gpurun_out/nr_${m}_2x2_graph$g.json 2> gpurun_out/nr_${m}_2x2_graph$g.err; echo "$m 2x2 graph=$g $?"
  done
done
EDIT_TEST_FULL=1 timeout 2400 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/nr_multirank_full.log 2>&1
tail -1 gpurun_out/nr_multirank_full.log
