# 4-GPU bench refresh at HEAD (bench.py as the driver runs it, plus mesh / model variants)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline"
run() { name=$1; shift; timeout 600 "$@" > gpurun_out/r2b4_$name.json 2> gpurun_out/r2b4_$name.err; echo "$name rc=$?"; }
run 7B_1x4 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 $C
run 7B_2x2 $T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --mesh 2x2 $C --gather --warmup-allreduce
for g in 0 1; do
  EDIT_GRAPH=$g run 350M_1x4_g$g $T --nproc-per-node 4 --master-port 2971$g bench.py --gpus 4 --model 350M $C --overlap-tokens 0 --no-e2e
  EDIT_GRAPH=$g run 1B_2x2_g$g $T --nproc-per-node 4 --master-port 2972$g bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 0 --no-e2e
  EDIT_GRAPH=$g run 350M_1x2_g$g $T --nproc-per-node 2 --master-port 2973$g bench.py --gpus 2 --model 350M $C --overlap-tokens 0 --no-e2e
done
run 3B_2x2_anom $T --nproc-per-node 4 --master-port 29741 bench.py --gpus 4 --model 3B --mesh 2x2 $C --overlap-tokens 0 --no-e2e --anomaly-sweep 0,0.125,0.25,0.5,1
run 7B_1x2 $T --nproc-per-node 2 --master-port 29751 bench.py --gpus 2 $C --overlap-tokens 0
