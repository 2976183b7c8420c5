mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
C="--gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --overlap-tokens 0"
for L in 6 8; do
  EDIT_LANES=$L timeout 300 $T --master-port 2954$L bench.py $C --model 350M > gpurun_out/b2_350M_lanes$L.json 2>/dev/null; echo lanes$L $?
done
for L in 2 4; do
  EDIT_LANES=$L timeout 300 $T --master-port 2955$L bench.py $C --model 7B --steps 5 > gpurun_out/b2_7B_lanes$L.json 2>/dev/null; echo 7B lanes$L $?
  EDIT_LANES=$L timeout 300 $T --master-port 2956$L bench.py $C --model 1B --steps 5 > gpurun_out/b2_1B_lanes$L.json 2>/dev/null; echo 1B lanes$L $?
done
