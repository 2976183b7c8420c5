# 4-GPU evidence run (gpurun --gpus 4): multi-rank parity on every <= 4-rank mesh, then benches
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1000 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/t4b_multi.log 2>&1; tail -1 gpurun_out/t4b_multi.log
C="--gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 500 $T --master-port 29621 bench.py $C --model 7B --mesh 1x4 --overlap-tokens 8192,65536 --partition 0,32 > gpurun_out/b4b_7B_1x4.json 2> gpurun_out/b4b_7B_1x4.err; echo 7B1x4 $?
timeout 300 $T --master-port 29622 bench.py $C --model 7B --mesh 2x2 --overlap-tokens 0 > gpurun_out/b4b_7B_2x2.json 2> gpurun_out/b4b_7B_2x2.err; echo 7B2x2 $?
timeout 300 $T --master-port 29623 bench.py $C --model 350M --mesh 1x4 --overlap-tokens 0 > gpurun_out/b4b_350M_1x4.json 2> gpurun_out/b4b_350M_1x4.err; echo 350M $?
timeout 300 $T --master-port 29624 bench.py $C --model 1B --mesh 2x2 --overlap-tokens 8192 --partition 0,32 > gpurun_out/b4b_1B_2x2.json 2> gpurun_out/b4b_1B_2x2.err; echo 1B2x2 $?
