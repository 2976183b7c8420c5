# 4-GPU evidence run (gpurun --gpus 4): multi-rank parity, 3B anomaly-rate sweeps, 350M, 7B overlap
mkdir -p gpurun_out
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multirank.py -x -q -k "1x4 or 2x2 or 4x1" > gpurun_out/t4_multi.log 2>&1; tail -1 gpurun_out/t4_multi.log
C="--gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 400 $T --master-port 29521 bench.py $C --model 3B --mesh 2x2 --overlap-tokens 0 --anomaly-sweep 0,0.125,0.25,0.5,1 > gpurun_out/b4_3B_2x2_anom.json 2> gpurun_out/b4_3B_2x2_anom.err; echo 3B2x2 $?
timeout 400 $T --master-port 29522 bench.py $C --model 3B --mesh 1x4 --overlap-tokens 0 --anomaly-sweep 0,0.125,0.25,0.5,1 > gpurun_out/b4_3B_1x4_anom.json 2> gpurun_out/b4_3B_1x4_anom.err; echo 3B1x4 $?
timeout 400 $T --master-port 29523 bench.py $C --model 350M --mesh 1x4 --overlap-tokens 8192 --partition 0,16 > gpurun_out/b4_350M_1x4.json 2> gpurun_out/b4_350M_1x4.err; echo 350M $?
timeout 600 $T --master-port 29524 bench.py $C --model 7B --mesh 1x4 --overlap-tokens 8192,65536 --partition 0,16 > gpurun_out/b4_7B_1x4_ov.json 2> gpurun_out/b4_7B_1x4_ov.err; echo 7B1x4 $?
