# 2-GPU: graph mode (opt-in) correctness + a 350M 1x2 A/B; default-path sanity at N = 2
mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "graph or round_api" > gpurun_out/g_t1.log 2>&1; tail -1 gpurun_out/g_t1.log
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
C="--gpus 2 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --overlap-tokens 0 --model 350M"
EDIT_GRAPH=1 timeout 90 $T --master-port 29701 bench.py $C > gpurun_out/g_350M_graph.json 2> gpurun_out/g_350M_graph.err; echo graph $?
timeout 90 $T --master-port 29702 bench.py $C > gpurun_out/g_350M_plain.json 2> gpurun_out/g_350M_plain.err; echo plain $?
timeout 120 $T --master-port 29703 tests/mp_parity_worker.py 1x2 bf16:ragged:peer:graph f32:toy:nccl:graph > gpurun_out/g_mp.log 2>&1; echo mp $?; grep -c "PARITY OK" gpurun_out/g_mp.log
