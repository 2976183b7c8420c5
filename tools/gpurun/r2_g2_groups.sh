# 2 GPUs: group cap x lanes sweep on the latency-bound small-unit configs (350M, 1B at 1x2)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
C="--gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --overlap-tokens 0"
for m in 350M 1B; do
 for cap in 0 16777216 33554432 67108864; do for l in 4 8; do
  EDIT_GROUP_NUMEL=$cap EDIT_LANES=$l timeout 300 $T --master-port 29801 bench.py --model $m $C > gpurun_out/r2g2_${m}_${cap}_${l}.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[2], round(d['ms_per_step'],3), round(d['sync_roofline']['frac_measured'],3), round(d['design_bound']['frac'],3))" gpurun_out/r2g2_${m}_${cap}_${l}.json "$m cap=$cap lanes=$l"
 done; done
done 2>&1 | tee gpurun_out/r2g2_summary.txt
