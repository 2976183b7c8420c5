# 4 GPUs: reduce-scatter variants -- the TMA pipeline vs the row-size-templated LDG kernel (1 or 2
# vectors per thread in flight), isolated (peer_kbench, 7B unit) and in full 7B rounds
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for g in 2 4; do
  EDIT_PEER_KERNELS=tma timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0 | head -1
  EDIT_PEER_KERNELS=ldgall EDIT_RS_LDG_P=1 timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0 | head -1
  EDIT_PEER_KERNELS=ldgall EDIT_RS_LDG_P=2 timeout 120 tools/peer_kbench 202383360 5 512 148 $g 0 | head -1
done 2>&1 | tee gpurun_out/r2rs_kbench.txt
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e --overlap-tokens 0"
for v in "ldg 2" "ldgall 1" "ldgall 2"; do set -- $v
  EDIT_PEER_KERNELS=$1 EDIT_RS_LDG_P=$2 timeout 600 $T --nproc-per-node 4 --master-port 29711 bench.py --gpus 4 $C > gpurun_out/r2rs_7B_1x4_$1_$2.json 2>/dev/null
  EDIT_PEER_KERNELS=$1 EDIT_RS_LDG_P=$2 timeout 600 $T --nproc-per-node 2 --master-port 29712 bench.py --gpus 2 $C > gpurun_out/r2rs_7B_1x2_$1_$2.json 2>/dev/null
  EDIT_PEER_KERNELS=$1 EDIT_RS_LDG_P=$2 timeout 600 $T --nproc-per-node 4 --master-port 29713 bench.py --gpus 4 --mesh 2x2 $C > gpurun_out/r2rs_7B_2x2_$1_$2.json 2>/dev/null
done
for f in gpurun_out/r2rs_7B_*.json; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step'],3), round(d['design_bound']['frac'],3), round(d['roofline_isolated']['phases_ms_per_round']['allreduce'],3))" $f; done 2>&1 | tee gpurun_out/r2rs_rounds.txt
