# 4 GPUs: warm-up all-reduce round API (sim parity + real ranks + timing), and the scheduler's
# serial plan on the small models (default-mode h)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_sim_mesh.py -k warmup -q --timeout 300 2>&1 | tail -3
W="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29611"
timeout 600 $W --nproc-per-node=4 tests/mp_parity_worker.py 1x4 bf16:warm:peer:unit f32:warm:nccl:unit > gpurun_out/r2w_mp_1x4.log 2>&1; echo "mp rc=$?"; grep -c "PARITY OK" gpurun_out/r2w_mp_1x4.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/r2w_$name.json 2> gpurun_out/r2w_$name.err; echo "$name rc=$?"; }
run 7B_2x2_warm $T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --mesh 2x2 $C --overlap-tokens 0 --warmup-allreduce
run 7B_1x4_warm $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 $C --overlap-tokens 0 --warmup-allreduce
run 350M_1x4_ov $T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --model 350M $C --overlap-tokens 8192,65536 --partition -1,0
run 1B_2x2_ov $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 8192 --partition -1,0
for f in gpurun_out/r2w_*.json; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step'],3), round(d['sync_roofline']['frac_measured'],3))
w=d.get('warmup_allreduce')
if w: print('   warm', {k: round(v,2) for k,v in w['ms_per_round'].items()})
ov=d.get('overlap')
if ov:
  for x in ov['runs']: print('   ov', x['tokens_per_gpu'], x['partition_sms'], x['depth'], round(x['hidden_fraction'],3), (x['plan'] or {}).get('candidate'))
" $f; done 2>&1 | tee gpurun_out/r2w_summary.txt
