# 4 GPUs: unit groups over real ranks (CUDA IPC) -- multi-rank parity of the grouped round API,
# then refreshed bench lines (groups on, live NVLink calibration)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
W="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29611"
for spec in "1x4 bf16:many_small:peer:round bf16:ragged:peer:round bf16:nan:peer:round f32:toy:peer:reg bf16:ragged:peer:graph bf16:rollback:peer:round" \
            "2x2 bf16:many_small:peer:reg f32:toy:peer:round bf16:ragged:peer:reg bf16:nan:peer:round bf16:ragged:peer:gather bf16:ragged:peer:schedpart" \
            "1x2 f32:many_small:peer:round bf16:ragged:peer:round f32:rollback:peer:reg bf16:llama350m_sample:peer:round"; do
  set -- $spec; mesh=$1; shift
  np=$(( ${mesh%x*} * ${mesh#*x} ))
  timeout 900 $W --nproc-per-node=$np tests/mp_parity_worker.py $mesh "$@" > gpurun_out/r2g4_mp_$mesh.log 2>&1; echo "mp $mesh rc=$?"
  grep -c "PARITY OK" gpurun_out/r2g4_mp_$mesh.log
done
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline"
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/r2g4_$name.json 2> gpurun_out/r2g4_$name.err; echo "$name rc=$?"; }
run 350M_1x4 $T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --model 350M $C --overlap-tokens 8192 --no-e2e
run 350M_1x2 $T --nproc-per-node 2 --master-port 29705 bench.py --gpus 2 --model 350M $C --overlap-tokens 0 --no-e2e
run 1B_2x2 $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 8192 --no-e2e
run 1B_1x4 $T --nproc-per-node 4 --master-port 29707 bench.py --gpus 4 --model 1B $C --overlap-tokens 0 --no-e2e
run 7B_1x4 $T --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 $C --overlap-tokens 8192
run 7B_2x2 $T --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --mesh 2x2 $C --overlap-tokens 0 --no-e2e
run 3B_1x4 $T --nproc-per-node 4 --master-port 29708 bench.py --gpus 4 --model 3B $C --overlap-tokens 0 --no-e2e
for f in gpurun_out/r2g4_*.json; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r=d['roofline']; c=d.get('calibration') or {}
print(sys.argv[1], d['config']['mesh'], round(d['ms_per_step'],3), 'Troof', round(d['sync_roofline']['frac_measured'],3), 'design', round(d['design_bound']['frac'],3), r['kernel'][:10], round(r['frac'] or 0,3), r.get('frac_vs_live_allpull'), c.get('nvlink_allpull_GBps_min_over_ranks'), c.get('nccl_allreduce_busbw_GBps'))
ov=d.get('overlap')
if ov:
  for x in ov['runs']: print('   ov', x['tokens_per_gpu'], x['partition_sms'], x['depth'], round(x['hidden_fraction'],3))
" $f; done 2>&1 | tee gpurun_out/r2g4_summary.txt
