# 4 GPUs: the scheduler's default (auto) mode on the small models after the serial-plan change
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
C="--steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
run() { name=$1; shift; timeout 900 "$@" > gpurun_out/r2o_$name.json 2> gpurun_out/r2o_$name.err; echo "$name rc=$?"; }
run 350M_1x4_ov $T --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 --model 350M $C --overlap-tokens 8192,65536 --partition=-1,0
run 1B_2x2_ov $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --model 1B --mesh 2x2 $C --overlap-tokens 8192,65536 --partition=-1,0
run 350M_1x2_ov $T --nproc-per-node 2 --master-port 29707 bench.py --gpus 2 --model 350M $C --overlap-tokens 8192 --partition=-1,0
for f in gpurun_out/r2o_*.json; do python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['ms_per_step'],3), round(d['sync_roofline']['frac_measured'],3))
ov=d.get('overlap')
if ov:
  print('   t_sync', round(ov['t_sync_ms'],3), {k: round(v['ms'],3) for k,v in ov['t_sync_sched_alone_ms_by_partition'].items()})
  for x in ov['runs']: print('   ov', x['tokens_per_gpu'], x['partition_sms'], x['depth'], round(x['t_fwd_ms'],2), round(x['exposed_ms_median_pair'],3), round(x['hidden_fraction'],3), (x['plan'] or {}).get('candidate'))
" $f; done 2>&1 | tee gpurun_out/r2o_summary.txt
