# 4 GPUs: the scheduler over unit-group items -- simulated meshes (child processes), real ranks,
# and the multi-round auto mode on 1B 2x2 (where the grouped serial plan once diverged)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_sim_mesh.py -k prefetch_scheduler -q --timeout 700 2>&1 | tail -4
W="python -m torch.distributed.run --nnodes=1 --master-addr=127.0.0.1 --master-port=29611"
timeout 600 $W --nproc-per-node=4 tests/mp_parity_worker.py 1x4 bf16:many_small:peer:sched bf16:many_small:peer:schedpart bf16:ragged:peer:sched > gpurun_out/r2s_mp_1x4.log 2>&1; echo "mp 1x4 rc=$?"; grep -c "PARITY OK" gpurun_out/r2s_mp_1x4.log
timeout 600 $W --nproc-per-node=4 tests/mp_parity_worker.py 2x2 bf16:many_small:peer:sched f32:toy:peer:schedpart > gpurun_out/r2s_mp_2x2.log 2>&1; echo "mp 2x2 rc=$?"; grep -c "PARITY OK" gpurun_out/r2s_mp_2x2.log
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 $T --nproc-per-node 4 --master-port 29706 bench.py --gpus 4 --model 1B --mesh 2x2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --overlap-tokens 8192 --partition=-1,0 > gpurun_out/r2s_1B_2x2_ov.json 2> gpurun_out/r2s_1B_2x2_ov.err; echo "1B rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2s_1B_2x2_ov.json').read().strip().splitlines()[-1]); ov=d['overlap']
print(round(d['ms_per_step'],3), 't_sync', round(ov['t_sync_ms'],3))
for x in ov['runs']: print('   ov', x['tokens_per_gpu'], x['partition_sms'], x['depth'], round(x['exposed_ms_median_pair'],3), round(x['hidden_fraction'],3), (x['plan'] or {}).get('candidate'))
"
