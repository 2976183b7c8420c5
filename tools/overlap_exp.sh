mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --overlap-steps 5 --overlap-tokens 8192 --partition 0,8,16,32"
timeout 300 env $B > gpurun_out/ov_base.json 2>/dev/null; echo base $?
EDIT_SCHED_GATE=1 timeout 300 $B > gpurun_out/ov_gate.json 2>/dev/null; echo gate $?
EDIT_LANES=1 timeout 300 $B > gpurun_out/ov_l1.json 2>/dev/null; echo l1 $?
EDIT_LANES=1 EDIT_SCHED_GATE=1 timeout 300 $B > gpurun_out/ov_l1gate.json 2>/dev/null; echo l1gate $?
