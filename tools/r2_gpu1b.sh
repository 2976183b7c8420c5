set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/r2_pytest_gpu.log 2>&1; tail -5 gpurun_out/r2_pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke > gpurun_out/r2_smoke.log 2>&1; tail -2 gpurun_out/r2_smoke.log
timeout 900 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; tail -c 600 gpurun_out/r2_bench1.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench1.json").read().strip().splitlines()[-1])
print("value", d["value"], "ms", d["ms_per_step"], "roof", d["roofline"]["frac"], "sync_roof", d["sync_roofline"]["frac_measured"])
ov=d.get("overlap") or {}
for r in ov.get("runs", []):
    print("ov", r["tokens_per_gpu"], r["partition_sms"], r["depth"], round(r["t_fwd_ms"],1), round(r["t_fwd_plus_sync_ms"],1), round(r["hidden_fraction"],3))
PY
