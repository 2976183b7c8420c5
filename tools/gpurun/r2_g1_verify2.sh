python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
free -g | head -2
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs --durations=8 > gpurun_out/r2v2_gputests.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/r2v2_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2v2_smoke.log
timeout 900 python bench.py > gpurun_out/r2v2_bench.json 2> gpurun_out/r2v2_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2v2_bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['roofline']['frac'], d['sync_roofline']['frac_measured'])
for r in d['overlap']['runs']: print(r['tokens_per_gpu'], r['partition_sms'], r['depth'], round(r['hidden_fraction'],3), (r['plan'] or {}).get('candidate'))
"
