# Round 2, 1-GPU verification at HEAD: full -m gpu suite (sim mesh incl.), smoke, default bench, launch list.
nvidia-smi -L
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rs > gpurun_out/r2v_gputests.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2v_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2v_smoke.log
timeout 900 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/r2v_bench.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2v_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --overlap-tokens 0 > gpurun_out/r2v_ncu.log 2>&1; echo "ncu rc=$?"
