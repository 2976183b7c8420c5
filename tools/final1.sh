# last 1-GPU validation of the round: smoke, default bench line, compute-sanitizer on smoke
mkdir -p gpurun_out
timeout 100 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke $?
timeout 240 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench $?
timeout 90 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_memcheck.log 2>&1; echo memcheck $?
timeout 90 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_racecheck.log 2>&1; echo racecheck $?
