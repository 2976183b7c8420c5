python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for L in 2 1; do
  EDIT_LANES=$L timeout 300 python tools/sched_ab.py tools/r1lib
  EDIT_LANES=$L timeout 300 python tools/sched_ab.py .
done
