python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for tok in 65536 8192; do
  timeout 600 python tools/overlap_ab.py tools/r1lib --tokens $tok --sms=0,16,32,64
  timeout 600 python tools/overlap_ab.py . --tokens $tok --sms=-1,0,16,32,64
done
