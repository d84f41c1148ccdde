python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in vb_debug=0 vb_debug=1 vb_debug=4 vb_debug=2 vb_debug=0; do
  echo "== $o"; timeout 300 python scripts/vb_trace.py $o 2>&1 | head -6
done > gpurun_out/trace_dbg.log
cat gpurun_out/trace_dbg.log
