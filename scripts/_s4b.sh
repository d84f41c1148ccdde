python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "edge_min or attn_generic" 2>&1 | tail -2
for o in "vb_debug=0" "vb_debug=1" "vb_debug=2" "vb_debug=3" "vb_debug=4" "vb_debug=16" "vb_debug=32" "vb_debug=0"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep -v "^  timeline\|^   " 
done
