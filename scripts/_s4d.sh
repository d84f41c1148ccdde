python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in "vb_debug=0" "vb_debug=256" "vb_debug=512" "vb_debug=0 vb_pair=0" "vb_debug=256 vb_pair=0"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep -v "^  timeline\|^   \|last commits"
done
