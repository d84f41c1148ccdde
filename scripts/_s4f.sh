python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in "vb_debug=0" "vb_debug=1024" "vb_debug=2048"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
done
