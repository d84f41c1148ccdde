for r in 1 2; do for l in head lean2; do
  echo "=== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | tail -1 | cut -c1-150
done; done
echo "=== trace lean2"; ATTNSM_LIB=$PWD/ablib/lean2.so timeout 120 python scripts/vb_trace.py 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
