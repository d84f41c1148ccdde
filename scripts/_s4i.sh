for r in 1 2; do for l in head base dbg; do
  echo "=== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | tail -2
done; done
for l in base dbg; do echo "=== trace $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_trace.py 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"; done
