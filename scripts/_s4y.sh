timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "default or order2 or g1wide or nb1" 2>&1 | tail -2
for r in 1 2 3; do for l in pre_cons cons; do
  echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | grep -v Warn | tail -1 | cut -c1-170
done; done
echo "=== trace cons"; ATTNSM_LIB=$PWD/ablib/cons.so timeout 120 python scripts/vb_trace.py 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
