timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for r in 1 2; do for l in head lean; do
  echo "=== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | tail -1 | cut -c1-200
done; done
echo "=== trace lean"; timeout 120 python scripts/vb_trace.py 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
for o in "vb_debug=1024" "vb_debug=4096"; do echo "=== trace dbg2 $o"; ATTNSM_LIB=$PWD/ablib/dbg2.so timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|G1 dl\|MMA-busy"; done
