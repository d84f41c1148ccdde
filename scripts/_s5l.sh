for l in s3 s3db; do echo "== parity $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "default or g1wide or order2 or single" 2>&1 | tail -1; done
for r in 1 2 3; do for l in s3base s3 s3db; do
  echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | grep -v Warn | tail -1 | cut -c40-190
done; done
for l in s3 s3db; do echo "=== trace $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_trace.py 2>&1 | grep "G1 dl\|G3 dHc\|G2 dW\|MMA-busy"; done
