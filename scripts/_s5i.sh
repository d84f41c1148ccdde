timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
for r in 1 2 3; do for l in lse0 lse1; do
  echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | grep -v Warn | tail -1 | cut -c40-200
done; done
