timeout 900 python -m pytest tests/test_gpu_lstm.py -q -x 2>&1 | tail -2
for r in 1 2; do for l in lse0 lstmg; do
  echo "== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 200 python scripts/hybrid_step.py 2>&1 | tail -4
done; done
