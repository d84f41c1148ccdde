for r in 1 2; do for l in nospin spin3; do
  echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 200 python scripts/hybrid_step.py 2>&1 | tail -1
  echo -n "$l "; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_debug=0" 2>&1 | grep -v Warn | tail -1 | awk '{print $1,$2,$3}'
done; done
