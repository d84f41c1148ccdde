#!/bin/bash
# same-box A/B of library builds in ablib/ on the GEMM microbenchmark
for l in "$@"; do
  echo "== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 200 python scripts/gemm_bench.py cta_pair=0 fwd dlogits dW_out dHc 2>&1 | grep -v Warn
done
