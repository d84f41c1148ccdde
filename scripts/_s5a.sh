for o in "config=small" "config=medium" "vb_claim=0" "vb_claim=1" "comm_max_ctas=0"; do
  echo "=== $o"; timeout 60 python scripts/comm1_check.py $o 2>&1 | grep -v "^NCCL" | tail -3; echo "rc=$?"
done
