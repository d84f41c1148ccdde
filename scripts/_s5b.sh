timeout 90 python scripts/comm1_check.py 2>&1 | grep -v "^NCCL" | tail -12; echo "rc=$?"
