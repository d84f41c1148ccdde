#!/bin/bash
# same-box A/B of the CTA-pair masks (3 rounds, alternating)
for round in 1 2 3; do
  for pm in 0 4 10 14; do
    echo -n "pair=$pm "; ATTN_PAIR=$pm timeout 100 python scripts/quick_time.py paper | tail -1
  done
done
