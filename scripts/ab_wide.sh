#!/bin/bash
# same-box A/B of the wide-tile masks (3 rounds, alternating)
for round in 1 2 3; do
  for w in 0 2 6 7; do
    echo -n "wide=$w "; ATTN_WIDE=$w timeout 100 python scripts/quick_time.py ${CFG:-paper} | tail -2 | tr '\n' ' '; echo
  done
done
