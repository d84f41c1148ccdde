#!/bin/bash
# wide-tile vocab backward vs V-chunk width (same box); VCS="w:vc ..." pairs
for round in 1 2; do
  for wv in ${VCS:-0:0 2:8448 2:12544 2:16896 2:25088}; do
    w=${wv%%:*}; vc=${wv##*:}
    echo -n "${CFG:-paper} wide=$w vc=$vc "; ATTN_WIDE=$w ATTN_VC=$vc timeout 120 python scripts/quick_time.py ${CFG:-paper} | tail -2 | sed "s/{.*vocab_bwd/vocab_bwd/; s/, .proj_bwd.*}//" | tr '\n' ' '; echo
  done
done
