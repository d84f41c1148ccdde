for i in 1 2; do
for W in 2 6; do echo "== wide $W"; ATTN_WIDE=$W ATTN_EV=2 python scripts/quick_time.py paper 2>&1 | tail -1; done
echo "== pair pbwd"; ATTN_PAIR=12 ATTN_EV=2 python scripts/quick_time.py paper 2>&1 | tail -1
done
