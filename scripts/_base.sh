set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/quick_time.py paper 2>&1 | tail -3
ATTN_SL=0 python scripts/quick_time.py paper 2>&1 | tail -3
ATTN_SL=0 ATTN_WIDE=0 ATTN_VC=2560 python scripts/quick_time.py paper 2>&1 | tail -3
ATTN_SL=0 ATTN_WIDE=0 ATTN_VC=4096 python scripts/quick_time.py paper 2>&1 | tail -3
ATTN_SL=0 ATTN_VC=4096 python scripts/quick_time.py paper 2>&1 | tail -3
