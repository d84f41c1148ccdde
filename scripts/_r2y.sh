python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python scripts/if_err.py paper 1
timeout 300 python scripts/if_err.py paper 0
ATTN_NVCC_EXTRA="-DLS_ACCURATE=1" python -c "from paper_1909_00562_b200 import build; build.build(force=True)"
timeout 300 python scripts/if_err.py paper 1
timeout 300 python scripts/if_err.py paper 0
