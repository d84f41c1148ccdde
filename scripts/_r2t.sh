python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vb_fwd_fused=1 default vb_fwd_fused=1 default vb_fwd_fused=1 2>&1 | cut -c1-230
