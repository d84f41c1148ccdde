python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vb_debug=8 default vb_debug=8 vb_debug=1 default 2>&1 | cut -c1-230
