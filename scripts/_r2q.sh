python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vb_l2hints=7 default vb_l2hints=7 vb_l2hints=5 vb_l2hints=6 "vb_l2hints=7,dl_budget_mb=80" "vb_l2hints=7,dl_budget_mb=160" default vb_l2hints=7 2>&1 | cut -c1-200
