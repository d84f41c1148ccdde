timeout 600 python scripts/vb_sweep.py "dl_budget_mb=120" "dl_budget_mb=200" "dl_budget_mb=120" "dl_budget_mb=200" "dl_budget_mb=120" "dl_budget_mb=200" 2>&1 | grep -v Warn | awk '{print $1, $2, $3, $6, $7}'
CFG=long timeout 600 python scripts/vb_sweep.py "dl_budget_mb=120" "dl_budget_mb=200" "dl_budget_mb=120" "dl_budget_mb=200" 2>&1 | grep -v Warn | awk '{print "long", $1, $2, $3, $6, $7}'
