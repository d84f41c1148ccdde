python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vb_debug=1 vb_debug=2 vb_debug=3 vb_debug=4 vb_debug=7 \
  dl_budget_mb=48 dl_budget_mb=64 dl_budget_mb=88 dl_budget_mb=100 dl_budget_mb=160 \
  dl_buffers=2 "dl_buffers=2,dl_budget_mb=80" vb_l2hints=0 vb_l2hints=1 vb_l2hints=2 vb_order=0 \
  vocab_chunk=4096 vocab_chunk=6144 default > gpurun_out/sweep1.log 2>&1
cat gpurun_out/sweep1.log
