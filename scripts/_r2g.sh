set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python scripts/vb_trace.py > gpurun_out/r2g_trace.log 2>&1
timeout 300 python scripts/vb_trace.py vb_pair=0 > gpurun_out/r2g_trace_single.log 2>&1
timeout 900 python scripts/vb_sweep.py default vb_debug=1 vb_debug=2 vb_debug=4 vb_debug=7 \
  dl_budget_mb=48 dl_budget_mb=80 dl_budget_mb=160 "dl_buffers=2,dl_budget_mb=80" vb_l2hints=0 vb_order=0 vb_pair=0 \
  vocab_chunk=2048 vocab_chunk=4096 vocab_chunk=6144 default > gpurun_out/r2g_sweep.log 2>&1
CFG=large timeout 900 python scripts/vb_sweep.py default dl_budget_mb=48 dl_budget_mb=80 vocab_chunk=2048 vocab_chunk=4096 > gpurun_out/r2g_sweep_large.log 2>&1
timeout 300 python scripts/vb_trace.py config=large > gpurun_out/r2g_trace_large.log 2>&1
cat gpurun_out/r2g_*.log
