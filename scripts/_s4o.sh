python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in "vb_debug=0" "vb_debug=8192" "vb_debug=16384" "vb_debug=24576" "vb_debug=1"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|MMA-busy"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:vocab_kernel -s 2 -c 1 python scripts/one_step.py $o 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
