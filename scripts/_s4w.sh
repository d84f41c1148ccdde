python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "g1wide or default" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "c1_full_oracle and g1wide" 2>&1 | tail -2
timeout 300 python scripts/vb_sweep.py "vb_g1wide=0" "vb_g1wide=1" "vb_g1wide=0" "vb_g1wide=1" "vb_g1wide=0" "vb_g1wide=1" 2>&1 | grep -v Warn | cut -c1-200
for o in "vb_g1wide=1"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
  timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:vocab_kernel -s 2 -c 1 python scripts/one_step.py $o 2>&1 | grep -E "dram__|gpu__time|hit_rate|tensor"
done
