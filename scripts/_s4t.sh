python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "order2 or default or claim0 or nb1" 2>&1 | tail -2
timeout 300 python scripts/vb_sweep.py "vb_order=1" "vb_order=2,vb_lag=8,dl_buffers=1,vocab_chunk=3072" "vb_order=1" "vb_order=2,vb_lag=8,dl_buffers=1,vocab_chunk=4096" "vb_order=1" "vb_order=2,vb_lag=8,dl_buffers=1,vocab_chunk=6144" 2>&1 | grep -v Warn | cut -c1-200
for o in "vb_order=2 vb_lag=8 dl_buffers=1 vocab_chunk=4096"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
  timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:vocab_kernel -s 2 -c 1 python scripts/one_step.py $o 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
