for o in "vb_l2hints=7" "vb_order=2 vb_lag=8 dl_buffers=1 vocab_chunk=4096 vb_l2hints=7" "vb_order=2 vb_lag=8 vb_l2hints=7"; do
  echo "=== $o"
  timeout 300 ncu --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:vocab_kernel -s 2 -c 1 python scripts/one_step.py $o 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
timeout 300 python scripts/vb_sweep.py "vb_order=1" "vb_order=2,vb_lag=8,dl_buffers=1,vocab_chunk=4096,vb_l2hints=7" "vb_order=1" "vb_order=2,vb_lag=8,dl_buffers=1,vocab_chunk=4096,vb_l2hints=7" 2>&1 | grep -v Warn | cut -c1-200
