python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
for o in "vocab_chunk=1536" "vocab_chunk=2048" "vocab_chunk=2560" "vocab_chunk=3072" "vocab_chunk=4096" "vocab_chunk=2048 dl_nbuf=4" "vocab_chunk=3072 dl_nbuf=2"; do
  echo "=== $o"; timeout 120 python scripts/vb_trace.py $o 2>&1 | grep "span first\|G1 dl\|G3 dHc\|G2 dW\|MMA-busy"
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct -k regex:vocab_kernel -s 2 -c 1 python scripts/one_step.py $o 2>&1 | grep -E "dram__|gpu__time|hit_rate"
done
