M=dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second
for h in 0 1 2 3; do
ncu --metrics $M --clock-control none -k regex:vocab_bwd -s 2 -c 1 --csv python scripts/one_step.py vb_l2hints=$h > gpurun_out/ncu_h$h.csv 2>&1
done
python scripts/vb_check.py time > gpurun_out/time_h.log 2>&1
