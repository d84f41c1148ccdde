M=dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum
ncu --metrics $M --clock-control none -k regex:vocab_bwd -s 2 -c 1 --csv python scripts/one_step.py > gpurun_out/ncu_vb_a.csv 2>&1
ncu --metrics $M --clock-control none -k regex:vocab_bwd -s 2 -c 1 --csv python scripts/one_step.py dl_budget_mb=48 > gpurun_out/ncu_vb_b.csv 2>&1
ncu --metrics $M --clock-control none -k regex:vocab_bwd -s 2 -c 1 --csv python scripts/one_step.py vb_debug=1 > gpurun_out/ncu_vb_c.csv 2>&1
ncu --metrics $M --clock-control none -k regex:gemm_tc -s 8 -c 3 --csv python scripts/one_step.py > gpurun_out/ncu_vb_d.csv 2>&1
