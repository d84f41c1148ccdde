python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
i=0
for W in 1 0 1 0; do i=$((i+1))
timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:vocab_kernel -s 1 -c 2 --csv --log-file gpurun_out/r3n_w${W}_$i.csv python scripts/one_step.py steps=3 vb_wide=$W > /dev/null 2>&1
done
