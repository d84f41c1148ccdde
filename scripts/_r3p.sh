python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 300 python scripts/decode_profile.py
timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum --clock-control none -s 40 -c 12 --csv --log-file gpurun_out/r3p_decode.csv python scripts/decode_profile.py > /dev/null 2>&1
