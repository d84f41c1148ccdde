python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "discard" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vb_discard=1 default vb_discard=1 default vb_discard=1 2>&1 | cut -c1-230
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:vocab_kernel -c 1 --csv python scripts/one_step.py steps=2 vb_discard=1 2>/dev/null | grep vocab | awk -F'","' '{print $(NF-2), $(NF)}'
