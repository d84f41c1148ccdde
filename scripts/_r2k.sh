python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -5
timeout 600 python scripts/vb_sweep.py default attn_fused=0 default > gpurun_out/r2k_sweep.log 2>&1; cat gpurun_out/r2k_sweep.log
for i in 1; do timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 12 --csv python scripts/one_step.py steps=4 2>/dev/null | grep -v "^==" | awk -F'","' '{print $5, $(NF)}'; done
