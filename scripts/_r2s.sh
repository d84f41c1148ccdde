python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_attn_shapes.py tests/test_gpu_parity.py -x -q 2>&1 | tail -8
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:lse_reduce -c 3 --csv python scripts/one_step.py steps=3 2>/dev/null | grep lse_reduce | awk -F'","' '{print $(NF)}'
