set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python scripts/vb_trace.py > gpurun_out/vb_trace_pair.log 2>&1
timeout 300 python scripts/vb_trace.py vb_pair=0 > gpurun_out/vb_trace_single.log 2>&1
timeout 300 python scripts/vb_trace.py vb_fwd_fused=1 > gpurun_out/vb_trace_fused.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 60 --csv --log-file gpurun_out/r02a_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vocab_kernel -s 2 -c 1 -o gpurun_out/r02a_vocab python scripts/one_step.py steps=4 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
