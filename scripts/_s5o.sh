python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s5o_bench_paper.log 2>&1; tail -1 gpurun_out/s5o_bench_paper.log | cut -c1-150
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5o_bench_reference.log 2>&1
timeout 600 python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/s5o_bench_large.log 2>&1
timeout 600 python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/s5o_bench_long.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 40 --csv --log-file gpurun_out/s5o_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vocab_kernel|attn_|gemm_tc" -s 12 -c 8 -o gpurun_out/s5o_full python scripts/one_step.py steps=3 > gpurun_out/s5o_ncu.log 2>&1
ls gpurun_out | grep s5o
