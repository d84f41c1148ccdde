nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5f_pytest_gpu.txt 2>&1; tail -2 gpurun_out/s5f_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/s5f_bench_paper.log 2>&1; tail -1 gpurun_out/s5f_bench_paper.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5f_bench_reference.log 2>&1; tail -1 gpurun_out/s5f_bench_reference.log | cut -c1-200
timeout 600 python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/s5f_bench_large.log 2>&1
timeout 600 python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/s5f_bench_long.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 40 --csv --log-file gpurun_out/s5f_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vocab_kernel|attn_|gemm_tc" -s 12 -c 8 -o gpurun_out/s5f_full python scripts/one_step.py steps=3 > gpurun_out/s5f_ncu.log 2>&1
ls gpurun_out | grep s5f
