python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5r_pytest_gpu.txt 2>&1; tail -2 gpurun_out/s5r_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s5r_bench_paper.log 2>&1; tail -1 gpurun_out/s5r_bench_paper.log | cut -c1-150
timeout 600 python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/s5r_bench_long.log 2>&1
timeout 600 python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/s5r_bench_large.log 2>&1
