python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4z_pytest_gpu.txt 2>&1; tail -2 gpurun_out/s4z_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/s4z_bench_paper.log 2>&1; tail -1 gpurun_out/s4z_bench_paper.log | cut -c1-400
timeout 600 python bench.py --force-comm --no-next --no-cpu-baseline > gpurun_out/s4z_bench_comm1.log 2>&1; tail -1 gpurun_out/s4z_bench_comm1.log | cut -c1-300
