python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5v_pytest_gpu.txt 2>&1; tail -1 gpurun_out/s5v_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/s5v_bench_paper.log 2>&1; tail -1 gpurun_out/s5v_bench_paper.log | cut -c1-120
timeout 600 python bench.py --force-comm --no-next --no-cpu-baseline > gpurun_out/s5v_bench_comm.log 2>&1; echo "force-comm rc=$?"
