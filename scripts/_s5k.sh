python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/s5k_pytest_gpu.txt 2>&1; tail -2 gpurun_out/s5k_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/s5k_bench_paper.log 2>&1; tail -1 gpurun_out/s5k_bench_paper.log | cut -c1-200
timeout 300 python bench.py --gpus 2 > gpurun_out/s5k_bench_gpus2.log 2>&1; echo "gpus2 rc=$?"; tail -2 gpurun_out/s5k_bench_gpus2.log
