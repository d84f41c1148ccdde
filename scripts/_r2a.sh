set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python scripts/vb_check.py all > gpurun_out/vb_check.log 2>&1
tail -30 gpurun_out/vb_check.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/bench.log
