set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4a_pytest_gpu.txt 2>&1; tail -3 gpurun_out/s4a_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/s4a_bench.json 2> gpurun_out/s4a_bench.err; tail -c 600 gpurun_out/s4a_bench.json
timeout 300 python scripts/vb_trace.py > gpurun_out/s4a_trace.txt 2>&1; cat gpurun_out/s4a_trace.txt
