python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4s_pytest_gpu.txt 2>&1; tail -3 gpurun_out/s4s_pytest_gpu.txt
timeout 300 python scripts/vb_sweep.py "vb_claim=0" "vb_claim=1" "vb_claim=0" "vb_claim=1" 2>&1 | grep -v Warn | cut -c1-200
timeout 600 python bench.py > gpurun_out/s4s_bench.json 2> gpurun_out/s4s_bench.err; tail -c 300 gpurun_out/s4s_bench.json
