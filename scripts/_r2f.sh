set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_paper.log 2>&1
tail -2 gpurun_out/bench_paper.log
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -15 gpurun_out/pytest_gpu.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 40 --csv --log-file gpurun_out/r02f_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:vocab_kernel -s 2 -c 1 -o gpurun_out/r02f_vocab python scripts/one_step.py steps=4 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
timeout 600 python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/bench_large.log 2>&1; tail -1 gpurun_out/bench_large.log
timeout 600 python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/bench_long.log 2>&1; tail -1 gpurun_out/bench_long.log
