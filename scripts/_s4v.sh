set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4v_pytest_gpu.txt 2>&1; tail -2 gpurun_out/s4v_pytest_gpu.txt
timeout 600 python bench.py > gpurun_out/s4v_bench_paper.log 2>&1; tail -1 gpurun_out/s4v_bench_paper.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4v_bench_reference.log 2>&1
timeout 600 python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/s4v_bench_large.log 2>&1
timeout 600 python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/s4v_bench_long.log 2>&1
timeout 300 python scripts/vb_sweep.py "vb_fwd_fused=0" "vb_fwd_fused=1" "vb_fwd_fused=0" "vb_fwd_fused=1" 2>&1 | grep -v Warn | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 40 --csv --log-file gpurun_out/s4v_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vocab_kernel|attn_|gemm_tc" -s 12 -c 8 -o gpurun_out/s4v_full python scripts/one_step.py steps=3 > gpurun_out/s4v_ncu.log 2>&1
mkdir -p gpurun_out/s4v_san
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py small small_o2 > gpurun_out/s4v_san/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/s4v_san/summary.txt
done
ls gpurun_out | grep s4v
