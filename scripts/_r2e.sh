python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san/summary.txt
done
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/fullsize.log 2>&1
tail -20 gpurun_out/fullsize.log
