python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k parity 2>&1 | tail -2
mkdir -p gpurun_out/san2
rm -f gpurun_out/san2/summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py > gpurun_out/san2/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san2/summary.txt
done
grep -c "Error" gpurun_out/san2/racecheck.txt
