python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
mkdir -p gpurun_out/san3
rm -f gpurun_out/san3/summary.txt
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python scripts/sanitize_run.py small512 lstm_train > gpurun_out/san3/$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/san3/summary.txt
done
tail -3 gpurun_out/san3/*.txt
