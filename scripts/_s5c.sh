PYTHONFAULTHANDLER=1 timeout -s SIGABRT 120 python -u bench.py --force-comm --no-next --no-cpu-baseline --steps 2 --warmup 3 > gpurun_out/s5c.log 2>&1; echo "rc=$?"
grep -v "^NCCL" gpurun_out/s5c.log | tail -40 | cut -c1-250
