python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
PYTHONFAULTHANDLER=1 timeout -s SIGABRT 300 python -u bench.py --force-comm --no-next --no-cpu-baseline > gpurun_out/s5d.log 2>&1; echo "rc=$?"
grep -v "^NCCL" gpurun_out/s5d.log | tail -3 | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/s5d.log').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['comm'], d['e2e']['value'])"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "single_rank" 2>&1 | tail -2
