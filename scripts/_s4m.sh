python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s4m_pytest_gpu.txt 2>&1; tail -3 gpurun_out/s4m_pytest_gpu.txt
for l in head lean2 head lean2; do echo "=== $l"; ATTNSM_LIB=$PWD/ablib/$l.so timeout 120 python scripts/vb_sweep.py "vb_fwd_fused=1" "vb_debug=0" 2>&1 | grep -v Warn | cut -c1-200; done
