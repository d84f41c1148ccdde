python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_lstm.py -q -x -k "backward" 2>&1 | tail -2
timeout 600 python scripts/hybrid_step.py
