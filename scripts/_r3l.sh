python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_lstm.py -q -k backward 2>&1 | tail -2
timeout 200 python scripts/lstm_trace.py 2>/dev/null | tail -4
timeout 120 python scripts/hybrid_step.py
