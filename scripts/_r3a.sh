python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 300 python scripts/decode_profile.py
timeout 1200 python -m pytest tests/test_gpu_decode.py tests/test_gpu_lstm.py -q -x 2>&1 | tail -4
