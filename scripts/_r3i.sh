python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
ATTN_LSTM_KSPLIT=4 timeout 300 python -m pytest tests/test_gpu_lstm.py -q -x -k "backward" 2>&1 | tail -2
for K in 4 2; do for C in 1 2; do echo "== ksplit $K cluster $C"; ATTN_LSTM_KSPLIT=$K ATTN_LSTM_CLUSTER=$C timeout 200 python scripts/lstm_trace.py 2>/dev/null | tail -1; ATTN_LSTM_KSPLIT=$K ATTN_LSTM_CLUSTER=$C timeout 120 python scripts/hybrid_step.py; done; done
