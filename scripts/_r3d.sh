python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for C in 2 4 1; do
  echo "== cluster $C"
  ATTN_LSTM_CLUSTER=$C timeout 300 python -m pytest tests/test_gpu_lstm.py -q -x -k "backward" 2>&1 | tail -2
  ATTN_LSTM_CLUSTER=$C timeout 120 python scripts/hybrid_step.py
done
