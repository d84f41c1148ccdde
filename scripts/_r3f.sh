python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for C in 1 2; do echo "== C $C"; ATTN_LSTM_CLUSTER=$C timeout 200 python scripts/lstm_trace.py; done
