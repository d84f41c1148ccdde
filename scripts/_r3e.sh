python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for C in 1 2; do
ATTN_LSTM_CLUSTER=$C timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/hyb_c$C.csv python scripts/hybrid_step.py > /dev/null 2>&1
done
for C in 1 2; do ATTN_LSTM_CLUSTER=$C timeout 120 python scripts/hybrid_step.py; done
