set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; tail -5 gpurun_out/r2h_smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "parity" > gpurun_out/r2h_parity.log 2>&1; tail -30 gpurun_out/r2h_parity.log
timeout 600 python scripts/vb_sweep.py default attn_fused=0 default attn_fused=0 > gpurun_out/r2h_sweep.log 2>&1
CFG=large timeout 600 python scripts/vb_sweep.py default attn_fused=0 vocab_chunk=3072 vocab_chunk=4096 vocab_chunk=6144 vocab_chunk=8192 >> gpurun_out/r2h_sweep.log 2>&1
CFG=long timeout 600 python scripts/vb_sweep.py default attn_fused=0 vocab_chunk=2048 vocab_chunk=3072 vocab_chunk=4096 vocab_chunk=6144 >> gpurun_out/r2h_sweep.log 2>&1
cat gpurun_out/r2h_sweep.log
