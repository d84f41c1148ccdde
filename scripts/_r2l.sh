python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -3
timeout 900 python scripts/vb_sweep.py default vocab_chunk=2560 vocab_chunk=3584 vocab_chunk=4096 vocab_chunk=5120 vocab_chunk=6144 default vocab_chunk=4096 > gpurun_out/r2l_c1.log 2>&1
CFG=large timeout 900 python scripts/vb_sweep.py vocab_chunk=8192 vocab_chunk=12288 vocab_chunk=16384 vocab_chunk=6144 vocab_chunk=10240 vocab_chunk=8192 > gpurun_out/r2l_c3.log 2>&1
CFG=long timeout 900 python scripts/vb_sweep.py default vocab_chunk=2304 vocab_chunk=2816 vocab_chunk=3328 default > gpurun_out/r2l_c4.log 2>&1
cat gpurun_out/r2l_c1.log gpurun_out/r2l_c3.log gpurun_out/r2l_c4.log | cut -c1-120
