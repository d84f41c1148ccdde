python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
timeout 300 python scripts/vb_sweep.py "gemm_claim=0" "gemm_claim=1" "gemm_claim=0" "gemm_claim=1" "gemm_claim=0" "gemm_claim=1" 2>&1 | grep -v Warn | cut -c1-260
