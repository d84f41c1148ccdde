python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_comm_first_call.py -q 2>&1 | tail -2
echo "=== pre-fix library (expect a timeout)"
ATTNSM_LIB=$PWD/ablib/stg0.so timeout 400 python -m pytest tests/test_gpu_comm_first_call.py -q -k small -x 2>&1 | tail -3
