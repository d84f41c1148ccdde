python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_decode.py -q 2>&1 | tail -2
timeout 300 python scripts/decode_profile.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 5 --csv --log-file gpurun_out/r3q_decode.csv python scripts/decode_profile.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 2 -o gpurun_out/r3q_decode_full python scripts/decode_profile.py > /dev/null 2>&1
ls gpurun_out | grep r3q
