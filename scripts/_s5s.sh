timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 36 -c 40 --csv --log-file gpurun_out/s5s_launches.csv python scripts/one_step.py steps=6 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"vocab_kernel|attn_|gemm_tc" -s 12 -c 8 -o gpurun_out/s5s_full python scripts/one_step.py steps=3 > gpurun_out/s5s_ncu.log 2>&1
ls gpurun_out | grep s5s
