bash scripts/profile.sh r01l paper
/usr/local/cuda/bin/ncu -i gpurun_out/prof_r01l.ncu-rep --page raw --csv > gpurun_out/prof_r01l_raw.csv 2>/dev/null
python bench.py > gpurun_out/bench_r01l_paper.json 2> gpurun_out/bench_r01l_paper.err
python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/bench_r01l_large.json 2> gpurun_out/bench_r01l_large.err
python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/bench_r01l_long.json 2> gpurun_out/bench_r01l_long.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01l_ref.json 2> gpurun_out/bench_r01l_ref.err
tail -c 300 gpurun_out/bench_r01l_large.json; tail -c 300 gpurun_out/bench_r01l_long.json
