bash scripts/profile.sh r01k paper
/usr/local/cuda/bin/ncu -i gpurun_out/prof_r01k.ncu-rep --page raw --csv > gpurun_out/prof_r01k_raw.csv 2>/dev/null
python bench.py > gpurun_out/bench_r01k_paper.json 2> gpurun_out/bench_r01k_paper.err
python bench.py --config large --no-next --no-cpu-baseline > gpurun_out/bench_r01k_large.json 2> gpurun_out/bench_r01k_large.err
python bench.py --config long --no-next --no-cpu-baseline > gpurun_out/bench_r01k_long.json 2> gpurun_out/bench_r01k_long.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01k_ref.json 2> gpurun_out/bench_r01k_ref.err
tail -c 300 gpurun_out/bench_r01k_large.json; tail -c 300 gpurun_out/bench_r01k_long.json
