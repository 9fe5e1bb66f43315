bash tools/profile_round.sh r09
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r09.json 2> gpurun_out/bench_r09.err
tail -1 gpurun_out/bench_r09.json | cut -c1-300
