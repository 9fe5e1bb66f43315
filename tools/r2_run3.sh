python -m pytest tests -q -m gpu -x --durations=20 > gpurun_out/r2_gpu_all.log 2>&1
tail -40 gpurun_out/r2_gpu_all.log
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.log 2>&1; tail -c 4000 gpurun_out/r2_bench1.log
