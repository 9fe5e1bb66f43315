set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g | head -2
python -m pytest tests/test_gpu_wide.py tests/test_gpu_api.py -x -q -m gpu --durations=15 > gpurun_out/r2_wide.log 2>&1
tail -30 gpurun_out/r2_wide.log
python bench.py > gpurun_out/r2_bench0.log 2>&1; tail -c 3000 gpurun_out/r2_bench0.log
