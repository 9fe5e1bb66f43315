python -m pytest tests/test_gpu_wide.py tests/test_gpu_api.py -q -m gpu --durations=15 > gpurun_out/r2_wide.log 2>&1
tail -30 gpurun_out/r2_wide.log
/usr/bin/time -v python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_ref.log 2> gpurun_out/r2_ref.err; tail -c 2500 gpurun_out/r2_ref.log; grep -E "Maximum resident|Elapsed" gpurun_out/r2_ref.err
