python -m pytest tests/test_gpu_optimize.py tests/test_gpu_symmetric.py -q -m gpu 2>&1 | tail -3
for s in 0 1; do python tools/opt_probe.py 26 4 300 $s; python tools/opt_probe.py 20 3 1000 $s; done
