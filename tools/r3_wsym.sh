python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_optimize.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -4
