python -m pytest tests/test_gpu_symmetric.py tests/test_gpu_sanitizers.py tests/test_gpu_layout_swap.py -q -m gpu 2>&1 | tail -8
python tools/sym_probe.py 30 10 5 2>&1 | tail -6
python tools/sym_probe.py 26 4 10 2>&1 | tail -3
