python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python -m pytest tests -q -m gpu -x --durations=8 > gpurun_out/r2_gpu_all2.log 2>&1; tail -12 gpurun_out/r2_gpu_all2.log
