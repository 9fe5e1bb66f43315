python -m pytest tests/test_gpu_parity.py tests/test_gpu_layout_swap.py tests/test_gpu_sharded.py -q -m gpu -x -k "not config_c3" 2>&1 | tail -3
tools/ab_r2.sh 2>&1 | tee gpurun_out/r2_ab2.log | cut -c 1-300
for k in 9; do
  echo "kind $k base"; PROBE=tools/ablib/sweep_probe_base tools/power_probe.sh 0 $k
  echo "kind $k new"; tools/power_probe.sh 0 $k
done 2>&1 | tee gpurun_out/r2_probe2.log
