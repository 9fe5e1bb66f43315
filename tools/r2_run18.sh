tools/sweep_probe check 13 22 2 2>&1 | grep -E "FAIL|check:" | tail -3
for rep in 1 2; do
  for b in tools/ablib/sweep_probe_base tools/sweep_probe; do echo -n "$b: "; $b 30 300 0 custom 3 12 0x1c; done
done 2>&1 | tee gpurun_out/r2_bar.log
tools/ab_r2.sh 2>&1 | tee gpurun_out/r2_ab4.log | cut -c 1-200
python -m pytest tests/test_gpu_sanitizers.py tests/test_gpu_parity.py -q -m gpu -x -k "not config_c3" 2>&1 | tail -2
