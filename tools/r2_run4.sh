python -m pytest tests -q -m gpu -x --durations=10 > gpurun_out/r2_gpu_all.log 2>&1
tail -15 gpurun_out/r2_gpu_all.log
tools/ab_r2.sh 2>&1 | tee gpurun_out/r2_ab1.log | cut -c 1-400
for k in 9 0; do
  echo "kind $k base"; PROBE=tools/ablib/sweep_probe_base tools/power_probe.sh 0 $k
  echo "kind $k new"; tools/power_probe.sh 0 $k
done 2>&1 | tee gpurun_out/r2_probe1.log
