tools/sweep_probe check 13 22 5 2>&1 | grep -E "FAIL|check:" | tail -3
for rep in 1 2; do
for spec in "3 12 0x1c" "12 0 0x4"; do
  for impl in 0 5; do echo -n "impl $impl: "; tools/sweep_probe 30 300 $impl custom $spec; done
done; done 2>&1 | tee gpurun_out/r2_loop.log
