tools/sweep_probe check 13 22 4 2>&1 | grep -E "FAIL|check:" | tail -5
for spec in "3 12 0x1c" "3 12 0x4" "12 0 0x4" "5 12 0x1c"; do
  for impl in 0 4; do
    n=30; [ "$spec" = "5 12 0x1c" ] && n=33
    echo -n "impl $impl n=$n: "; tools/sweep_probe $n 300 $impl custom $spec
  done
done 2>&1 | tee gpurun_out/r2_pk1.log
