bash tools/build_probe_variants.sh 0 16 32 48 >/dev/null 2>&1 || echo build failed
for k in 0 16 32 48; do
  for impl in 0 2; do
    for f in 0x7 0x107; do echo -n "skip=$k "; tools/ablib/sweep_probe_skip$k 30 20 $impl custom 3 12 $f; done
  done
done
