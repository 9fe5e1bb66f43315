bash tools/build_probe.sh >/dev/null 2>&1 || echo build failed
for impl in 0 2; do
  for f in 0x7 0x107; do tools/sweep_probe 30 20 $impl custom 3 12 $f; done
done
for r in 1 2; do
tools/sweep_probe 30 50 0 0
tools/sweep_probe 30 50 0 9
tools/sweep_probe 30 50 0 custom 12 0 0x4
done
tools/sweep_probe check 13 22 2 2>&1 | grep -E "FAIL|check" | tail -3
