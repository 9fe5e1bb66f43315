bash tools/build_probe.sh >/dev/null 2>&1 || echo build failed
for impl in 0 2; do
  for f in 0x7 0x107 0x5 0x105 0x3 0x103; do tools/sweep_probe 30 20 $impl custom 3 12 $f; done
done
tools/sweep_probe 30 20 0 0
tools/sweep_probe 30 20 0 9
