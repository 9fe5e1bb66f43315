#!/bin/bash
# 128 x 32 C = 3 kernel (qaoa_sweep32.cu): parity against the 256 x 16 flow
# (sweep_probe check ... 32, 1e-13), then the per-sweep policy with it (impl 3)
# and without it (impl 30) per sweep kind, with SM clock / power.  Tooling only.
cd "$(dirname "$0")/.."
tools/sweep_probe check 13 ${CHECK_HI:-24} 32 | grep -E "C= 3|check:" | tail -${CHECK_TAIL:-8}
for round in 1 2; do
for kind in "3 12 0x1c merged-S1" "3 21 0x1c merged-S2" "3 12 0x4 single-S1" "3 12 0x64 last-S1" "3 21 0x64 last-S2"; do
  set -- $kind
  for impl in 30 3; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/ab.log &
    P=$!
    sleep 0.3
    r=$(tools/sweep_probe 30 ${REPS:-200} $impl custom $1 $2 $3)
    kill $P
    clk=$(python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/ab.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'{statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')")
    echo "$4 impl=$impl: $r | $clk"
  done
done
done
