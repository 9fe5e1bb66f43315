#!/bin/bash
# Cost of the per-tile cut basis (warp 0 + barrier) per sweep kind at N=30:
# probe builds with the basis (skip0) and with a zero basis (skip64), timed
# interleaved with SM clock / power under load.  Tooling only.
cd "$(dirname "$0")/.."
for round in 1 2; do
for kind in "3 12 0x1c merged-S1" "3 12 0x7 gen-S1" "3 21 0x7 gen-S2" "3 12 0x64 last-S1" "12 0 0x4 S0"; do
  set -- $kind
  for k in 0 64; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/bp.log &
    P=$!
    sleep 0.3
    r=$(tools/ablib/sweep_probe_skip$k 30 ${REPS:-200} 3 custom $1 $2 $3)
    kill $P
    clk=$(python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/bp.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'{statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')")
    echo "$4 skip=$k: $r | $clk"
  done
done
done
