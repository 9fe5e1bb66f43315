#!/bin/bash
# Cache-policy variants (tools/build_ld_variants.sh) on the merged S1 and S0 sweeps.
cd "$(dirname "$0")/.."
for spec in "3 12 0x1c" "12 0 0x4" "3 12 0x1c"; do
  set -- $spec
  for k in ${KS:-0 1 2}; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/dp.log &
    P=$!
    sleep 0.3
    r=$(tools/ablib/sweep_probe_ld$k 30 ${REPS:-300} 0 custom $1 $2 $3)
    kill $P
    clk=$(python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/dp.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'{statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')")
    echo "ld=$k: $r | $clk"
  done
done
