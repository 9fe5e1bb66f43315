#!/bin/bash
# Merged S1 sweep (C=3, q=12, N=30) timed with parts compiled out (QB_SKIP),
# full and on-chip only (kGen | kNoStore), with SM clock / power under load.
cd "$(dirname "$0")/.."
for k in ${KS:-0 1 2 4 8 3 15}; do
  for fl in ${FLAGS:-0x1c 0x11d}; do
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/dp.log &
    P=$!
    sleep 0.3
    r=$(tools/ablib/sweep_probe_skip$k 30 ${REPS:-300} 0 custom ${C:-3} ${Q:-12} $fl)
    kill $P
    clk=$(python3 -c "
import statistics
rows=[l.split(',') for l in open('/tmp/dp.log') if l.strip()]
hot=[(float(a),float(b)) for a,b in rows if float(b)>400]
print(f'{statistics.median([h[0] for h in hot]):.0f} MHz {statistics.median([h[1] for h in hot]):.0f} W' if hot else 'idle')")
    echo "skip=$k flags=$fl: $r | $clk"
  done
done
